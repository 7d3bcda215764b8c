#!/bin/bash
# A/B library variants on the probe (dev experiment): VARIANTS="base dg" PROBE="P3 F"
mkdir -p gpurun_out
for rep in 1 2; do
for v in ${VARIANTS:-base dg}; do
  echo "== $v" >> gpurun_out/ab.log
  SPCG_LIB=build/libspcg_$v.so timeout 300 python scripts/probe.py ${PROBE:-P3 F} >> gpurun_out/ab.log 2>&1
done
done
