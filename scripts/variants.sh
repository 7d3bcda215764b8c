#!/bin/bash
# probe each library variant in build/ (dev experiment)
for v in ${VARIANTS:-b512 b256 b128 b256m3 b512m1}; do
  echo "== $v" >> gpurun_out/variants.log
  SPCG_LIB=build/libspcg_$v.so SPCG_TRACE=1 timeout 300 python scripts/probe.py ${PROBE:-P3 F} >> gpurun_out/variants.log 2>&1
done
