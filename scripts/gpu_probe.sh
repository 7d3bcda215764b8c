#!/bin/bash
mkdir -p gpurun_out
SPCG_TRACE=1 timeout 900 python scripts/probe.py ${PROBE:-F P3 Q27F Q27P Q27} > gpurun_out/probe.log 2>&1; echo probe_exit=$? >> gpurun_out/probe.log
