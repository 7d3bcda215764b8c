#!/bin/bash
# parity tests + traced probe (run under gpurun from the repo root)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
SPCG_TRACE=1 timeout 600 python scripts/probe.py ${PROBE:-F S SA CSC P3 Q27 Q27P} > gpurun_out/probe.log 2>&1; echo probe_exit=$? >> gpurun_out/probe.log
