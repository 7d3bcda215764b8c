# engine-6 check: A/B timing (in-tree vs ab/<libs>), correctness tests, stress
bash scripts/gpu_ab6.sh "$@" > gpurun_out/ab6.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "pipe or clus or cond or random or reference or engine" > gpurun_out/mbar_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/mbar_tests.log
timeout 600 python scripts/clus_stress.py 200 6 > gpurun_out/stress6.log 2>&1; cat gpurun_out/stress6.log
