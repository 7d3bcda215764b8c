#!/bin/bash
# round-end evidence: full GPU suite, smoke, default bench line, reference arm, Table I
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rs > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench_exit=$? >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo ref_exit=$? >> gpurun_out/bench_ref.err
timeout 600 python bench.py --table1 > gpurun_out/table1.json 2> gpurun_out/table1.err; echo table1_exit=$? >> gpurun_out/table1.err
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; tail -1 gpurun_out/bench.err; tail -1 gpurun_out/bench_ref.err; tail -1 gpurun_out/table1.err
