#!/bin/bash
# Session-4 final check of the committed build (outputs under gpurun_out/).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/f4_pytest.log 2>&1; echo pytest_exit=$? >> gpurun_out/f4_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/f4_pytest.log 2>&1
for w in s f; do
  timeout 600 python bench.py --workload $w > gpurun_out/f4_bench_$w.json 2> gpurun_out/f4_bench_$w.err
done
timeout 900 python bench.py > gpurun_out/f4_bench_p3.json 2> gpurun_out/f4_bench_p3.err
echo done
