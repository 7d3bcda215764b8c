#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --engine sharded --steps 3 --warmup 1 > gpurun_out/bench_sharded.log 2>&1; echo exit=$? >> gpurun_out/bench_sharded.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --engine sharded --workload q27 --steps 2 --warmup 1 > gpurun_out/bench_sharded_q27.log 2>&1; echo exit=$? >> gpurun_out/bench_sharded_q27.log
