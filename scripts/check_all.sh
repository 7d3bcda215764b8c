mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/f_pytest.log 2>&1; echo pytest_exit=$? >> gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/f_smoke.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --engine sharded --workload q27 --steps 3 --warmup 3 > gpurun_out/f_sh_q27.json 2> gpurun_out/f_sh_q27.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --engine sharded --workload p3 --steps 3 --warmup 3 > gpurun_out/f_sh_p3.json 2> gpurun_out/f_sh_p3.err
