mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_multigpu_gpu.py -q -m gpu --timeout 400 -p no:cacheprovider -rf -x -k "not sharded" > gpurun_out/pytest_r2o.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2o.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29617 tools/phase_probe.py . > gpurun_out/phase_c5_r2o.json 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --config c5 --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_n4_c5_r2o.json 2>&1
timeout 600 python bench.py --config c5 --no-e2e --no-cpu > gpurun_out/bench_n1_c5_r2o.json 2>&1
