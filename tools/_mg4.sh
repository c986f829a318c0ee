cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_multigpu_gpu.py tests/test_multigpu_fuzz_gpu.py -x -q > gpurun_out/mg_pytest4.log 2>&1; echo rc=$? >> gpurun_out/mg_pytest4.log; tail -3 gpurun_out/mg_pytest4.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29545 bench.py --gpus 4 --config c5 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_c5_g4.log 2>&1
echo "C5 G=4 $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_c5_g4.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/bench_c5_g4.log)"
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29546 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_c2_g4.log 2>&1
echo "C2 G=4 $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_c2_g4.log | head -2) $(grep -o '"frac": [0-9.]*' gpurun_out/bench_c2_g4.log)"
