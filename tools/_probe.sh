cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_multigpu_gpu.py tests/test_multigpu_fuzz_gpu.py -x -q 2>&1 | tail -1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29710 bench.py --gpus 4 --config c5 --no-e2e --steps 5 --timing 2>&1 | grep -o 'phases.*\|"ms_per_step": [0-9.]*' | tail -2
