cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_multigpu_gpu.py -x -q > gpurun_out/mg_pytest4.log 2>&1; echo rc=$? >> gpurun_out/mg_pytest4.log; tail -3 gpurun_out/mg_pytest4.log
for G in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2954$G bench.py --gpus $G --steps 10 --warmup 3 > gpurun_out/bench_fused_g$G.log 2>&1
  echo "G=$G $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_fused_g$G.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/bench_fused_g$G.log)"
done
for nb in 10 12; do
echo "NB=$nb G=4: $(BFLY_FUSED_NB=$nb timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 tools/ring_fused_probe.py 2>&1 | grep '^{"rank": 0' | cut -c1-60)"
done
