cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_all.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_all.log; tail -3 gpurun_out/pytest_gpu_all.log
for G in 2 4; do for nb in 6 8 10 12; do
echo "G=$G NB=$nb: $(BFLY_FUSED_NB=$nb timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2953$nb tools/ring_fused_probe.py 2>&1 | grep '^{"rank": 0' | cut -c1-45)"
done; done
timeout 300 python bench.py --config c4 --no-e2e --no-cpu --steps 5 > gpurun_out/bench_c4.log 2>&1; grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*\|"gpu_launches": [0-9]*' gpurun_out/bench_c4.log
