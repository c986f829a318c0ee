cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/final_pytest_gpu.log; tail -2 gpurun_out/final_pytest_gpu.log
for G in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port $((29700 + G)) bench.py --gpus $G > gpurun_out/final_bench_n$G.log 2>&1
echo "N=$G $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/final_bench_n$G.log | head -2 | tr '\n' ' ') $(grep -o '"frac": [0-9.]*' gpurun_out/final_bench_n$G.log) $(grep -o '"gpu_launches": [0-9]*' gpurun_out/final_bench_n$G.log)"
done
echo "G=4 NB=12 $(BFLY_FUSED_NB=12 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29412 tools/ring_fused_probe.py 2>&1 | grep '^{"rank": 0' | cut -c1-40)"
