cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/final_pytest_gpu.log; tail -2 gpurun_out/final_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_bench_n1.log 2>&1; tail -1 gpurun_out/final_bench_n1.log | cut -c1-300
timeout 600 python bench.py --impl reference > gpurun_out/final_bench_ref.log 2>&1
for G in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port $((29700 + G)) bench.py --gpus $G > gpurun_out/final_bench_n$G.log 2>&1
echo "N=$G $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/final_bench_n$G.log | head -2 | tr '\n' ' ') $(grep -o '"frac": [0-9.]*' gpurun_out/final_bench_n$G.log)"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29710 bench.py --gpus 4 --config c5 --no-e2e > gpurun_out/final_bench_c5_n4.log 2>&1
echo "C5 N=4 $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/final_bench_c5_n4.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/final_bench_c5_n4.log)"
