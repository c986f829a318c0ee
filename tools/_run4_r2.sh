mkdir -p gpurun_out
for N in 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --timing > gpurun_out/bench_n${N}_c3_r2b.json 2> gpurun_out/bench_n${N}_c3_r2b.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --config c5 --steps 20 --warmup 5 --no-e2e --timing > gpurun_out/bench_n4_c5_r2b.json 2> gpurun_out/bench_n4_c5_r2b.err
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q -m gpu --timeout 400 -p no:cacheprovider -rf -k "not loopback and (P2000039 or P600011 or P400009 or P300007)" > gpurun_out/pytest_multigpu4_r2b.log 2>&1; echo rc=$? >> gpurun_out/pytest_multigpu4_r2b.log
