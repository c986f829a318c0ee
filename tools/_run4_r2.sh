mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo4_r2.txt 2>&1
timeout 900 python -m pytest tests/test_multigpu_gpu.py tests/test_multigpu_fuzz_gpu.py -q -m gpu --timeout 400 -p no:cacheprovider -rf -k "not loopback" > gpurun_out/pytest_multigpu4_r2.log 2>&1; echo rc=$? >> gpurun_out/pytest_multigpu4_r2.log
for N in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/bench_n${N}_c3_r2.json 2> gpurun_out/bench_n${N}_c3_r2.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --config c5 --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_n4_c5_r2.json 2> gpurun_out/bench_n4_c5_r2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 4 --impl reference --steps 3 --warmup 3 > gpurun_out/bench_n4_ref_r2.json 2> gpurun_out/bench_n4_ref_r2.err
