mkdir -p gpurun_out
for fs in "" "--fuse-stats"; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --config c5 --steps 20 --warmup 5 --no-e2e $fs > gpurun_out/bench_n4_c5_r2d$fs.json 2>&1
done
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q -m gpu --timeout 400 -p no:cacheprovider -rf -k "P2000029" > gpurun_out/pytest_fuse_r2d.log 2>&1; echo rc=$? >> gpurun_out/pytest_fuse_r2d.log
