mkdir -p gpurun_out
for fs in "" "--fuse-stats" "" "--fuse-stats"; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --config c5 --steps 20 --warmup 5 --no-e2e $fs > gpurun_out/ab_fs$fs.json 2>&1
tail -1 gpurun_out/ab_fs$fs.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$fs', round(d['ms_per_step'],3))" >> gpurun_out/ab_fs.log
done
