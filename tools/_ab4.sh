mkdir -p gpurun_out
rm -f gpurun_out/sweep_ring.log
for t in '{}' '{"slots": 8}' '{"slots": 12}' '{"slots": 14}' '{"lag": 2}' '{"slots": 12, "lag": 2}' '{"pub_every": 2, "slots": 12}' '{}'; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --ring-tuning "$t" > gpurun_out/sweep_one.json 2>&1
tail -1 gpurun_out/sweep_one.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', round(d['ms_per_step'],3))" >> gpurun_out/sweep_ring.log 2>&1
done
