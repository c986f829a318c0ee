# persistent ring stage depths on 4 GPUs, config 3 (build/ab/<V>: B the tree; O5 / O6 out
# stages 5 / 6; A5 incoming running-sum stages 5)
mkdir -p gpurun_out; rm -f gpurun_out/ab_stages.log
for i in 1 2; do for v in B O5 O6 A5; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) build/ab/$v/bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/ab_one.json 2> gpurun_out/ab_one.err
  tail -1 gpurun_out/ab_one.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])" >> gpurun_out/ab_stages.log 2>&1
done; done
