# config 5 on 4 / 2 GPUs: FINISH's k_stats after the ring vs the stats warps inside it
mkdir -p gpurun_out
rm -f gpurun_out/ab_fuse.log
run() {  # $1 tag, $2 gpus, rest: bench args
  tag=$1; g=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $g --config c5 --steps 20 --warmup 5 --no-e2e "$@" > gpurun_out/ab_one.json 2> gpurun_out/ab_one.err
  tail -1 gpurun_out/ab_one.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', round(d['ms_per_step'],3), d['roofline']['frac'], d['clocks'])" >> gpurun_out/ab_fuse.log 2>&1
  cp gpurun_out/ab_one.json gpurun_out/ab_$tag.json
}
run n4_plain_1 4
run n4_fuse_1 4 --fuse-stats
run n4_plain_2 4
run n4_fuse_2 4 --fuse-stats
run n2_plain_1 2
run n2_fuse_1 2 --fuse-stats
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29951 tools/phase_probe.py . 16 6 10 fuse > gpurun_out/phase_c5_fuse.json 2>&1
