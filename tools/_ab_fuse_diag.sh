# config 5 on 4 GPUs: the stats-warps variants (build/ab/<V>: F full, D dequeue only, W1 one stats warp) vs plain
mkdir -p gpurun_out
rm -f gpurun_out/ab_diag.log
run() {  # $1 tag, $2 root, rest: bench args
  tag=$1; r=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) $r/bench.py --gpus 4 --config c5 --steps 20 --warmup 5 --no-e2e --no-cpu "$@" > gpurun_out/ab_one.json 2> gpurun_out/ab_one.err
  tail -1 gpurun_out/ab_one.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> gpurun_out/ab_diag.log 2>&1
}
for i in 1 2; do
run plain_$i build/ab/F
run F_$i build/ab/F --fuse-stats
run D_$i build/ab/D --fuse-stats
run W1_$i build/ab/W1 --fuse-stats
done
