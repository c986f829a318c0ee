# config 5 on 4 GPUs: where the stats warps' cost comes from (build/ab/<V>: package copies
# built from a scratch edit of bfly_ring.cu, not kept in the tree — D: ring_stats frees
# each entry without computing (the queue alone); N: stats_offer's admit forced to 0, so
# the compute warps run the admit barriers but never enqueue; F: the tree as is)
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
run N_$i build/ab/N --fuse-stats
done
