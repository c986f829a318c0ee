# k_reduce tile order: grid-stride (G, the tree) vs chunked per CTA (C: every wave samples
# the whole range, so special and fast tiles mix on the SMs) — config 2 and 5 on one GPU
mkdir -p gpurun_out; rm -f gpurun_out/ab_tile.log
for i in 1 2; do for v in G C; do for c in c5 c2; do
  timeout 600 python build/ab/$v/bench.py --config $c --no-e2e --no-cpu > gpurun_out/ab_one.json 2>/dev/null
  tail -1 gpurun_out/ab_one.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])" >> gpurun_out/ab_tile.log
done; done; done
