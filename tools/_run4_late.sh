# late round-2 evidence on a 4-GPU box (after the k_stats change)
mkdir -p gpurun_out
P=29700
b() { tag=$1; g=$2; shift 2; P=$((P+1)); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port $P bench.py --gpus $g "$@" > gpurun_out/r02_late_$tag.json 2> gpurun_out/r02_late_$tag.err; }
b n4_c3 4 --steps 20 --warmup 5
b n4_c5 4 --config c5 --steps 20 --warmup 5 --no-e2e
b n2_c3 2 --steps 20 --warmup 5
b n2_c5 2 --config c5 --steps 20 --warmup 5 --no-e2e
b n4_ref 4 --impl reference --steps 5 --warmup 3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29799 tools/phase_probe.py . 16 6 10 > gpurun_out/r02_late_phase_c5.json 2>&1
for f in gpurun_out/r02_late_*.json; do echo $f; tail -n1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d.get('ms_per_step'), d.get('value'), (d.get('roofline') or {}).get('frac'), d.get('clocks'), (d.get('e2e') or {}).get('value'))" 2>/dev/null || tail -n1 $f | cut -c1-400; done
