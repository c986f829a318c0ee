# end-of-round 4-GPU evidence with the final code
mkdir -p gpurun_out
P=29800
b() { tag=$1; g=$2; shift 2; P=$((P+1)); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port $P bench.py --gpus $g "$@" > gpurun_out/r02_final_$tag.json 2> gpurun_out/r02_final_$tag.err; }
b n4_c5 4 --config c5 --steps 20 --warmup 5 --no-e2e
b n4_c3 4 --steps 20 --warmup 5
b n2_c5 2 --config c5 --steps 20 --warmup 5 --no-e2e
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29899 tools/phase_probe.py . 16 6 10 > gpurun_out/r02_final_phase_c5.json 2>&1
for f in gpurun_out/r02_final_n*.json; do echo $f; tail -n1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d.get('ms_per_step'), d.get('value'), (d.get('roofline') or {}).get('frac'), d.get('clocks'), (d.get('e2e') or {}).get('value'))"; done
tail -n1 gpurun_out/r02_final_phase_c5.json
