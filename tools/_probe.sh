cd $GRAFT_REPO_ROOT
BFLY_RING_PROFILE=1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 tools/ring_fused_probe.py 2>&1 | grep '^{' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['rank'], d['round_ms'], d.get('cta_ms'))"
BFLY_RING_TIMING=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e 2>&1 | grep -o 'phases.*\|"ms_per_step": [0-9.]*'
