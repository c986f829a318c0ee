cd $GRAFT_REPO_ROOT
for G in 2 4; do
BFLY_RING_PROFILE=1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2953$G tools/ring_fused_probe.py 2>&1 | grep '^{'
done
