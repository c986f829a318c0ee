cd $GRAFT_REPO_ROOT
for cfg in "16 1" "16 3" "32 1" "32 3" "64 1"; do
  set -- $cfg
  echo "NB=$1 LAG=$2 G=4: $(BFLY_FUSED_NB=$1 BFLY_RING_LAG=$2 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 tools/ring_fused_probe.py 2>&1 | grep '^{"rank": 0' | cut -c1-60)"
done
echo "NB=32 LAG=1 G=2: $(BFLY_FUSED_NB=32 BFLY_RING_LAG=1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 tools/ring_fused_probe.py 2>&1 | grep '^{"rank": 0' | cut -c1-60)"
