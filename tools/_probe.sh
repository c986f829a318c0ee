cd $GRAFT_REPO_ROOT
for G in 2 4; do for nb in 10 14 20; do
echo "G=$G NB=$nb $(BFLY_FUSED_NB=$nb timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port $((29000 + G * 100 + nb)) tools/ring_fused_probe.py 2>&1 | grep '^{"rank": 0' | cut -c1-40)"
done; done
