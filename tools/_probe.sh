cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_multigpu_gpu.py -x -q -k "P3000017 or P4000037 or P1500007 or P777777 or P30007" 2>&1 | tail -1
for G in 2 4; do for nb in 8 10; do
echo "G=$G NB=$nb $(BFLY_FUSED_NB=$nb timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port $((29000 + G * 100 + nb)) tools/ring_fused_probe.py 2>&1 | grep '^{"rank": 0' | cut -c1-40)"
done; done
