cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_multigpu_gpu.py tests/test_multigpu_fuzz_gpu.py -x -q > gpurun_out/mg_pytest4.log 2>&1; echo rc=$? >> gpurun_out/mg_pytest4.log; tail -3 gpurun_out/mg_pytest4.log
for G in 2 4; do
BFLY_RING_PROFILE=1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2953$G tools/ring_fused_probe.py 2>&1 | grep '^{'
done
