mkdir -p gpurun_out
i=0
for root in ab_r1 . ab_r1 .; do
  i=$((i+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2961$i tools/phase_probe.py $root > gpurun_out/phase_$i.json 2>&1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29619 tools/phase_probe.py . 16 0 > gpurun_out/phase_c3.json 2>&1
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q -m gpu --timeout 400 -p no:cacheprovider -rf > gpurun_out/pytest_multigpu4_r2k.log 2>&1; echo rc=$? >> gpurun_out/pytest_multigpu4_r2k.log
