mkdir -p gpurun_out
i=0
for root in ab_r1 . ab_v1 ab_v2 ab_r1 .; do
  i=$((i+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2961$i tools/phase_probe.py $root > gpurun_out/phase_$i.json 2>&1
done
