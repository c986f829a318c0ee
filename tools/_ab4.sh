mkdir -p gpurun_out
for i in 1 2; do
  (cd ab_r1 && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2961$i bench.py --gpus 4 --config c5 --steps 20 --warmup 5 --no-e2e > ../gpurun_out/ab_r1_c5_$i.json 2>&1)
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2962$i bench.py --gpus 4 --config c5 --steps 20 --warmup 5 --no-e2e > gpurun_out/ab_r2_c5_$i.json 2>&1
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2963$i bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e > gpurun_out/ab_r2_c3_$i.json 2>&1
done
