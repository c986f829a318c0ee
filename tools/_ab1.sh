mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 400 -p no:cacheprovider -rf -x > gpurun_out/pytest_gpu_r2l.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_r2l.log
for i in 1 2; do
  timeout 600 python bench.py --config c5 --no-e2e --no-cpu --steps 10 > gpurun_out/ab1_cur_c5_$i.json 2>&1
  timeout 600 python bench.py --no-e2e --no-cpu --steps 10 > gpurun_out/ab1_cur_c2_$i.json 2>&1
done
