mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 400 -p no:cacheprovider -rf > gpurun_out/pytest_gpu_final1.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_final1.log
timeout 900 python bench.py > gpurun_out/bench_n1_final.json 2> gpurun_out/bench_n1_final.err
timeout 600 python bench.py --config c5 --no-e2e --no-cpu > gpurun_out/bench_n1_c5_final.json 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_final.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_n1_final.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_reduce --launch-skip 4 --launch-count 1 -o gpurun_out/r02_ncu_k_reduce_c2 -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_reduce --launch-skip 4 --launch-count 1 -o gpurun_out/r02_ncu_k_reduce_c5 -f python bench.py --config c5 --params 268435456 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_ring_loop --launch-skip 2 --launch-count 1 -o gpurun_out/r02_ncu_k_ring_loop_g2 -f python tools/loopback_bench.py 2 8 134217728 3 > gpurun_out/ncu_loop.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_ring_loop --launch-skip 2 --launch-count 1 -o gpurun_out/r02_ncu_k_ring_loop_g4_adv -f python tools/loopback_bench.py 4 4 134217728 3 3 > gpurun_out/ncu_loop4.log 2>&1
python tools/loopback_bench.py 2 8 134217728 5 > gpurun_out/loopback_final.log 2>&1
python tools/loopback_bench.py 4 4 134217728 5 3 >> gpurun_out/loopback_final.log 2>&1
