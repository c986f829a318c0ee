mkdir -p gpurun_out
for i in 1 2; do
  for v in ab_v1 ab_v2 ab_v3 .; do
    (cd $v && timeout 600 python bench.py --config c5 --no-e2e --no-cpu --steps 10 > $GRAFT_REPO_ROOT/gpurun_out/ab1_$(basename $v)_c5_$i.json 2>&1)
  done
done
