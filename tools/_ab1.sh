mkdir -p gpurun_out
rm -f gpurun_out/e2e_variants.log
for v in . ab_b1r4 ab_b1r6 ab_b2r4 ab_b384r6 .; do
  (cd $v && timeout 900 python tools/e2e_probe.py 1000000000 0 2>&1 | sed "s|^|$v |" >> $GRAFT_REPO_ROOT/gpurun_out/e2e_variants.log)
done
