# k_stats variants (build/ab/<V>: launch bound x element-loop unroll) at full size,
# 2-rank loopback of 16 miners x 1e9 with 6 noise-deceptive: ncu duration of k_stats
mkdir -p gpurun_out; rm -f gpurun_out/ab_kstats.log
for v in V1 V2 V3 V4 V5 V1; do
  (cd build/ab/$v && timeout 400 ncu --kernel-name regex:"k_stats" --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv python tools/finish_probe.py 2 16 1e9 6 1 2>/dev/null | grep '"k_stats' | awk -F'","' -v v=$v '{print v, $(NF-2), $NF}') >> gpurun_out/ab_kstats.log
done
