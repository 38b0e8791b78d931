mkdir -p gpurun_out
for v in -1 60 50 40; do echo "CARVE=$v"
for cfg in "100000 1.0 0.01 21" "100000 16.0 0.001 11"; do W1G_WSPD_DFS_CARVEOUT=$v timeout 120 python tools/fe_once.py $cfg | head -1; done
W1G_WSPD_DFS_CARVEOUT=$v ncu --metrics gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:k_wspd_dfs --log-file gpurun_out/dfs_c.csv python tools/fe_once.py 100000 16.0 0.001 > /dev/null 2>&1
grep k_wspd_dfs gpurun_out/dfs_c.csv | awk -F'","' '{print $(NF-2), $NF}' | tail -3
done > gpurun_out/bm.log 2>&1
