set -x
mkdir -p gpurun_out
timeout 120 ./tools/l2_policy > gpurun_out/l2_policy.jsonl 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__sectors_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --csv --log-file gpurun_out/l2_policy_ncu.csv ./tools/l2_policy > gpurun_out/l2_policy_ncu.log 2>&1; echo rc=$?
