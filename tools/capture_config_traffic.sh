#!/bin/bash
# Per-config roofline evidence: DRAM and L2 bytes of every iteration-kernel launch of one
# bench step (ncu metrics pass; the same command first exits 0 without ncu), written to
# gpurun_out/cfg_<name>.csv.  Afterwards, here:
#   python tools/ncu_traffic.py gpurun_out/cfg_<name>.csv <config>[@tau]:<loop>:nice 0 \
#       --kernels '<regex>' --total-iters <iterations of the captured runs>
# usage: tools/capture_config_traffic.sh "<config> <tau> <kernel regex>" ...
mkdir -p gpurun_out
for spec in "$@"; do
  set -- $spec
  cfg=$1; tau=$2; rx=$3
  CMD="python bench.py --config $cfg --tau $tau --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-parity"
  $CMD > gpurun_out/cfg_${cfg}_${tau}_plain.log 2>&1 &&
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum \
      --clock-control none -k regex:$rx --csv --log-file gpurun_out/cfg_${cfg}_${tau}.csv $CMD \
      > gpurun_out/cfg_${cfg}_${tau}_ncu.log 2>&1
  echo "$cfg $tau rc=$? launches=$(grep -c gpu__time_duration gpurun_out/cfg_${cfg}_${tau}.csv)"
done
