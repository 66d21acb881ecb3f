# launch lists (ncu, cold/serialised) for skewed tau=65536 and large: where the step goes
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in "skewed 65536 62" "large 65536 40"; do
  set -- $cfg
  CMD="python bench.py --config $1 --tau $2 --steps 1 --warmup 3 --iters $3 --no-cpu-baseline --no-e2e"
  timeout 600 $CMD > gpurun_out/plain_$1.log 2>&1; echo "plain rc=$?"
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv $CMD > gpurun_out/ncu_$1.log 2>&1; echo "ncu rc=$?"
  python tools/ncu_summary.py launches gpurun_out/launches_$1.csv --only-lib > gpurun_out/launches_$1_summary.csv 2>&1
  cat gpurun_out/launches_$1_summary.csv
done
