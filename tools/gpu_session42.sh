# warm-cache launch list of one short huge run (where the sampler time goes now)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --iters 45 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain_short.log 2>&1; echo "plain rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_warm.csv $CMD > gpurun_out/ncu_warm.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py launches gpurun_out/launches_warm.csv --only-lib
