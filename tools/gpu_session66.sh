# skewed tau=65536: warm launch list of the refresh kernels (steady-state x after a long warm-up)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --config skewed --tau 65536 --steps 1 --warmup 3 --iters 3100 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_skw.csv $CMD > gpurun_out/ncu_skw.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py launches gpurun_out/launches_skw.csv --only-lib
