# BATCHED: parity tests + per-pass launch list (ncu, cold/serialised) on huge
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_batched.py -x -q > gpurun_out/pytest_batched.log 2>&1; echo "batched rc=$?"
tail -30 gpurun_out/pytest_batched.log
CMD="python bench.py --variant batched --steps 1 --warmup 3 --iters 45 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain_short.log 2>&1; echo "plain rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_batched.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_summary.py launches gpurun_out/launches_batched.csv --only-lib 2>&1 | head -30
