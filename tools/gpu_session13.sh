set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_async.py -x -q > gpurun_out/pytest_async.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_async.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --async > gpurun_out/bench_async.log 2>&1; echo "bench rc=$?"
timeout 900 python tools/theory_vs_reality.py --omegas 100 --eps 1e-5 --out gpurun_out/theory_vs_reality_eps1e-5.jsonl > gpurun_out/tvr2.log 2>&1
