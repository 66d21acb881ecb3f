set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_theory_vs_reality.py -m gpu -x -q > gpurun_out/pytest_tvr.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_tvr.log
timeout 2400 python tools/theory_vs_reality.py --out gpurun_out/theory_vs_reality.jsonl > gpurun_out/tvr.log 2>&1; echo "tvr rc=$?"
tail -5 gpurun_out/tvr.log
