# full-size huge parity test (bench launch configuration)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/pytest_full.log 2>&1; echo "full rc=$?"
tail -30 gpurun_out/pytest_full.log
