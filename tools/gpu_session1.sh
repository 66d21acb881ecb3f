set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python bench.py --config medium --steps 3 --warmup 3 > gpurun_out/bench_medium.log 2>&1; echo "medium rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_huge.log 2>&1; echo "huge rc=$?"
tail -3 gpurun_out/*.log
