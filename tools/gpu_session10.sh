set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
rm -f gpurun_out/samplings.jsonl
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/bench_default.log >> gpurun_out/samplings.jsonl
for smp in "--sampling independent" "--sampling binomial --p-b 0.5"; do
  timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e $smp 2>&1 | grep '^{' >> gpurun_out/samplings.jsonl
done
