set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/logistic.jsonl
timeout 900 python bench.py --loss logistic --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_logistic.log 2>&1; echo "rc=$?"
grep '^{' gpurun_out/bench_logistic.log >> gpurun_out/logistic.jsonl
timeout 900 python bench.py --loss logistic --config logistic_small --steps 3 --warmup 3 --no-e2e 2>&1 | grep '^{' >> gpurun_out/logistic.jsonl
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_default.log 2>&1; echo "rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
