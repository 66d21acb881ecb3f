# final evidence (records sized by max len, overlapped presampler): GPU tests, smoke, default bench, reference arm, all configs,
# NEXT rows, ncu launch list + full capture of one snapshot's batched passes
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"
bash tools/gpu_configs.sh > gpurun_out/configs_run.log 2>&1; echo "configs rc=$?"
rm -f gpurun_out/next.jsonl
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --sampling independent 2>&1 | grep '^{' >> gpurun_out/next.jsonl
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --sampling binomial --p-b 0.5 2>&1 | grep '^{' >> gpurun_out/next.jsonl
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --async 2>&1 | grep '^{' >> gpurun_out/next.jsonl
timeout 1200 python bench.py --loss logistic --steps 3 --warmup 3 --no-e2e 2>&1 | grep '^{' >> gpurun_out/next.jsonl
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --variant packed 2>&1 | grep '^{' >> gpurun_out/next.jsonl
CMD="python bench.py --steps 1 --warmup 3 --iters 54 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain_short.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
