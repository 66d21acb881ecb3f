# sampler rounds kernel with 1024 threads per iteration: sampler tests + skewed/large/huge benches
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sampler or sampling" > gpurun_out/pytest_samp.log 2>&1; echo "samp rc=$?"
tail -2 gpurun_out/pytest_samp.log
rm -f gpurun_out/samp2.jsonl
for cfg in "skewed 65536" "skewed 4096" "large 65536" "huge 262144"; do
  set -- $cfg
  timeout 900 python bench.py --config $1 --tau $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/samp2.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/samp2.jsonl'):
    d=json.loads(l); print(d['config']['workload'], d['config']['tau'], '%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'])
PY
