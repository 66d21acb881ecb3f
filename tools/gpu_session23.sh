# sampler ILP round0 (CAS-first, recorded entry) + one-load check: tests and benches
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
rm -f gpurun_out/samp.jsonl
for cfg in "huge 262144" "skewed 65536" "large 65536"; do
  set -- $cfg
  timeout 900 python bench.py --config $1 --tau $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/samp.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/samp.jsonl'):
    d=json.loads(l); print(d['config']['workload'], d['config']['tau'], d['value'], d['ms_per_step'], d['breakdown_ms_per_step'])
PY
