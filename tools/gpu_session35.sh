# dirty list restarted at each refresh: full GPU suite + skewed benches
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
rm -f gpurun_out/hotres.jsonl
for tau in 65536 4096 256; do
  timeout 900 python bench.py --config skewed --tau $tau --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/hotres.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/hotres.jsonl'):
    d=json.loads(l); print(d['config']['workload'], d['config']['tau'], '%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'])
PY
