# release/acquire grid barrier: full GPU suite + configs
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
rm -f gpurun_out/bar.jsonl
for cfg in "medium 1024" "skewed 256" "skewed 65536" "large 65536" "huge 262144"; do
  set -- $cfg
  timeout 900 python bench.py --config $1 --tau $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/bar.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/bar.jsonl'):
    d=json.loads(l); print(d['config']['workload'], d['config']['tau'], '%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'])
PY
