# BATCHED variant: parity tests, huge bench A/B (packed vs batched)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_batched.py -x -q > gpurun_out/pytest_batched.log 2>&1; echo "batched rc=$?"
tail -30 gpurun_out/pytest_batched.log
rm -f gpurun_out/bat.jsonl
for v in packed batched; do
  timeout 900 python bench.py --variant $v --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/bat.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/bat.jsonl'):
    d=json.loads(l); print(d['variant'], d['value'], d['ms_per_step'], d['breakdown_ms_per_step'], d['F_final'])
PY
