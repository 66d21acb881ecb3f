# skewed tau=65536: one- vs two-barrier scheme (replayed scatters into hot rows)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/ob.jsonl
for ob in 1 0; do
  echo "== PCDM_ONE_BARRIER=$ob" >> gpurun_out/ob.jsonl
  PCDM_ONE_BARRIER=$ob timeout 900 python bench.py --config skewed --tau 65536 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/ob.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/ob.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print('%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'], d['nonzero_step_frac'])
PY
