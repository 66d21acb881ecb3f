# sampler pass size (PCDM_SAMPLER_MB) A/B on huge + the full skewed tau sweep 2^8..2^16
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/smb.jsonl gpurun_out/sweep.jsonl
for mb in 32 64 128; do
  echo "== PCDM_SAMPLER_MB=$mb" >> gpurun_out/smb.jsonl
  PCDM_SAMPLER_MB=$mb timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' >> gpurun_out/smb.jsonl
done
for e in 8 9 10 11 12 13 14 15 16; do
  tau=$((1 << e))
  timeout 900 python bench.py --config skewed --tau $tau --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' >> gpurun_out/sweep.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/smb.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print('%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'])
for l in open('gpurun_out/sweep.jsonl'):
    d=json.loads(l); print('skewed', d['config']['tau'], '%.4g'%d['value'], round(d['ms_per_step'],2), d['beta'], d['breakdown_ms_per_step'], d['grid'])
PY
