# sampler pass size (PCDM_SAMPLER_MB) 128 / 192 / 256 on huge, large, skewed 65536
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/smb2.jsonl
for cfg in "huge 262144" "large 65536" "skewed 65536"; do
  set -- $cfg
  for mb in 64 128 256; do
    echo "== $1 PCDM_SAMPLER_MB=$mb" >> gpurun_out/smb2.jsonl
    PCDM_SAMPLER_MB=$mb timeout 900 python bench.py --config $1 --tau $2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' >> gpurun_out/smb2.jsonl
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/smb2.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print('%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'])
PY
