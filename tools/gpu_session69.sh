# packed kernel at 3 vs 4 CTAs per SM (launch bounds), huge / large / medium
set -x
mkdir -p gpurun_out
rm -f gpurun_out/minb.jsonl
for mb in 3 4; do
  PCDM_NVCC_EXTRA="-DPCDM_PACKED_MINB=$mb" python -m paper_1212_0873_b200.build > gpurun_out/build_$mb.log 2>&1
  for cfg in "huge 262144" "large 65536" "skewed 65536"; do
    set -- $cfg
    echo "== minb=$mb $1" >> gpurun_out/minb.jsonl
    timeout 900 python bench.py --config $1 --tau $2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' >> gpurun_out/minb.jsonl
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/minb.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print('%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'], d['grid'])
PY
