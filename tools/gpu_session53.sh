# barrier spin with __nanosleep (32 / 128 ns) vs plain spin: medium, skewed 256, huge
set -x
mkdir -p gpurun_out
rm -f gpurun_out/sleep.jsonl
for sl in 0 32 128; do
  if [ $sl = 0 ]; then EXTRA=""; else EXTRA="-DPCDM_BARRIER_SLEEP=$sl"; fi
  PCDM_NVCC_EXTRA="$EXTRA" python -m paper_1212_0873_b200.build > gpurun_out/build_$sl.log 2>&1
  for cfg in "medium 1024" "skewed 256" "huge 262144"; do
    set -- $cfg
    echo "== sleep=$sl $1" >> gpurun_out/sleep.jsonl
    timeout 900 python bench.py --config $1 --tau $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/sleep.jsonl
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/sleep.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print('%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'])
PY
