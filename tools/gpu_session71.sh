# round-0 launch shape A/B (threads per block, waves) on huge and large
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/r0.jsonl
for v in "128 8" "128 16" "128 32" "64 16" "64 32"; do
  set -- $v
  for cfg in "huge 262144" "large 65536"; do
    set -- $v $cfg
    echo "== tpb=$1 waves=$2 $3" >> gpurun_out/r0.jsonl
    PCDM_R0_TPB=$1 PCDM_R0_WAVES=$2 timeout 900 python bench.py --config $3 --tau $4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' >> gpurun_out/r0.jsonl
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/r0.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print('%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step']['sampler'])
PY
