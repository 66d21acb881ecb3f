# sampler hash-table load factor A/B (PCDM_TABLE_X = 2, 4, 8)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PCDM_TABLE_X=4 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sampler or sampling" > gpurun_out/pytest_samp.log 2>&1; echo "samp rc=$?"
tail -2 gpurun_out/pytest_samp.log
rm -f gpurun_out/tx.jsonl
for cfg in "huge 262144" "large 65536" "skewed 65536"; do
  set -- $cfg
  for x in 2 4 8; do
    echo "== $1 PCDM_TABLE_X=$x" >> gpurun_out/tx.jsonl
    PCDM_TABLE_X=$x timeout 900 python bench.py --config $1 --tau $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/tx.jsonl
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/tx.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print('%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'])
PY
