# sampler check pass: recorded entry index vs probe (A/B) + sampler tests
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PCDM_CHECK_AT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sampler or sampling" > gpurun_out/pytest_samp.log 2>&1; echo "samp rc=$?"
tail -2 gpurun_out/pytest_samp.log
rm -f gpurun_out/checkat.jsonl
for cfg in "huge 262144" "large 65536" "skewed 65536"; do
  set -- $cfg
  for f in 0 1; do
    echo "== $1 PCDM_CHECK_AT=$f" >> gpurun_out/checkat.jsonl
    PCDM_CHECK_AT=$f timeout 900 python bench.py --config $1 --tau $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/checkat.jsonl
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/checkat.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print('%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'])
PY
