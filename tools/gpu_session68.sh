# round 0 split into a draw kernel and an insert kernel: tests + A/B
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sampler or sampling" > gpurun_out/pytest_samp.log 2>&1; echo "samp rc=$?"
tail -3 gpurun_out/pytest_samp.log
rm -f gpurun_out/split.jsonl
for cfg in "huge 262144" "large 65536" "skewed 65536"; do
  set -- $cfg
  for cm in 0 1; do
    echo "== $1 PCDM_SPLIT_R0=$cm" >> gpurun_out/split.jsonl
    PCDM_SPLIT_R0=$cm timeout 900 python bench.py --config $1 --tau $2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' >> gpurun_out/split.jsonl
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/split.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print('%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'], d['F_final'])
PY
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
