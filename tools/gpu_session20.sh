# grid sized to the CTAs that own slots (small tau) + hot-row cache rule: tests and A/B
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_hot_rows.py -x -q > gpurun_out/pytest_hot.log 2>&1; echo "hot rc=$?"
tail -3 gpurun_out/pytest_hot.log
rm -f gpurun_out/ctas_ab.jsonl
for cfg in "medium 1024" "skewed 256" "skewed 4096" "skewed 65536"; do
  set -- $cfg
  for ctas in 100000 0; do
    echo "== $1 tau=$2 PCDM_CTAS=$ctas" >> gpurun_out/ctas_ab.jsonl
    PCDM_CTAS=$ctas timeout 900 python bench.py --config $1 --tau $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/ctas_ab.jsonl
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/ctas_ab.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print(d['value'], d['ms_per_step'], d['breakdown_ms_per_step'], d.get('grid'))
PY
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
