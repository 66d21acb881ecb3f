# hot-row shared-memory cache: GPU tests + skewed A/B (PCDM_HOT_ROWS=0 vs default)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_hot_rows.py -x -q > gpurun_out/pytest_hot.log 2>&1; echo "hot rc=$?"
tail -3 gpurun_out/pytest_hot.log
rm -f gpurun_out/hot_ab.jsonl
for tau in 256 4096 65536; do
  for hot in 0 1; do
    echo "== tau=$tau PCDM_HOT_ROWS=$hot" >> gpurun_out/hot_ab.jsonl
    PCDM_HOT_ROWS=$hot timeout 900 python bench.py --config skewed --tau $tau --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/hot_ab.jsonl
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/hot_ab.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print(d['value'], d['ms_per_step'], d['breakdown_ms_per_step'])
PY
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
