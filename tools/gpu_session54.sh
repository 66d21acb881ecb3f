# cluster barrier for grids of <= 16 CTAs: tests on small-tau paths + A/B
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
PCDM_CTAS=16 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hot_rows.py -x -q -k "packed or medium or hot or staged" > gpurun_out/pytest_cl16.log 2>&1; echo "cl16 rc=$?"
tail -2 gpurun_out/pytest_cl16.log
rm -f gpurun_out/clsync.jsonl
for v in "medium 1024 0 0" "medium 1024 16 1" "medium 1024 16 0" "skewed 256 0 1" "skewed 256 0 0"; do
  set -- $v
  echo "== $1 tau=$2 PCDM_CTAS=$3 PCDM_CLUSTER_SYNC=$4" >> gpurun_out/clsync.jsonl
  PCDM_CTAS=$3 PCDM_CLUSTER_SYNC=$4 timeout 900 python bench.py --config $1 --tau $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/clsync.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/clsync.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print('%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'], d['grid'])
PY
