# one-cluster grids of 1024-thread CTAs for small tau: full tests + A/B
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
rm -f gpurun_out/cl1024.jsonl
for v in "medium 1024 1" "medium 1024 0" "skewed 256 1" "skewed 256 0" "skewed 4096 1" "tiny 32 1"; do
  set -- $v
  echo "== $1 tau=$2 PCDM_CLUSTER_SYNC=$3" >> gpurun_out/cl1024.jsonl
  PCDM_CLUSTER_SYNC=$3 timeout 900 python bench.py --config $1 --tau $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/cl1024.jsonl
done
PCDM_CLUSTER_SYNC=1 timeout 900 python bench.py --config tiny --variant packed --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/cl1024.jsonl
python - <<'PY'
import json
for l in open('gpurun_out/cl1024.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print(d['variant'], '%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'], d['grid'])
PY
