# CLUSTER variant: parity tests + medium A/B (packed vs cluster)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_cluster.py -x -q > gpurun_out/pytest_cluster.log 2>&1; echo "cluster rc=$?"
tail -30 gpurun_out/pytest_cluster.log
rm -f gpurun_out/cl.jsonl
for v in packed cluster; do
  timeout 900 python bench.py --config medium --variant $v --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/cl.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/cl.jsonl'):
    d=json.loads(l); print(d['variant'], d['value'], d['ms_per_step'], d['breakdown_ms_per_step'], d['grid'], d['F_final'])
PY
