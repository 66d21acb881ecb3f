# dense-step bookkeeping (no dirty x list, CTA-staged step lists): tests + logistic bench + huge bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "staged or host or packed" > gpurun_out/pytest_dense.log 2>&1; echo "dense rc=$?"
tail -3 gpurun_out/pytest_dense.log
timeout 900 python -m pytest tests -x -q -m gpu -k "logistic" > gpurun_out/pytest_log.log 2>&1; echo "logistic rc=$?"
tail -2 gpurun_out/pytest_log.log
rm -f gpurun_out/dense.jsonl
timeout 1200 python bench.py --loss logistic --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/dense.jsonl
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/dense.jsonl
python - <<'PY'
import json
for l in open('gpurun_out/dense.jsonl'):
    d=json.loads(l); print(d['config']['workload'], '%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'], d.get('F_final'))
PY
