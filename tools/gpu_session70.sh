# replay after phase A for sparse-step runs (count loaded before phase A): tests + configs + logistic
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
bash tools/gpu_configs.sh > gpurun_out/configs_run.log 2>&1; echo "configs rc=$?"
timeout 1200 python bench.py --loss logistic --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/configs.jsonl
python - <<'PY'
import json
for l in open('gpurun_out/configs.jsonl'):
    d=json.loads(l); print(d['config']['workload'], d['config']['tau'], '%.4g'%d['value'], round(d['ms_per_step'],2), d['variant'], d['breakdown_ms_per_step'])
PY
