# in-kernel residual refresh of the shared-memory variant: tests + tiny bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4
timeout 900 python bench.py --config tiny --steps 3 --warmup 3 --no-e2e 2>&1 | grep '^{' > gpurun_out/tiny.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/tiny.jsonl').read()); print('%.4g'%d['value'], d['ms_per_step'], d['breakdown_ms_per_step'], d['cpu_baseline'])"
