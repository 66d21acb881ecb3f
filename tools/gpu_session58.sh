# NEXT rows re-measured on the current build: samplings and async on huge, logistic, default bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/next.jsonl
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --sampling independent 2>&1 | grep '^{' >> gpurun_out/next.jsonl
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --sampling binomial --p-b 0.5 2>&1 | grep '^{' >> gpurun_out/next.jsonl
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --async 2>&1 | grep '^{' >> gpurun_out/next.jsonl
timeout 1200 python bench.py --loss logistic --steps 3 --warmup 3 --no-e2e 2>&1 | grep '^{' >> gpurun_out/next.jsonl
timeout 900 python bench.py --loss logistic --config logistic_small --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/next.jsonl
python - <<'PY'
import json
for l in open('gpurun_out/next.jsonl'):
    d=json.loads(l); c=d['config']; print(c['workload'], c.get('sampling'), d.get('async'), '%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'], d.get('cpu_baseline',{}) and d['cpu_baseline'].get('value'))
PY
