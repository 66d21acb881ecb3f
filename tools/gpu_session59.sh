# tau-independent sampler with CAS-first inserts and recorded entries: tests + huge bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "sampling or independent or sampler" > gpurun_out/pytest_ind.log 2>&1; echo "ind rc=$?"
tail -2 gpurun_out/pytest_ind.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --sampling independent 2>&1 | grep '^{' > gpurun_out/ind.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/ind.jsonl').read()); print('%.4g'%d['value'], d['ms_per_step'], d['breakdown_ms_per_step'])"
