# iteration-kernel launches spanning several sampler chunks: full GPU suite + config benches
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
rm -f gpurun_out/ichunk.jsonl
for cfg in "huge 262144" "large 65536" "medium 1024" "skewed 65536"; do
  set -- $cfg
  for ic in 1 64; do
    echo "== $1 PCDM_ITER_CHUNK=$ic" >> gpurun_out/ichunk.jsonl
    PCDM_ITER_CHUNK=$ic timeout 900 python bench.py --config $1 --tau $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/ichunk.jsonl
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/ichunk.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print('%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'])
PY
