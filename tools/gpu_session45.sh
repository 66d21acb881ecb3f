# sampler rounds kernel with CAS-first inserts and recorded entries: sampler tests + benches
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sampler or sampling" > gpurun_out/pytest_samp.log 2>&1; echo "samp rc=$?"
tail -2 gpurun_out/pytest_samp.log
rm -f gpurun_out/rounds.jsonl
for cfg in "huge 262144" "large 65536" "skewed 65536"; do
  set -- $cfg
  timeout 900 python bench.py --config $1 --tau $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/rounds.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/rounds.jsonl'):
    d=json.loads(l); print(d['config']['workload'], '%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'])
PY
