# row-major residual for logistic problems: logistic tests + kddb_like bench A/B; ncu full capture of the packed kernel (huge)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_logistic.py tests/test_gpu_hot_rows.py tests/test_gpu_batched.py tests/test_gpu_cluster.py -x -q -k "logistic" > gpurun_out/pytest_log.log 2>&1; echo "logistic rc=$?"
tail -3 gpurun_out/pytest_log.log
rm -f gpurun_out/rowres.jsonl
for rr in 0 1; do
  echo "== PCDM_ROW_RESIDUAL=$rr" >> gpurun_out/rowres.jsonl
  PCDM_ROW_RESIDUAL=$rr timeout 1200 python bench.py --loss logistic --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/rowres.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/rowres.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print('%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'], d.get('F_final'))
PY
CMD="python bench.py --steps 1 --warmup 3 --iters 50 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:pcdm_packed -s 2 -c 1 -o gpurun_out/prof_packed_s3b $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -2 gpurun_out/ncu_full.log
