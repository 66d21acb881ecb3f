# logistic regression check: session-start tree (e5491cb) vs current, kddb_like bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
(cd old_tree && python -c "import __graft_entry__ as g; g.build()" > ../gpurun_out/build_old.log 2>&1)
rm -f gpurun_out/logreg.jsonl
echo "== old e5491cb" >> gpurun_out/logreg.jsonl
(cd old_tree && timeout 1200 python bench.py --loss logistic --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> ../gpurun_out/logreg.jsonl)
echo "== current PCDM_ITER_CHUNK=1 PCDM_ROW_RESIDUAL=0" >> gpurun_out/logreg.jsonl
PCDM_ITER_CHUNK=1 PCDM_ROW_RESIDUAL=0 timeout 1200 python bench.py --loss logistic --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/logreg.jsonl
python - <<'PY'
import json
for l in open('gpurun_out/logreg.jsonl'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print('%.4g'%d['value'], round(d['ms_per_step'],2), d['breakdown_ms_per_step'], d.get('F_final'), d.get('grid'))
PY
