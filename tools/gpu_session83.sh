# BATCHED vs packed across configs (decides the AUTO rule)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/ab83.txt
run() { # label args...
  lab=$1; shift
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" 2>&1 | grep '^{' > gpurun_out/b.jsonl
  python -c "
import json
d=json.loads(open('gpurun_out/b.jsonl').read()); e=d.get('e2e') or {}
print('$lab', '%.4g'%d['value'], 'e2e=%s'%('%.4g'%e['value'] if e else None), d['ms_per_step'], d['breakdown_ms_per_step'])" | tee -a gpurun_out/ab83.txt
}
for v in packed batched; do
  run "large $v" --config large --variant $v --no-e2e
  run "skewed65536 $v" --config skewed --tau 65536 --variant $v --no-e2e
  run "kddb $v" --config kddb_like --loss logistic --variant $v --no-e2e
  run "huge-indep $v" --sampling independent --variant $v --no-e2e
  run "huge-e2e $v" --variant $v
done
