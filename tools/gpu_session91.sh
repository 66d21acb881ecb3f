# AUTO rule: batched vs packed crossover in active slots per iteration on huge
mkdir -p gpurun_out
rm -f gpurun_out/ab91.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() {
  lab=$1; shift
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>&1 | grep '^{' > gpurun_out/b.jsonl
  python -c "
import json
d=json.loads(open('gpurun_out/b.jsonl').read())
print('$lab', d['variant'], '%.4g'%d['value'], d['ms_per_step'], d['breakdown_ms_per_step'])" | tee -a gpurun_out/ab91.txt
}
for tau in 131072 196608 524288; do
  run "nice tau=$tau batched" --tau $tau --variant batched
  run "nice tau=$tau packed" --tau $tau --variant packed
done
run "binomial 0.5 AUTO" --sampling binomial --p-b 0.5
run "binomial 0.75 batched" --sampling binomial --p-b 0.75 --variant batched
run "binomial 0.75 packed" --sampling binomial --p-b 0.75 --variant packed
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
