# BATCHED: snapshot length A/B + full ncu capture of the three passes
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in 18 36 72 144; do
PCDM_BATCHED_CHUNK=$c timeout 900 python bench.py --variant batched --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' > gpurun_out/bat_c$c.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/bat_c$c.jsonl').read()); print('chunk=$c', '%.4g'%d['value'], d['ms_per_step'], d['breakdown_ms_per_step'])"
done
CMD="python bench.py --variant batched --steps 1 --warmup 1 --iters 36 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"batch_expand|batch_sweep|pcdm_batched_slot" -s 3 -c 3 -o gpurun_out/bat_full $CMD > gpurun_out/ncu_bat_full.log 2>&1; echo "ncu rc=$?"
