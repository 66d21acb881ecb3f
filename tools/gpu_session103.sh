# snapshot length A/B with the presampled slots (no sampler-window coupling)
mkdir -p gpurun_out
rm -f gpurun_out/ab103.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in 12 18 24 30 36; do
PCDM_BATCHED_CHUNK=$c timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' > gpurun_out/b.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/b.jsonl').read()); print('chunk=$c', d['variant'], '%.4g'%d['value'], round(d['ms_per_step'],3), d['breakdown_ms_per_step'])" | tee -a gpurun_out/ab103.txt
done
