# expand: slots in flight per group A/B
mkdir -p gpurun_out
rm -f gpurun_out/ab89.txt
for u in 4 6 8; do
PCDM_NVCC_EXTRA="-DPCDM_EXPAND_U=$u" python -c "from paper_1212_0873_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' > gpurun_out/b.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/b.jsonl').read()); print('U=$u', d['variant'], '%.4g'%d['value'], d['ms_per_step'], d['breakdown_ms_per_step'])" | tee -a gpurun_out/ab89.txt
done
