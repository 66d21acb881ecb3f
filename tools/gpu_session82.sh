# sweep lanes-per-segment A/B, then chunk A/B at the best
set -x
mkdir -p gpurun_out
for hw in 8 32; do
PCDM_NVCC_EXTRA="-DPCDM_SWEEP_HW=$hw" python -c "from paper_1212_0873_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --variant batched --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' > gpurun_out/b.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/b.jsonl').read()); print('hw=$hw', '%.4g'%d['value'], d['ms_per_step'], d['breakdown_ms_per_step'])" | tee -a gpurun_out/ab82.txt
done
python -c "from paper_1212_0873_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
for c in 12 27 36; do
PCDM_BATCHED_CHUNK=$c timeout 900 python bench.py --variant batched --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' > gpurun_out/b.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/b.jsonl').read()); print('chunk=$c', '%.4g'%d['value'], d['ms_per_step'], d['breakdown_ms_per_step'])" | tee -a gpurun_out/ab82.txt
done
