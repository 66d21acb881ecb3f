# BATCHED: pass-3 prefetch depth and expand occupancy A/B (compile-time knobs)
set -x
mkdir -p gpurun_out
for cfg in "-DPCDM_BATCHED_UP=2 -DPCDM_EXPAND_MINB=3" "-DPCDM_BATCHED_UP=1 -DPCDM_EXPAND_MINB=3" "-DPCDM_BATCHED_UP=2 -DPCDM_EXPAND_MINB=2"; do
PCDM_NVCC_EXTRA="$cfg" python -c "from paper_1212_0873_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --variant batched --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' > gpurun_out/b.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/b.jsonl').read()); print('$cfg', '%.4g'%d['value'], d['ms_per_step'], d['breakdown_ms_per_step'])" | tee -a gpurun_out/ab77.txt
done
