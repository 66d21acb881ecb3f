# expand CTA size x sweep lanes-per-segment
mkdir -p gpurun_out
rm -f gpurun_out/ab107.txt
for cfg in "-DPCDM_EXPAND_THREADS=128 -DPCDM_SWEEP_HW=4" "-DPCDM_EXPAND_THREADS=128 -DPCDM_SWEEP_HW=8" "-DPCDM_EXPAND_THREADS=256 -DPCDM_SWEEP_HW=8"; do
PCDM_NVCC_EXTRA="$cfg" python -c "from paper_1212_0873_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' > gpurun_out/b.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/b.jsonl').read()); print('$cfg', d['variant'], '%.4g'%d['value'], round(d['ms_per_step'],3), d['breakdown_ms_per_step'])" | tee -a gpurun_out/ab107.txt
done
