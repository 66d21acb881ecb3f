# steps pass: second slot staged by cp.async, CTA size A/B
mkdir -p gpurun_out
rm -f gpurun_out/ab87.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_batched.py -x -q 2>&1 | tail -2
for cfg in "-DPCDM_STEP_STAGE2=1 -DPCDM_STEP_THREADS=512" "-DPCDM_STEP_STAGE2=1 -DPCDM_STEP_THREADS=1024" "-DPCDM_STEP_STAGE2=0 -DPCDM_STEP_THREADS=1024"; do
PCDM_NVCC_EXTRA="$cfg" python -c "from paper_1212_0873_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' > gpurun_out/b.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/b.jsonl').read()); print('$cfg', d['variant'], '%.4g'%d['value'], d['ms_per_step'], d['breakdown_ms_per_step'])" | tee -a gpurun_out/ab87.txt
done
