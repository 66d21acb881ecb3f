# split-counter grid barrier A/B (K = 1, 4, 8) on medium, large, huge; tests at the default
mkdir -p gpurun_out
rm -f gpurun_out/ab92.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py -x -q 2>&1 | tail -2
for k in 1 4 8; do
PCDM_NVCC_EXTRA="-DPCDM_BARRIER_SPLIT=$k" python -c "from paper_1212_0873_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
[ $k = 8 ] && timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for cfg in medium large huge; do
timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' > gpurun_out/b.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/b.jsonl').read()); print('K=$k $cfg', d['variant'], '%.4g'%d['value'], round(d['ms_per_step'],3), d['breakdown_ms_per_step'])" | tee -a gpurun_out/ab92.txt
done
done
