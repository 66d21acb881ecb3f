# presampler passes overlapping the iteration kernels (PCDM_PRESAMPLE_DEV=1): tests + A/B
mkdir -p gpurun_out
rm -f gpurun_out/ab96.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PCDM_PRESAMPLE_DEV=1 timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for cfg in huge large; do
for pd in 0 1; do
PCDM_PRESAMPLE_DEV=$pd timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/b.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/b.jsonl').read()); print('$cfg presample_dev=$pd', d['variant'], '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], round(d['ms_per_step'],3), d['breakdown_ms_per_step'])" | tee -a gpurun_out/ab96.txt
done
done
