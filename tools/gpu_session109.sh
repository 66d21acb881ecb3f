# sampler pass size with the snapshot held at 18 iterations (presampled, overlapped)
mkdir -p gpurun_out
rm -f gpurun_out/ab109.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for mb in 64 128 256 512; do
PCDM_SAMPLER_MB=$mb PCDM_BATCHED_CHUNK=18 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/b.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/b.jsonl').read()); print('sampler_mb=$mb', d['variant'], '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], round(d['ms_per_step'],3), d['breakdown_ms_per_step'])" | tee -a gpurun_out/ab109.txt
done
