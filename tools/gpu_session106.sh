# expand CTA size A/B (its slot range scales with it)
mkdir -p gpurun_out
rm -f gpurun_out/ab106.txt
for t in 512 256 128; do
PCDM_NVCC_EXTRA="-DPCDM_EXPAND_THREADS=$t" python -c "from paper_1212_0873_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
[ $t = 256 ] && timeout 900 python -m pytest tests/test_gpu_batched.py -x -q 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' > gpurun_out/b.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/b.jsonl').read()); print('expand_threads=$t', d['variant'], '%.4g'%d['value'], round(d['ms_per_step'],3), d['breakdown_ms_per_step'])" | tee -a gpurun_out/ab106.txt
done
CMD="python bench.py --steps 1 --warmup 2 --iters 54 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_bat.csv $CMD > gpurun_out/ncu_bat.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py launches gpurun_out/launches_bat.csv --only-lib | grep "batch\|pcdm_b"
