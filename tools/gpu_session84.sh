# AUTO -> batched on huge: tests, bench, ncu launch list + full capture of one chunk's passes
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_batched.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -4
timeout 900 python bench.py --steps 3 --warmup 3 2>&1 | grep '^{' > gpurun_out/bench84.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/bench84.jsonl').read()); print('bench', d['variant'], '%.4g'%d['value'], d['e2e']['value'], d['ms_per_step'], d['breakdown_ms_per_step'], d['roofline'])"
CMD="python bench.py --steps 1 --warmup 1 --iters 36 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"batch_expand|batch_sweep|pcdm_batched_slot|batch_fold" -s 4 -c 4 -o gpurun_out/bat84_full $CMD > gpurun_out/ncu84_full.log 2>&1; echo "ncu rc=$?"
