# BATCHED: blocked Bloom filter (3 bits in one word); tests + bench + warm launch list
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' > gpurun_out/b.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/b.jsonl').read()); print('bench', '%.4g'%d['value'], d['ms_per_step'], d['breakdown_ms_per_step'])"
CMD="python bench.py --steps 1 --warmup 2 --iters 54 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_bat.csv $CMD > gpurun_out/ncu_bat.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py launches gpurun_out/launches_bat.csv --only-lib | grep "batch\|pcdm_b\|sample"
