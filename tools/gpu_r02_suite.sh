mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu.txt 2>&1
tail -5 gpurun_out/r02_pytest_gpu.txt
python bench.py --no-parity --no-cpu-baseline --steps 5 > gpurun_out/r02_bench_create.json 2> gpurun_out/r02_bench_create.err
tail -n 2 gpurun_out/r02_bench_create.err
python -c "import json; d=json.loads(open('gpurun_out/r02_bench_create.json').read().strip().splitlines()[-1]); print(d['setup_s'], d['value'])"
