# compact host-x copy-back: tests + default bench (e2e)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "host" > gpurun_out/pytest_host.log 2>&1; echo "host rc=$?"
tail -15 gpurun_out/pytest_host.log
timeout 900 python bench.py > gpurun_out/bench_e2e.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_e2e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e'])"
