# session 3 baseline check + batched-snapshot prototype
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 ./tools/batch_proto 50000000 8 > gpurun_out/batch_proto_b8.jsonl 2>&1; echo "proto rc=$?"
timeout 300 ./tools/batch_proto 50000000 16 > gpurun_out/batch_proto_b16.jsonl 2>&1; echo "proto16 rc=$?"
cat gpurun_out/batch_proto_b8.jsonl
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_s3.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_s3.log | cut -c1-400
