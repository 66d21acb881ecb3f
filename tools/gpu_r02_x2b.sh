mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "test_gpu_ragged or hot_rows or logistic" > gpurun_out/r02_pytest_x2b.txt 2>&1
tail -3 gpurun_out/r02_pytest_x2b.txt
O=gpurun_out/r02_bulk_stage_ab.jsonl
: > $O
for bs in 0 1 0 1; do
PCDM_BULK_STAGE=$bs python bench.py --config ragged --steps 5 --no-e2e --no-parity --no-cpu-baseline > gpurun_out/bs.json 2> gpurun_out/bs.err; tail -n 1 gpurun_out/bs.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['PCDM_BULK_STAGE']=$bs; print(json.dumps(d))" >> $O
done
tail -n 2 gpurun_out/bs.err
