mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "test_gpu_ragged or many_chunks or long_columns" > gpurun_out/r02_pytest_ragged.txt 2>&1
tail -3 gpurun_out/r02_pytest_ragged.txt
O=gpurun_out/r02_ragged_ab2.jsonl
: > $O
python bench.py --config ragged --steps 5 --no-e2e --no-parity --no-cpu-baseline > gpurun_out/rb1.json 2> gpurun_out/rb1.err; tail -1 gpurun_out/rb1.json >> $O
PCDM_PRESAMPLE_DEV=0 python bench.py --config ragged --steps 5 --no-e2e --no-parity --no-cpu-baseline > gpurun_out/rb1b.json 2> gpurun_out/rb1b.err; tail -1 gpurun_out/rb1b.json >> $O
PCDM_LAYOUT=ragged python bench.py --config large --steps 5 --no-e2e --no-parity --no-cpu-baseline > gpurun_out/rb4.json 2>gpurun_out/rb4.err; tail -1 gpurun_out/rb4.json >> $O
for f in gpurun_out/rb*.err; do tail -n 2 $f; done
