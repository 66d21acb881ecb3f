set -x
mkdir -p gpurun_out
python bench.py --config medium --steps 5 > gpurun_out/r02_medium_parity.json 2> gpurun_out/r02_medium_parity.err
python bench.py > gpurun_out/r02_bench1.json 2> gpurun_out/r02_bench1.err
timeout 1500 python -m pytest tests -m gpu -x -q -s -k "fullrun or fullsize" > gpurun_out/r02_pytest_fullrun.txt 2>&1
tail -5 gpurun_out/r02_pytest_fullrun.txt
