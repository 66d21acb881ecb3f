mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "hot_rows" > gpurun_out/r02_pytest_hot.txt 2>&1
tail -3 gpurun_out/r02_pytest_hot.txt
python tools/scatter_ab.py > gpurun_out/r02_hot_stage_ab.jsonl 2> gpurun_out/r02_hot_stage_ab.err
tail -3 gpurun_out/r02_hot_stage_ab.err
