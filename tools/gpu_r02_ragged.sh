mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "test_gpu_ragged or many_chunks" > gpurun_out/r02_pytest_ragged.txt 2>&1
tail -30 gpurun_out/r02_pytest_ragged.txt
