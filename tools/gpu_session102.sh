# configs + NEXT rows with the committed defaults (presampler overlapped for every tau-nice run)
mkdir -p gpurun_out
bash tools/gpu_configs.sh > gpurun_out/configs_run.log 2>&1; echo "configs rc=$?"
rm -f gpurun_out/next.jsonl
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --sampling independent 2>&1 | grep '^{' >> gpurun_out/next.jsonl
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --sampling binomial --p-b 0.5 2>&1 | grep '^{' >> gpurun_out/next.jsonl
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --async 2>&1 | grep '^{' >> gpurun_out/next.jsonl
timeout 1200 python bench.py --loss logistic --steps 3 --warmup 3 --no-e2e 2>&1 | grep '^{' >> gpurun_out/next.jsonl
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --variant packed 2>&1 | grep '^{' >> gpurun_out/next.jsonl
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?"
