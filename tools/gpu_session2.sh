# microbenchmarks + bench + ncu evidence for the current hot path (huge config)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 ./tools/gather_order > gpurun_out/gather_order.jsonl 2>&1; echo "gather_order rc=$?"
timeout 300 ./tools/microbench > gpurun_out/microbench.jsonl 2>&1; echo "microbench rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --iters 50 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain_short.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_short.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pcdm_packed -s 4 -c 2 -o gpurun_out/prof_packed_huge $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
