# ncu --set full of sample_round0 (huge), warm caches
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --iters 45 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --set full --clock-control none --cache-control none --import-source on -k regex:sample_round0 -s 3 -c 1 -o gpurun_out/prof_round0 $CMD > gpurun_out/ncu_r0.log 2>&1; echo "ncu rc=$?"
