# ncu full capture of the sampler kernels on huge (what bounds round0 / check)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --iters 50 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain_short.log 2>&1; echo "plain rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:sample_ -s 12 -c 4 -o gpurun_out/prof_sampler $CMD > gpurun_out/ncu_sampler.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_sampler.log
