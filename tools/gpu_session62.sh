# ncu --set full of the packed kernel on large (tau = 65536)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --config large --steps 1 --warmup 1 --iters 128 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --set full --clock-control none --cache-control none --import-source on -k regex:pcdm_packed -s 2 -c 1 -o gpurun_out/prof_large $CMD > gpurun_out/ncu_large.log 2>&1; echo "ncu rc=$?"
