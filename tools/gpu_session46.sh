# ncu --set full of the packed kernel on skewed tau=65536 (steady state: one 10^4-iteration warm-up run first)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --config skewed --tau 65536 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --set full --clock-control none --cache-control none --import-source on -k regex:pcdm_packed -s 330 -c 1 -o gpurun_out/prof_skewed $CMD > gpurun_out/ncu_skewed_full.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_skewed_full.log
