# BATCHED: ncu --set full of one launch of each pass on huge
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --variant batched --steps 1 --warmup 3 --iters 27 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"pcdm_batched" -s 2 -c 1 -o gpurun_out/prof_batched $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -2 gpurun_out/ncu_full.log
