# full ncu capture of the restructured steps kernel (source-level stalls)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --iters 36 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"pcdm_batched_slot" -s 1 -c 1 -o gpurun_out/steps86 $CMD > gpurun_out/ncu86.log 2>&1; echo "ncu rc=$?"
