# ncu: fused-sampler packed kernel vs standalone sampler kernels (huge, short run)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --iters 20 --no-cpu-baseline --no-e2e"
PCDM_FUSED_SAMPLER=1 timeout 600 $CMD > gpurun_out/plain_fused.log 2>&1 && \
PCDM_FUSED_SAMPLER=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcdm_packed -s 3 -c 1 -o gpurun_out/prof_fused $CMD > gpurun_out/ncu_fused.log 2>&1; echo "ncu fused rc=$?"
PCDM_FUSED_SAMPLER=0 timeout 600 $CMD > gpurun_out/plain_nofused.log 2>&1 && \
PCDM_FUSED_SAMPLER=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sample_|pcdm_packed" -s 12 -c 4 -o gpurun_out/prof_sampler $CMD > gpurun_out/ncu_sampler.log 2>&1; echo "ncu sampler rc=$?"
