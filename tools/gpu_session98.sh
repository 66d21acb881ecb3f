# overlapped presampler on every config (PCDM_PRESAMPLE_DEV=1) + full ncu of the batched passes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/configs_pd.jsonl
for cfg in tiny medium large; do
  PCDM_PRESAMPLE_DEV=1 timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/configs_pd.jsonl
done
for tau in 256 4096 65536; do
  PCDM_PRESAMPLE_DEV=1 timeout 900 python bench.py --config skewed --tau $tau --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/configs_pd.jsonl
done
PCDM_PRESAMPLE_DEV=1 timeout 1200 python bench.py --loss logistic --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/configs_pd.jsonl
CMD="python bench.py --steps 1 --warmup 1 --iters 36 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"batch_expand|batch_sweep|pcdm_batched_slot|batch_fold" -s 4 -c 4 -o gpurun_out/bat98_full $CMD > gpurun_out/ncu98_full.log 2>&1; echo "ncu rc=$?"
