# bench every config at its default tau (and skewed over its tau sweep) -> gpurun_out/configs.jsonl
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/configs.jsonl
for cfg in tiny medium large huge; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e 2>&1 | grep '^{' >> gpurun_out/configs.jsonl
done
for tau in 256 4096 65536; do
  timeout 900 python bench.py --config skewed --tau $tau --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/configs.jsonl
done
