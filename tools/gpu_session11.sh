set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PCDM_OVERLAP=1 timeout 1200 python -m pytest tests -m gpu -x -q -k "many_chunks or packed or sampling_runs or tiny" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
rm -f gpurun_out/ab.log
for cfg in "PCDM_OVERLAP=0" "PCDM_OVERLAP=1 PCDM_CTAS_PER_SM=2" "PCDM_OVERLAP=1 PCDM_CTAS_PER_SM=3" "PCDM_OVERLAP=1 PCDM_CTAS_PER_SM=2 PCDM_SAMPLER_BLOCKS_PER_SM=2" "PCDM_OVERLAP=1 PCDM_CTAS_PER_SM=2 PCDM_SAMPLER_MB=32"; do
  echo "== $cfg" >> gpurun_out/ab.log
  env $cfg timeout 600 $B 2>&1 | grep '^{' | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({k:d[k] for k in ['value','ms_per_step','breakdown_ms_per_step','F_final']}), json.dumps(d['roofline']['launch_ms']), d['roofline']['iters_per_launch'])" >> gpurun_out/ab.log 2>&1
done
cat gpurun_out/ab.log
