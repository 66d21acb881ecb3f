set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
rm -f gpurun_out/ab.log
for cfg in "PCDM_X_IN_BLOCK=0" "PCDM_X_IN_BLOCK=1" "PCDM_X_IN_BLOCK=0" "PCDM_X_IN_BLOCK=1"; do
  echo "== $cfg" >> gpurun_out/ab.log
  env $cfg timeout 600 $B 2>&1 | grep '^{' | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({k:d[k] for k in ['value','ms_per_step','breakdown_ms_per_step','F_final']}))" >> gpurun_out/ab.log 2>&1
done
cat gpurun_out/ab.log
