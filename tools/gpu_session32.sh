# e2e A/B: presampling during the host-x copy on/off (bench with an untimed e2e warm-up step)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for ps in 0 1; do
  PCDM_PRESAMPLE=$ps timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ps$ps.log 2>&1; echo "bench rc=$?"
  echo "PCDM_PRESAMPLE=$ps"; tail -1 gpurun_out/bench_ps$ps.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e'])"
done
