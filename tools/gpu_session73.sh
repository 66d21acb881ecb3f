# smem kernel lanes per column A/B on tiny (4 / 8 / 16)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for l in 4 8 16; do
  echo "== lanes=$l"
  PCDM_SMEM_LANES=$l timeout 900 python bench.py --config tiny --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], d['ms_per_step'], d['breakdown_ms_per_step'], d['grid'])"
done
