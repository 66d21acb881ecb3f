# sampler alone: device time per iteration + warm-cache launch list of its kernels (huge shape)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PYTHONPATH=. python tools/sampler_timing.py > gpurun_out/sampler_timing.jsonl 2>&1; cat gpurun_out/sampler_timing.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active --cache-control none --clock-control none --csv -k regex:sample_ -c 6 --log-file gpurun_out/sampler_warm.csv PYTHONPATH=. python tools/sampler_timing.py huge > /dev/null 2>&1; echo "ncu rc=$?"
grep -v "^==" gpurun_out/sampler_warm.csv | python -c "
import csv,sys
r=list(csv.reader(sys.stdin))
h=r[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
for row in r[1:]:
    print(row[ii], row[ki][:30], row[mi], row[vi])
"
