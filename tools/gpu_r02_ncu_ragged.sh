mkdir -p gpurun_out
C1="python bench.py --config large --steps 1 --warmup 3 --no-e2e --no-parity --no-cpu-baseline"
PCDM_LAYOUT=ragged $C1 > gpurun_out/plain1.log 2>&1 && \
PCDM_LAYOUT=ragged ncu --set full --clock-control none --import-source on -k regex:pcdm_ragged -s 10 -c 1 -o gpurun_out/r02_ragged_large $C1 > gpurun_out/ncu1.log 2>&1
$C1 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pcdm_packed -s 10 -c 1 -o gpurun_out/r02_packed_large $C1 > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu1.log gpurun_out/ncu2.log
