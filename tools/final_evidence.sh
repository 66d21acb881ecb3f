#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): the GPU suite, smoke, the default bench
# line (huge), every config's bench line with first-step oracle parity, the reference arm
# and the ncu launch list of the bench command.  Outputs under gpurun_out/final_*.
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/final_smi.txt
python -m pytest tests -m gpu -q > $O/final_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/final_pytest.txt
python __graft_entry__.py smoke > $O/final_smoke.txt 2>&1; echo "smoke rc=$?" >> $O/final_smoke.txt
python bench.py > $O/final_bench_huge.json 2> $O/final_bench_huge.err; echo "bench rc=$?" >> $O/final_bench_huge.err
rm -f $O/final_configs.jsonl
for spec in "tiny 32" "medium 1024" "skewed 256" "skewed 4096" "skewed 65536" "large 65536" "ragged 65536"; do
  set -- $spec
  python bench.py --config $1 --tau $2 --steps 5 --warmup 3 >> $O/final_configs.jsonl 2>> $O/final_configs.err
done
python bench.py --steps 5 --warmup 3 >> $O/final_configs.jsonl 2>> $O/final_configs.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/final_reference.json 2> $O/final_reference.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-parity"
$CMD > $O/final_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'pcdm_|batch_|screen_|sample_|xhdr_|neg_b|scatter_x|round_r|residual_|objective_|row_counts|validate_|col_norms|pack_kernel|max_kernel|max_len|hot_cand|gather_list|check_finite' -c 1500 --csv --log-file $O/final_launches.csv $CMD > $O/final_ncu.log 2>&1
tools/capture_config_traffic.sh "large 65536 pcdm_packed" "skewed 65536 pcdm_packed" > $O/final_capture.txt 2>&1
tail -n 3 $O/final_pytest.txt; tail -n 2 $O/final_smoke.txt; wc -l $O/final_configs.jsonl; cut -c1-300 $O/final_bench_huge.json
