# Round-2 experiment pass 1 (run from the repo root on the GPU box):
# product sanity after the lab/product split, the attacker's schedule search,
# the 2-CTA cluster hybrid (c2c) and L2 residency variants for the HBM region (c3).
O=gpurun_out/r2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo tests_rc=$? >> $O/gpu_tests.log
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi_start.csv
for i in 1 2; do timeout 900 bench/variants_r2_atk 100000 8192 >> $O/atk.jsonl 2>> $O/atk.err; done
for i in 1 2; do timeout 600 bench/variants_r2_c2c 100000 524288 >> $O/c2c.jsonl 2>> $O/c2c.err; done
timeout 600 bench/variants_r2_c3 10000 268435456 > $O/c3_base.jsonl 2> $O/c3_base.err
for pb in 33554432 67108864 100663296 134217728; do
  PERSIST_BYTES=$pb timeout 600 bench/variants_r2_c3 10000 268435456 -1 LD > $O/c3_persist_$pb.jsonl 2> $O/c3_persist_$pb.err
done
for wb in 33554432 67108864 100663296 134217728; do
  WINDOW_BYTES=$wb timeout 600 bench/variants_r2_c3 10000 268435456 -1 LD0 > $O/c3_window_$wb.jsonl 2> $O/c3_window_$wb.err
done
M=gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,dram__bytes_read.sum,dram__sectors_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_requests_srcunit_tex_op_read.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/c3_ncu_base.csv bench/variants_r2_c3 10000 268435456 -1 "P1 global xs16 unroll16 LD" > /dev/null 2>&1
for pb in 67108864 134217728; do
  PERSIST_BYTES=$pb timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/c3_ncu_persist_$pb.csv bench/variants_r2_c3 10000 268435456 -1 "P1 global xs16 unroll16 LD" > /dev/null 2>&1
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi_end.csv
