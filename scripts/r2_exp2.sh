# Round-2 experiment pass 2: cache operators for the HBM (c3) and L2-sized (c2c)
# GLOBAL picks, the random-gather probe per cache operator, the pipe-balanced
# round prototype (BAL) with and without an injected IMAD, and counters for the
# 2-CTA cluster hybrid.
O=gpurun_out/r2
mkdir -p $O
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi2_start.csv
for op in 0 1 2 3; do for mb in 256 2048; do timeout 120 bench/microbench gather $mb $op >> $O/gather_ops.jsonl 2>&1; done; done
timeout 600 bench/variants_r2_c3ld 10000 268435456 > $O/c3ld.jsonl 2> $O/c3ld.err
timeout 900 bench/variants_r2_c3ld 10000 2147483648 > $O/c3ld_2g.jsonl 2> $O/c3ld_2g.err
M=gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_requests_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__sectors_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__m_xbar2l1tex_read_sectors.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/c3ld_ncu.csv bench/variants_r2_c3ld 2000 268435456 > /dev/null 2>&1
for i in 1 2; do timeout 600 bench/variants_r2_c2cld 100000 524288 >> $O/c2cld.jsonl 2>> $O/c2cld.err; done
timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/c2cld_ncu.csv bench/variants_r2_c2cld 20000 524288 > /dev/null 2>&1
for i in 1 2; do timeout 1200 bench/variants_r2_bal 100000 8192 >> $O/bal.jsonl 2>> $O/bal.err; done
timeout 900 ncu --set full --clock-control none -c 1 -k regex:sage_checksum_kernel -o $O/c2c_cluster2 bench/variants_r2_c2c 20000 524288 -1 "hybrid9 cluster2 unroll2 ILP2 stage196608 PAD8" > /dev/null 2>&1
ncu --page raw --csv -i $O/c2c_cluster2.ncu-rep > $O/c2c_cluster2_raw.csv 2>/dev/null
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi2_end.csv
