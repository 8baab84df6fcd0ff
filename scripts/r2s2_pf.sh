# Round 2 (session 2): whole-line L1 prefetch on the hybrid's global picks (lab ADDR 11)
O=${1:-gpurun_out/pf}
mkdir -p $O
for pass in 1 2; do timeout 600 bench/variants_pf 100000 524288 -1 >> $O/pf_524288.jsonl 2>> $O/pf.err; done
M=gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_miss.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__m_xbar2l1tex_read_sectors.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__m_l1tex2xbar_req.sum,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second
for v in "P1 hybrid8 unroll2 ILP2 stage196608 PAD8" "P1 hybrid11 unroll2 ILP2 stage196608 PAD8 LD0" "P1 hybrid11 unroll2 ILP2 stage131072 PAD8 LD0"; do
  tag=$(echo "$v" | tr ' ' '_')
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/ncu_$tag.csv bench/variants_pf 20000 524288 -1 "$v" > /dev/null 2>&1
done
