# Round-2 pass 9: SAGE_HYBRID with a fixed L1 window of the in-place part (evict_last)
O=gpurun_out/r2p9
mkdir -p $O
for w in 0 16384 32768 49152 65536 98304; do
  NO_PERSIST_LIMIT=1 PERSIST_BYTES=$w timeout 600 bench/variants_r2_c2cl1 100000 524288 > $O/c2c_l1win_$w.jsonl 2> $O/c2c_l1win_$w.err
done
M=gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_sectors.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
for w in 32768 65536; do
  NO_PERSIST_LIMIT=1 PERSIST_BYTES=$w timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/c2c_l1win_ncu_$w.csv bench/variants_r2_c2cl1 20000 524288 > /dev/null 2>&1
done
