# Round-2 pass 3: attacker schedule searches, HBM size sweep, new GPU tests, bench.
O=gpurun_out/r2
mkdir -p $O
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi3_start.csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke3.log 2>&1
SAGE_ADV_OUT=$O/adversary_test.json timeout 1200 python -m pytest tests/test_gpu_adversary.py tests/test_gpu_boundary.py tests/test_gpu_parity_large.py -x -q -s > $O/gpu_tests_new.log 2>&1; echo rc=$? >> $O/gpu_tests_new.log
for spec in "8-14 a1" "15-21 a2" "22-28 a3" "29-36 a4"; do set -- $spec
  timeout 900 python scripts/schedule_search.py --no-build --run --passes 2 --unroll $1 --pad 0-12 --extra -1 --every 1 --binary bench/variants_atk_$2 --out $O/attacker_search_$2.jsonl > $O/attacker_search_$2.log 2>&1
done
timeout 900 python scripts/schedule_search.py --no-build --run --passes 2 --unroll 7,14,21,28,35 --pad 0-12 --extra -1 --every 7 --binary bench/variants_atk7 --out $O/attacker_search_every7.jsonl > $O/attacker_search_every7.log 2>&1
for mb in 64 128 192 256 384 512 768 1024 1536 2048 3072 4096; do timeout 120 bench/microbench gather $mb 0 >> $O/gather_sizes.jsonl 2>&1; done
for b in 134217728 268435456 536870912 1073741824 2147483648 4294967296; do
  timeout 600 bench/variants_r2_c3ld 10000 $b -1 "P1 global xs16 unroll16 LD0" >> $O/c3_sizes.jsonl 2>> $O/c3_sizes.err
done
M=gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_requests_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__sectors_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__m_xbar2l1tex_read_sectors.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__issue_active.avg.pct_of_peak_sustained_active
for b in 268435456 1073741824 2147483648; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/c3_ncu_size_$b.csv bench/variants_r2_c3ld 2000 $b -1 "P1 global xs16 unroll16 LD0" > /dev/null 2>&1
done
timeout 900 python bench.py > $O/bench_c2a.json 2> $O/bench_c2a.err
timeout 900 python -m pytest tests/test_bench_contract.py -x -q > $O/bench_contract.log 2>&1; echo rc=$? >> $O/bench_contract.log
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi3_end.csv
