# Round 2 (session 3) GPU pass over the product at HEAD (run from the repo root on
# the GPU box): smoke, every GPU test, bench lines for every config, the reference
# arm, the c2a launch list, ncu --set full of the c2a / c2c / c2cp4 / c2cp8 kernels,
# compute-sanitizer.  Config 4 runs separately (scripts/c4_full.sh, c4_slice.sh).
O=${1:-gpurun_out/r2s3final}
mkdir -p $O
nvidia-smi --query-gpu=name,uuid,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi_start.csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
SAGE_ADV_OUT=$O/adversary_test.json timeout 1500 python -m pytest tests -m gpu -q -rs --durations=15 > $O/gpu_tests.log 2>&1; echo tests_rc=$? >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_c2a.json 2> $O/bench_c2a.err
for c in c2b c2c c2cp4 c2cp8 c3p1 c3p4 c3p8 c3big c3bigp8 c1; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 python bench.py --config c3p1 --rounds 100000 --steps 10 --no-cpu-baseline > $O/bench_c3p1_r1e5.json 2> $O/bench_c3p1_r1e5.err
timeout 600 python bench.py --config c3big --rounds 100000 --steps 5 --no-cpu-baseline > $O/bench_c3big_r1e5.json 2> $O/bench_c3big_r1e5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c2a_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
for c in c2a c2c c2cp4 c2cp8; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sage_checksum_kernel -s 3 -c 1 -o $O/${c}_full python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-extra > $O/ncu_$c.log 2>&1
  ncu --page raw --csv -i $O/${c}_full.ncu-rep > $O/${c}_ncu_full_raw.csv 2>/dev/null
  ncu --page details --csv -i $O/${c}_full.ncu-rep > $O/${c}_ncu_full_details.csv 2>/dev/null
done
# compute-sanitizer is closed on this pool (runs under it left GPUs needing a reset); the last
# sanitizer pass at HEAD of session 2 is profiles/r02/final_s2/sanitizer_*.txt

for t in 524288:196608 524288:0 327680:0 1048576:196608 262144:196608; do bench/microbench l2gather ${t%:*} ${t#*:} >> $O/l2gather.jsonl; done
nvidia-smi --query-gpu=name,uuid,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi_end.csv
