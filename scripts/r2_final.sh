# Round-2 GPU pass over the product (run from the repo root on the GPU box):
# smoke, every GPU test, bench lines, ncu launch list + full capture of the c2a
# kernel, the reference arm, compute-sanitizer, and a config-4 capture.
O=${1:-gpurun_out/r2final}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi_start.csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
SAGE_ADV_OUT=$O/adversary_test.json timeout 2400 python -m pytest tests -m gpu -q -rs > $O/gpu_tests.log 2>&1; echo tests_rc=$? >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_c2a.json 2> $O/bench_c2a.err
for c in c2b c3big c3bigp8 c1; do timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c2a_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sage_checksum_kernel -c 1 -o $O/c2a_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra > $O/ncu_c2a.log 2>&1
ncu --page raw --csv -i $O/c2a_full.ncu-rep > $O/c2a_ncu_full_raw.csv 2>/dev/null
ncu --page details --csv -i $O/c2a_full.ncu-rep > $O/c2a_ncu_full_details.csv 2>/dev/null
timeout 1200 ncu --set full --clock-control none -k regex:sage_checksum_kernel -c 1 -o $O/c2c_full python bench.py --config c2c --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c2c.log 2>&1
ncu --page raw --csv -i $O/c2c_full.ncu-rep > $O/c2c_ncu_full_raw.csv 2>/dev/null
bash scripts/sanitize.sh $O
timeout 1200 python scripts/timing_distribution.py --rounds 10000,100000,1000000 --counts 1000,1000,200 --out $O/c4_timing.json > $O/c4_timing.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi_end.csv
rm -f $O/*.ncu-rep.bak
