O=${O:-gpurun_out/r2s3_tuned}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tuned.py -q -rs > $O/tuned_tests.log 2>&1; echo rc=$? >> $O/tuned_tests.log
SAGE_ADV_OUT=$O/adversary_test.json timeout 1400 python -m pytest tests -m gpu -x -q -rs --durations=10 > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 600 python bench.py > $O/bench_c2a.json 2> $O/bench_c2a.err
SAGE_NO_TUNED=1 timeout 600 python bench.py --no-extra --no-cpu-baseline > $O/bench_c2a_untuned.json 2> $O/bench_c2a_untuned.err
timeout 600 python bench.py --no-extra --no-cpu-baseline > $O/bench_c2a_tuned2.json 2> $O/bench_c2a_tuned2.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sage_checksum_kernel -s 3 -c 1 -o $O/c2a_full python bench.py --config c2a --steps 1 --warmup 3 --no-cpu-baseline --no-extra > $O/ncu_c2a.log 2>&1
ncu --page raw --csv -i $O/c2a_full.ncu-rep > $O/c2a_ncu_full_raw.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c2a_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
tail -3 $O/tuned_tests.log; tail -3 $O/gpu_tests.log
