# Session-3 closing GPU pass at HEAD: smoke, the GPU suite as the driver runs it (-x),
# the default bench line (c2a + extra), the reference arm, the c2a launch list.
O=${1:-gpurun_out/r2s3final2}
mkdir -p $O
nvidia-smi --query-gpu=name,uuid,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi_start.csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
SAGE_ADV_OUT=$O/adversary_test.json timeout 1500 python -m pytest tests -m gpu -x -q -rs --durations=15 > $O/gpu_tests.log 2>&1; echo tests_rc=$? >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_c2a.json 2> $O/bench_c2a.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c2a_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
nvidia-smi --query-gpu=name,uuid,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi_end.csv
tail -3 $O/gpu_tests.log
