O=${O:-gpurun_out/r2s2_head}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi_start.csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
SAGE_ADV_OUT=$O/adversary_test.json timeout 2400 python -m pytest tests -m gpu -q -rs --durations=25 > $O/gpu_tests.log 2>&1; echo tests_rc=$? >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_c2a.json 2> $O/bench_c2a.err
