O=${1:-gpurun_out/p4}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py tests/test_sass_evidence.py -q -rs > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for c in c2cp4 c2cp8 c2c; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
