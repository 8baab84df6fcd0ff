# Round-2 pass 6: new parity boundary tests, memory-copy probe per placement, bench line.
O=gpurun_out/r2p6
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "boundaries" > $O/boundary_tests.log 2>&1; echo rc=$? >> $O/boundary_tests.log
timeout 1200 python scripts/memcopy_probe.py --runs 48 --out $O/memcopy_probe.json > $O/memcopy_probe.log 2>&1; echo rc=$? >> $O/memcopy_probe.log
timeout 900 python bench.py > $O/bench_c2a.json 2> $O/bench_c2a.err
