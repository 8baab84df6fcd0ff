# One GPU pass over the product: smoke, GPU tests, bench lines for the configs, ncu launch list + full capture of c2a.
# Usage (from the repo root, on the GPU box): bash scripts/gpu_round.sh
mkdir -p gpurun_out
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
for c in c2a c2b c2c c3p1 c3p4 c3p8; do python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2a_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sage_checksum_kernel -c 1 -o gpurun_out/c2a_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c2a.log 2>&1
ncu --page raw --csv -i gpurun_out/c2a_full.ncu-rep > gpurun_out/c2a_ncu_full_raw.csv 2>/dev/null
ncu --page details --csv -i gpurun_out/c2a_full.ncu-rep > gpurun_out/c2a_ncu_full_details.csv 2>/dev/null
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
