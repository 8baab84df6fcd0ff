# Run the GPU suite N times back to back (flake check), as the driver does (-x).
O=${1:-gpurun_out/suite}; N=${2:-2}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
for i in $(seq 1 $N); do
  timeout 1200 python -m pytest tests -x -q -m gpu > $O/gpu_tests_$i.log 2>&1; echo rc=$? >> $O/gpu_tests_$i.log
done
