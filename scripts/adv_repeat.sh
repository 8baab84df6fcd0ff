O=gpurun_out/adv3
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_bench_contract.py -q -m gpu > $O/contract.log 2>&1; echo rc=$? >> $O/contract.log
for i in 1 2 3; do SAGE_ADV_OUT=$O/adv_$i.json timeout 600 python -m pytest tests/test_gpu_adversary.py -q -m gpu > $O/adv_$i.log 2>&1; echo rc=$? >> $O/adv_$i.log; done
