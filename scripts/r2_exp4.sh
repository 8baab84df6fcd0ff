# Round-2 pass 4: adversary test with the attacker-searched schedules (raw times
# recorded), hybrid stage sweep with L1-bypassing global loads.
O=gpurun_out/r2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build4.log 2>&1
SAGE_ADV_OUT=$O/adversary_test4.json timeout 1200 python -m pytest tests/test_gpu_adversary.py -x -q -s > $O/adv_test4.log 2>&1; echo rc=$? >> $O/adv_test4.log
for i in 1 2; do timeout 600 bench/variants_r2_c2cst 100000 524288 >> $O/c2cst.jsonl 2>> $O/c2cst.err; done
