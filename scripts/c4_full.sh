# Config 4 at full size (BASELINE configs[3]): 1000 nonces at R = 10^4, 10^5 and
# 10^6 (~10 min).  R = 10^7 (~90 min of attestations) runs in slices that fit a
# one-hour GPU call: scripts/c4_slice.sh, merged with timing_distribution.py --merge.
O=${1:-gpurun_out/c4full}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi --query-gpu=name,uuid,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi_start.csv
timeout 3000 python scripts/timing_distribution.py --rounds 10000,100000,1000000 --counts 1000,1000,1000 --out $O/c4_timing_1000.json > $O/c4.log 2>&1
echo rc=$? >> $O/c4.log
nvidia-smi --query-gpu=name,uuid,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi_end.csv
