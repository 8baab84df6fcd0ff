# One slice of config 4 at R = 10^7 (nonces [FIRST, FIRST + COUNT) of the R = 10^7
# stream; ~5.4 s per attestation); slices are merged with
# scripts/timing_distribution.py --merge.
FIRST=${1:-0}; COUNT=${2:-450}; O=${3:-gpurun_out/c4slice}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build_$FIRST.log 2>&1
nvidia-smi --query-gpu=name,uuid,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/smi_start_$FIRST.csv
timeout 3300 python scripts/timing_distribution.py --rounds 10000000 --counts $COUNT --first $FIRST --out $O/c4_r1e7_$FIRST.json > $O/c4_$FIRST.log 2>&1
echo rc=$? >> $O/c4_$FIRST.log
