# Round-2 pass 7: the attacker's search widened -- lowering knobs (XS, ADDR) for +1 IMAD
# per round, and +2 / +4 IMADs and +1 ALU op per round over UNROLL x PAD.
O=gpurun_out/r2p7
mkdir -p $O
for spec in "16 1 a" "16 2 b" "16 5 c" "16 6 d" "0 4 e"; do set -- $spec
  timeout 900 python scripts/schedule_search.py --no-build --run --passes 2 --xs $1 --addr $2 --unroll 9,12,15,17,18,21 --pad 0-12 --extra -1 --every 1 --binary bench/variants_atkx_$3 --out $O/attacker_x_xs$1_addr$2.jsonl > $O/attacker_x_$3.log 2>&1
done
for e in 2 4; do
  timeout 1200 python scripts/schedule_search.py --no-build --run --passes 2 --unroll 8-24 --pad 0-12 --extra -$e --every 1 --binary bench/variants_atk$e --out $O/attacker_imad$e.jsonl > $O/attacker_imad$e.log 2>&1
done
timeout 1200 python scripts/schedule_search.py --no-build --run --passes 2 --unroll 8-24 --pad 0-12 --extra 1 --every 1 --binary bench/variants_atkalu --out $O/attacker_alu1.jsonl > $O/attacker_alu1.log 2>&1
