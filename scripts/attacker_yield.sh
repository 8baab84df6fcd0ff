# The attacker's side of the scheduling-hint search: the same
# hill-climb as the product's (scripts/yield_search.py) on the adversary test's fastest
# attacker kernel (+1 IMAD / round, UNROLL 9 / PAD 1), from ptxas' hints; then the
# attacker's best and the shipped product timed back to back on the same box.
O=${O:-gpurun_out/r2s3_atk}
mkdir -p $O
run() {  # gens K margin
  for g in $(seq $1 $2); do
    python scripts/yield_search.py --target attacker --state $O/state.json --gen $g --out $O/cand.json --init "" --n 30 --k $3
    timeout 300 python scripts/sass_ctl_probe.py --target attacker --reps 3 --modes orig --flipsets $O/cand.json --out $O/res_$g.jsonl > $O/probe_$g.log 2>&1 || return
    python scripts/yield_search.py --target attacker --state $O/state.json --update $O/res_$g.jsonl --margin $4 >> $O/history.jsonl
  done
}
run 1 12 30 0.001
run 13 40 3 0.0005
python - <<PY
import json
s = json.load(open("$O/state.json"))
json.dump({"best": s["best"]}, open("$O/attacker_best.json", "w"))
spec = json.load(open("paper_2209_03125_b200/csrc/c2a_yield.json"))
json.dump({"shipped": [int(a) for a in spec["yield"]]}, open("$O/product_shipped.json", "w"))
PY
for k in 1 2; do
  timeout 300 python scripts/sass_ctl_probe.py --target attacker --reps 5 --modes orig --flipsets $O/attacker_best.json --out $O/final_attacker.jsonl >> $O/final.log 2>&1
  timeout 300 python scripts/sass_ctl_probe.py --target product --reps 5 --modes orig --flipsets $O/product_shipped.json --out $O/final_product.jsonl >> $O/final.log 2>&1
done
