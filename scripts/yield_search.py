"""Hill-climb over the c2a loop's yield hints (lab).

Each generation writes a flip-set file -- the current best set and N mutants of
it (each toggles ~K random loop instructions' yield bit) -- for
scripts/sass_ctl_probe.py --flipsets, and `--update RESULTS.jsonl` adopts the
fastest mutant if it beats the re-measured best by more than --margin.

    python scripts/yield_search.py --state S.json --gen G --out cand.json
    (GPU) python scripts/sass_ctl_probe.py --modes orig --flipsets cand.json --out res.jsonl
    python scripts/yield_search.py --state S.json --update res.jsonl
"""
import argparse
import json
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import sass_ctl_probe as probe  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--state", required=True)
    ap.add_argument("--gen", type=int)
    ap.add_argument("--out")
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--init", default=None, help="comma-separated loop addresses of the starting set")
    ap.add_argument("--update")
    ap.add_argument("--margin", type=float, default=0.001)
    ap.add_argument("--emit-spec", default=None, help="write the best set as the build's yield spec "
                                                     "(paper_2209_03125_b200/csrc/c2a_yield.json)")
    ap.add_argument("--note", default="")
    ap.add_argument("--target", choices=("product", "attacker"), default="product")
    a = ap.parse_args()
    if a.target == "attacker":
        probe.FN, probe.CUBIN = probe.FN_ATTACKER, probe.build_attacker_cubin()
    state = json.load(open(a.state)) if os.path.exists(a.state) else {"best": [], "history": []}
    if a.init is not None and not state["best"]:
        state["best"] = sorted(int(x) for x in a.init.split(",") if x)
    if a.emit_spec:
        import hashlib
        blob = open(probe.CUBIN, "rb").read()
        off, size = probe.text_section(blob, ".text." + probe.FN)
        text = blob[off:off + size]
        spec = {"function": probe.FN, "yield_bit": probe.YIELD,
                "untuned_text_sha256": hashlib.sha256(text).hexdigest(),
                "yield": {str(x): 1 - ((int.from_bytes(text[x + 8:x + 16], "little") >> probe.YIELD) & 1)
                          for x in sorted(state["best"])},
                "note": a.note}
        json.dump(spec, open(a.emit_spec, "w"), indent=0)
        print("wrote", a.emit_spec, len(spec["yield"]), "hints")
        return
    if a.update:
        res = {json.loads(l)["mode"]: json.loads(l) for l in open(a.update)}
        orig = res["orig"]["ms_min"]
        best_ms = res["set:best"]["ms_min"]
        cands = {m: r["ms_min"] for m, r in res.items() if m.startswith("set:m")}
        m, ms = min(cands.items(), key=lambda kv: kv[1])
        rec = {"gen": state.get("gen"), "orig": orig, "best": best_ms, "best_vs_orig": best_ms / orig - 1,
               "top": m, "top_ms": ms, "top_vs_orig": ms / orig - 1,
               "all_ok": all(r["checksum_ok"] for r in res.values())}
        if ms < best_ms * (1 - a.margin):
            state["best"] = state["pending"][m[4:]]
            rec["adopted"] = True
        state["history"].append(rec)
        json.dump(state, open(a.state, "w"))
        print(json.dumps(rec))
        return
    lo, hi = probe.main_loop(probe.CUBIN)
    addrs = list(range(lo, hi, 16))
    rng = random.Random(1000 + a.gen)
    best = set(state["best"])
    cand = {"best": sorted(best)}
    for j in range(a.n):
        cand["m%d" % j] = sorted(best ^ set(rng.sample(addrs, a.k)))
    state["pending"] = cand
    state["gen"] = a.gen
    json.dump(state, open(a.state, "w"))
    json.dump(cand, open(a.out, "w"))


if __name__ == "__main__":
    main()
