"""Per-round SASS histogram of the checksum kernels' main loop (dev aid).

    python scripts/sass_loop.py <cubin-or-so> [name-filter]

For every kernel: the backward-branch loop with the most SHFL.IDX (one per
SCS-2 round) is the main loop; prints instructions per round split by pipe
(FMA: IMAD*, ALU: LOP3/SHF/IADD3/LEA/..., other)."""
import re
import subprocess
import sys
from collections import Counter

ALU = ("LOP3", "SHF", "IADD3", "LEA", "SEL", "ISETP", "MOV", "PRMT", "IABS", "IMNMX", "FLO", "POPC")


def analyse(path, filt=""):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", out)
    res = {}
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if filt not in name:
            continue
        ins = []
        for ln in f.splitlines():
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        best = None
        for addr, txt in ins:
            m = re.search(r"BRA.*?(0x[0-9a-f]+)\s*$", txt)
            if m:
                tgt = int(m.group(1), 16)
                if tgt < addr:
                    body = [t for a, t in ins if tgt <= a <= addr]
                    if any("EXIT" in t or "SHFL.DOWN" in t for t in body):
                        continue  # an outer loop around the prologue/epilogue, not the round loop
                    nsh = sum("SHFL.IDX" in t for t in body)
                    if nsh and (best is None or nsh > best[0] or (nsh == best[0] and len(body) < len(best[1]))):
                        best = (nsh, body)
        if not best:
            continue
        nsh, body = best
        c = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in body)
        # VIADD issues to the FMA pipe on sm_100 (ncu c2a: ALU 31.2, FMA-heavy 26 per round)
        fma = sum(v for k, v in c.items() if k.startswith("IMAD") or k.startswith("VIADD"))
        wide = sum(v for k, v in c.items() if k.startswith("IMAD.WIDE") or k.startswith("IMAD.HI"))
        alu = sum(v for k, v in c.items() if k.split(".")[0] in ALU)
        res[name] = dict(rounds=nsh, per_round=len(body) / nsh, fma=fma / nsh, wide=wide / nsh, alu=alu / nsh,
                         hist={k: v for k, v in c.most_common()})
    return res


if __name__ == "__main__":
    r = analyse(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
    for name, d in r.items():
        print("%-70s instr/round %.2f  FMA %.2f (wide %.2f)  ALU %.2f" % (name[:70], d["per_round"], d["fma"],
                                                                           d["wide"], d["alu"]))
        if "-v" in sys.argv:
            print("    ", d["hist"])
