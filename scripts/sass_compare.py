"""Compare the instruction streams of two cubins' kernels, ignoring code
addresses, encodings and constant-bank offsets (a kernel-parameter layout
change moves c[0x0][...] offsets but not the schedule).

    python scripts/sass_compare.py A.cubin NAME_A B.cubin NAME_B
"""
import re
import subprocess
import sys


def functions(path):
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    parts = re.split(r"\n\s+Function : ", sass)
    return {p.split("\n", 1)[0].strip(): p for p in parts[1:]}


def normalise(body):
    out = []
    for ln in body.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(.*?)\s*;?\s*(/\*.*\*/)?\s*$", ln)
        if not m:
            continue
        ins = m.group(1).rstrip(" ;")
        ins = re.sub(r"c\[0x0\]\[0x[0-9a-f]+\]", "c[0x0][K]", ins)
        ins = re.sub(r"\b0x[0-9a-f]+\b", "IMM", ins) if ins.startswith(("BRA", "CALL", "BSSY", "BSYNC")) else ins
        out.append(ins)
    return out


def same(a_path, a_name, b_path, b_name):
    fa, fb = functions(a_path), functions(b_path)
    na, nb = normalise(fa[a_name]), normalise(fb[b_name])
    if na == nb:
        return True, len(na), None
    for k, (x, y) in enumerate(zip(na, nb)):
        if x != y:
            return False, len(na), (k, x, y)
    return False, len(na), (min(len(na), len(nb)), "len %d" % len(na), "len %d" % len(nb))


if __name__ == "__main__":
    ok, n, diff = same(*sys.argv[1:5])
    print("same" if ok else "DIFFERENT", n, diff or "")
    sys.exit(0 if ok else 1)


def main_loop(path, name):
    """Normalised instruction stream of a kernel's main round loop (the
    backward branch whose body holds the most SHFL.IDX, as scripts/sass_loop.py)."""
    f = functions(path)[name]
    ins = []
    for ln in f.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    best = None
    for addr, txt in ins:
        m = re.search(r"BRA.*?(0x[0-9a-f]+)\s*$", txt)
        if m and int(m.group(1), 16) < addr:
            body = [t for a, t in ins if int(m.group(1), 16) <= a <= addr]
            if any("EXIT" in t or "SHFL.DOWN" in t for t in body):
                continue
            nsh = sum("SHFL.IDX" in t for t in body)
            if nsh and (best is None or nsh > best[0]):
                best = (nsh, body)
    if best is None:
        return []
    return [re.sub(r"0x[0-9a-f]+$", "ADDR", re.sub(r"c\[0x0\]\[0x[0-9a-f]+\]", "c[0x0][K]", t)) for t in best[1]]
