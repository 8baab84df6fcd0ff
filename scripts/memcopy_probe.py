"""Memory-copy attack per placement (DESIGN.md sections 9 and 11).

The attacker keeps modified code at the attested address and a clean copy
elsewhere, and makes the kernel READ the copy while folding the original
address (P:434-438 binds the address, not the location read).  For each
placement the product's honest attestation (sage_attest) and the attacker's
kernel (test-only bench/libsage_adv.so, lab MEMCOPY knob) are interleaved;
the attacker must return the honest checksum, and the script reports its
slowdown and what the per-run and 16-challenge session rules reject.

    python scripts/memcopy_probe.py [--runs 48] [--out memcopy.json]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import adversary_lib  # noqa: E402
from paper_2209_03125_b200 import sage, verifier  # noqa: E402
from paper_2209_03125_b200.inputs import kernel_code_prefix, make_region, nonces  # noqa: E402

CASES = [  # (name, region bytes, rounds, context kwargs, adversary name)
    ("SMEM (c2a, 8 KiB)", 8192, 100_000, {}, "memory copy: stage a clean copy, fold the original address"),
    ("GLOBAL (8 KiB, L1-resident)", 8192, 100_000, {"placement": sage.SAGE_GLOBAL}, "memory copy on GLOBAL placement"),
    ("SAGE_HYBRID (c2c, 512 KiB)", 512 << 10, 100_000, {}, "memory copy on SAGE_HYBRID placement"),
    ("GLOBAL (c3, 256 MiB HBM)", 256 << 20, 10_000, {}, "memory copy on GLOBAL placement"),
]


def run_case(name, nbytes, R, cfg, adv_name, runs, dev):
    advs = {n: k for k, n, _ in adversary_lib.adversaries(True) + adversary_lib.adversaries(False)}
    k = advs[adv_name]
    with sage.Context(**cfg) as ctx:
        code = kernel_code_prefix(ctx, nbytes)
        if nbytes <= (1 << 20):
            region = torch.from_numpy(make_region(nbytes, prefix=code)).to(dev)
        else:
            g = torch.Generator(device=dev)
            g.manual_seed(0x5EED0001)
            region = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=dev, generator=g)
            region[:len(code)].copy_(torch.frombuffer(bytearray(code), dtype=torch.uint8))
        buf = torch.empty(2 * nbytes + 4096, dtype=torch.uint8, device=dev)
        off = (-buf.data_ptr()) % 256
        d, clean = buf[off:off + nbytes], buf[off + nbytes + 1024:off + 2 * nbytes + 1024]
        d.copy_(region)
        clean.copy_(region)
        delta = clean.data_ptr() - d.data_ptr()
        tampered_bytes = d[256:264].clone() ^ 0xFF
        original_bytes = d[256:264].clone()
        ns = nonces(runs + 3, master_seed=0x3E3C0 + nbytes)
        honest, attack, wrong = [], [], 0
        for i in range(-3, runs):
            nonce = ns[i + 3]
            h = ctx.attest(nonce, d, R)
            d[256:264].copy_(tampered_bytes)                    # the attacker's code at the attested address
            cs, t = adversary_lib.attest(k, nonce, d.data_ptr(), nbytes, R, copy_delta=delta)
            d[256:264].copy_(original_bytes)
            if i >= 0:
                honest.append(h.elapsed_ns * 1e-9)
                attack.append(t * 1e-9)
                wrong += cs != h.checksum
    half = len(honest) // 2
    rm = verifier.calibrate_robust(honest[:half], min_runs=min(30, half))
    sm = verifier.calibrate_session(honest[:half], 16, min_runs=min(30, half))
    med = float(np.median(honest[:half]))

    def sess(ts):
        return [verifier.verify_session([(j, 1, t, 1) for j, t in enumerate(ts[s:s + 16])], sm).accepted
                for s in range(0, len(ts) - 15, 16)]
    return {"case": name, "region_bytes": nbytes, "rounds": R, "runs": runs, "attacker": adv_name,
            "wrong_checksums": int(wrong), "honest_median_s": med,
            "slowdown": float(np.median(attack)) / med - 1.0,
            "per_run_rejected": float(np.mean([t > rm.threshold for t in attack])),
            "honest_per_run_rejected": float(np.mean([t > rm.threshold for t in honest[half:]])),
            "sessions_rejected": 1.0 - float(np.mean(sess(attack))) if len(attack) >= 16 else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=48)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    rows = []
    for case in CASES:
        r = run_case(*case, runs=a.runs, dev=dev)
        print(json.dumps(r), flush=True)
        rows.append(r)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rows, f, indent=1)
    return 0 if all(r["wrong_checksums"] == 0 for r in rows) else 1


if __name__ == "__main__":
    sys.exit(main())
