"""Throughput of the GPU kernel hash h = SHA-256(r || code) (Eq. 9) vs host
hashlib, for a few code sizes; one JSON line per size (dev aid; results in
profiles/)."""
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2209_03125_b200 import sage  # noqa: E402

if __name__ == "__main__":
    r = bytes(range(32))
    with sage.Context(blocks=1, threads=32) as ctx:
        for n in (4096, 65536, 1 << 20, 16 << 20):
            code = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
            ctx.kernel_hash(r, code)
            ts = []
            for _ in range(5):
                h, ns = ctx.kernel_hash(r, code)
                ts.append(ns / 1e9)
            host = code.cpu().numpy().tobytes()
            t0 = time.perf_counter()
            hh = hashlib.sha256(r + host).digest()
            t_cpu = time.perf_counter() - t0
            t = min(ts)
            print(json.dumps({"code_bytes": n, "gpu_s": t, "gpu_MBps": n / t / 1e6, "gpu_blocks_per_s": (n + 41) / 64 / t,
                              "hashlib_s": t_cpu, "hashlib_MBps": n / t_cpu / 1e6, "match": hh == h}), flush=True)
