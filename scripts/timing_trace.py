"""Per-run attestation timings with a concurrent nvidia-smi trace (dev aid for
the config-4 tail): writes JSON with, per run, host t0/t1 (monotonic),
elapsed_ns, device_ns, cycles; and the smi samples (timestamp, clocks, power,
throttle reasons).  Used to correlate slow runs with clock/power events.

    python scripts/timing_trace.py --rounds 100000 --runs 300 --gap-ms 0 --out gpurun_out/trace.json
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2209_03125_b200 import sage  # noqa: E402
from paper_2209_03125_b200.inputs import launched_kernel_prefix, make_region, nonces  # noqa: E402

Q = ("timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active,"
     "clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
     "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.hw_power_brake_slowdown")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=100000)
    ap.add_argument("--runs", type=int, default=300)
    ap.add_argument("--gap-ms", type=float, default=0.0)
    ap.add_argument("--out", default="gpurun_out/trace.json")
    a = ap.parse_args()
    lines = []
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=" + Q, "--format=csv,noheader", "-lms", "20"],
                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

    def rd():
        for ln in p.stdout:
            lines.append((time.time(), ln.strip()))
    th = threading.Thread(target=rd, daemon=True)
    th.start()
    dev = torch.device("cuda:0")
    region = torch.from_numpy(make_region(8192, prefix=launched_kernel_prefix(8192))).to(dev)
    runs = []
    with sage.Context() as ctx:
        ns = nonces(a.runs + 3, master_seed=0x7ACE)
        for k in range(3):
            ctx.attest(ns[k], region, a.rounds)
        for k in range(a.runs):
            t0 = time.time()
            r = ctx.attest(ns[3 + k], region, a.rounds)
            runs.append({"t0": t0, "elapsed_ns": r.elapsed_ns, "device_ns": r.device_ns, "cycles": r.cycles})
            if a.gap_ms:
                time.sleep(a.gap_ms / 1e3)
    time.sleep(0.2)
    p.terminate()
    th.join(timeout=2)
    with open(a.out, "w") as f:
        json.dump({"rounds": a.rounds, "gap_ms": a.gap_ms, "runs": runs, "smi": lines}, f)
    el = sorted(x["elapsed_ns"] for x in runs)
    print(json.dumps({"runs": len(runs), "p50_ms": el[len(el) // 2] / 1e6, "p99_ms": el[int(len(el) * 0.99)] / 1e6,
                      "max_ms": el[-1] / 1e6, "smi_samples": len(lines)}))


if __name__ == "__main__":
    main()
