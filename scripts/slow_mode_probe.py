"""Attestation-time slow mode vs NVML counters
(dev aid): for each attestation record elapsed/device time and cycles, the
deltas of NVML's cumulative perf-policy violation times (power, thermal,
board limit, reliability, sync boost, ...), the energy consumed, and the SM
clock right after.  Writes JSON; prints a summary correlating slow runs with
violation deltas.

    python scripts/slow_mode_probe.py --runs 400 --out gpurun_out/slow_mode.json
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_2209_03125_b200 import sage  # noqa: E402
from paper_2209_03125_b200.inputs import launched_kernel_prefix, make_region, nonces  # noqa: E402

POLICIES = {name: getattr(pynvml, "NVML_PERF_POLICY_" + name) for name in
            ("POWER", "THERMAL", "SYNC_BOOST", "BOARD_LIMIT", "LOW_UTILIZATION", "RELIABILITY",
             "TOTAL_APP_CLOCKS", "TOTAL_BASE_CLOCKS")}


def violations(h):
    out = {}
    for name, pol in POLICIES.items():
        try:
            v = pynvml.nvmlDeviceGetViolationStatus(h, pol)
            out[name] = int(v.violationTime)
        except pynvml.NVMLError:
            out[name] = None
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=400)
    ap.add_argument("--rounds", type=int, default=100_000)
    ap.add_argument("--out", default="gpurun_out/slow_mode.json")
    a = ap.parse_args()
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    region = torch.from_numpy(make_region(8192, prefix=launched_kernel_prefix(8192))).to("cuda")
    runs = []
    with sage.Context() as ctx:
        ns = nonces(a.runs + 3, master_seed=0x51070)
        for k in range(3):
            ctx.attest(ns[k], region, a.rounds)
        for k in range(a.runs):
            v0 = violations(h)
            e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
            r = ctx.attest(ns[3 + k], region, a.rounds)
            e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
            v1 = violations(h)
            clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            runs.append({"elapsed_ns": r.elapsed_ns, "device_ns": r.device_ns, "cycles": r.cycles,
                         "energy_mj": e1 - e0, "sm_mhz_after": clk,
                         "viol_ns": {n: (v1[n] - v0[n]) if v0[n] is not None else None for n in POLICIES}})
    with open(a.out, "w") as f:
        json.dump(runs, f)
    cyc = [r["cycles"] for r in runs]
    med = statistics.median(cyc)
    slow = [r for r in runs if r["cycles"] > med * 1.01]
    fast = [r for r in runs if r["cycles"] <= med * 1.01]

    def agg(rs, key):
        vals = [r["viol_ns"][key] for r in rs if r["viol_ns"][key] is not None]
        return (statistics.mean(vals) if vals else None, sum(1 for x in vals if x > 0))
    summary = {"runs": len(runs), "slow_runs": len(slow), "median_cycles": med,
               "energy_mj_fast": statistics.mean(r["energy_mj"] for r in fast) if fast else None,
               "energy_mj_slow": statistics.mean(r["energy_mj"] for r in slow) if slow else None}
    for key in POLICIES:
        summary["viol_" + key] = {"fast_mean_ns_nonzero_count": agg(fast, key), "slow_mean_ns_nonzero_count":
                                  agg(slow, key)}
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
