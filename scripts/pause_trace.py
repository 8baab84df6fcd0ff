"""Arrival times of B200's whole-chip pauses.

Runs back-to-back short attestations (c2a geometry, R = 10^4, ~5.4 ms each) for
`--seconds`, records each run's %globaltimer span and host start time, and
reports the runs that took > `--excess` ms longer than the median: their
times, the inter-arrival distribution (Poisson -> exponential, coefficient of
variation ~1; a periodic source -> CV << 1 and a dominant period).

    python scripts/pause_trace.py --seconds 60 --out pauses.json
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2209_03125_b200 import sage  # noqa: E402
from paper_2209_03125_b200.inputs import launched_kernel_prefix, make_region  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=60.0)
    ap.add_argument("--rounds", type=int, default=10_000)
    ap.add_argument("--excess", type=float, default=0.8, help="ms above the median that marks a pause")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    region = torch.from_numpy(make_region(8192, prefix=launched_kernel_prefix(8192))).to("cuda")
    starts, spans, walls = [], [], []
    with sage.Context() as ctx:
        for k in range(5):
            ctx.attest(k, region, a.rounds)
        t_end = time.monotonic() + a.seconds
        k = 0
        while time.monotonic() < t_end:
            t0 = time.monotonic()
            r = ctx.attest(0x9A05E + k, region, a.rounds)
            starts.append(t0)
            spans.append(r.device_ns * 1e-6)
            walls.append(r.elapsed_ns * 1e-6)
            k += 1
    med = statistics.median(spans)
    t_first = starts[0]
    events = [(starts[i] - t_first, spans[i] - med) for i in range(len(spans)) if spans[i] - med > a.excess]
    gaps = [events[i + 1][0] - events[i][0] for i in range(len(events) - 1)]
    cv = statistics.pstdev(gaps) / statistics.mean(gaps) if len(gaps) > 1 else None
    res = {"runs": len(spans), "seconds": starts[-1] - t_first, "median_span_ms": med, "pauses": len(events),
           "rate_per_s": len(events) / (starts[-1] - t_first), "pause_excess_ms_median":
           statistics.median([e for _, e in events]) if events else None,
           "interarrival_s_mean": statistics.mean(gaps) if gaps else None,
           "interarrival_cv": cv, "interarrival_s_sorted": sorted(round(g, 4) for g in gaps),
           "events": [[round(t, 4), round(e, 4)] for t, e in events]}
    print(json.dumps({k: v for k, v in res.items() if k not in ("events", "interarrival_s_sorted")}))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
