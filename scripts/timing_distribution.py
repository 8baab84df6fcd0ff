"""Config 4: attestation wall-time distribution over many nonces.

For each round count R, runs `n` attestations with independent nonces through
the public C ABI (sage_attest_debug: synchronous, per-warp partials), records
the verifier's timing quantity elapsed_ns (host t1 - t0) plus the
device span and cycles, and reports p50/p99/sigma, the paper's threshold
T_avg + 2.5 sigma calibrated on the first half of the runs, and the empirical
false-positive rate of that threshold on the second half (Q16).

Parity: every attestation checks sum(per-warp partials) == checksum (mod 2^64)
on the spot; for a few nonces per R it stores one sampled warp's partial,
which tests/test_c4_samples.py recomputes with the CPU oracle (this script does
not import the oracle).

    python scripts/timing_distribution.py --out profiles/r01/c4_timing.json
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench.clocks import ClockSampler  # noqa: E402
from paper_2209_03125_b200 import sage, verifier  # noqa: E402
from paper_2209_03125_b200.inputs import launched_kernel_prefix, make_region, nonces  # noqa: E402

M64 = (1 << 64) - 1


def moments(xs):
    m = statistics.mean(xs)
    sd = statistics.pstdev(xs)
    if sd == 0:
        return 0.0, 0.0
    n = len(xs)
    skew = sum(((x - m) / sd) ** 3 for x in xs) / n
    kurt = sum(((x - m) / sd) ** 4 for x in xs) / n - 3.0
    return skew, kurt


def summarize(R, n, el, dv, cyc, samples, sum_ok, wall_s, clocks):
    """Statistics of one round count's attestations (el: elapsed s in nonce order)."""
    half = len(el) // 2
    model = verifier.calibrate(el[:half], min_runs=min(30, half))
    fp = sum(1 for x in el[half:] if x > model.threshold) / max(1, len(el) - half)
    model_all = verifier.calibrate(el, min_runs=min(30, len(el)))
    quantile_fp = {}
    for q in (0.95, 0.99):                               # SPEC S:311 empirical-quantile rule
        qm = verifier.calibrate_quantile(el[:half], q=q, min_runs=min(30, half))
        quantile_fp["q%.2f" % q] = {"threshold": qm.threshold,
                                    "false_positive_rate_second_half":
                                        sum(1 for x in el[half:] if x > qm.threshold) / max(1, len(el) - half)}
    rm = verifier.calibrate_robust(el[:half], min_runs=min(30, half))   # median/MAD relative rule
    robust = {"threshold": rm.threshold, "margin": rm.margin,
              "false_positive_rate_second_half": sum(1 for x in el[half:] if x > rm.threshold) /
              max(1, len(el) - half)}
    sess = {}
    if half >= 32:
        sm = verifier.calibrate_session(el[:half], 16, min_runs=min(30, half))
        rest = el[half:]
        verdicts = [verifier.verify_session([(i, 1, t, 1) for i, t in enumerate(rest[j:j + 16])], sm).accepted
                    for j in range(0, len(rest) - 15, 16)]
        sess = {"m": 16, "threshold": sm.threshold, "margin": sm.margin, "sessions": len(verdicts),
                "false_positive_rate_second_half": (1.0 - sum(verdicts) / len(verdicts)) if verdicts else None}
    skew, kurt = moments(el)
    return {"rounds": R, "n_attest": len(el), "wall_s": wall_s, "clocks": clocks,
            "elapsed_s": {"p50": verifier.percentile(el, 50), "p99": verifier.percentile(el, 99),
                          "min": min(el), "max": max(el), "mean": model_all.t_avg, "sigma": model_all.sigma,
                          "threshold_2p5sigma": model_all.threshold, "skew": skew, "excess_kurtosis": kurt,
                          "cv": model_all.sigma / model_all.t_avg},
            "device_s": {"p50": verifier.percentile(dv, 50), "p99": verifier.percentile(dv, 99),
                         "sigma": statistics.pstdev(dv)},
            "cycles": {"p50": verifier.percentile(cyc, 50), "max": max(cyc)},
            "calibrated_on_first_half": {"t_avg": model.t_avg, "sigma": model.sigma,
                                         "threshold": model.threshold},
            "false_positive_rate_second_half": fp, "normal_tail_2p5": verifier.normal_tail(2.5),
            "quantile_rule": quantile_fp, "robust_rule": robust, "session_rule": sess,
            "stalls": verifier.stall_estimate(el),
            "thread_rounds_per_s_p50": n * R / verifier.percentile(el, 50),
            "sum_of_partials_ok": sum_ok, "samples": samples,
            "elapsed_ns_all": [int(round(x * 1e9)) for x in el],
            "device_ns_all": [int(round(x * 1e9)) for x in dv], "cycles_all": cyc}


BIG = ("samples", "elapsed_ns_all", "device_ns_all", "cycles_all")


def gpu_uuid():
    try:
        return subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=uuid", "--format=csv,noheader"],
                              capture_output=True, text=True, timeout=30).stdout.strip()
    except (OSError, subprocess.SubprocessError):
        return None


def run(rounds_list, counts, samples_per_r, out, first=0):
    """Attest nonces [first, first + count) of each round count's nonce stream."""
    dev = torch.device("cuda:0")
    region_np = make_region(8192, prefix=launched_kernel_prefix(8192))
    region = torch.from_numpy(region_np).to(dev)
    stream = torch.cuda.Stream()
    result = {"what": "SAGE attestation-time distribution (config 4)", "gpu": torch.cuda.get_device_name(0),
              "gpu_uuid": gpu_uuid(), "region_hex": region_np.tobytes().hex(), "region_va": region.data_ptr(),
              "P": 1, "first_nonce_index": first, "per_R": []}

    def dump():
        with open(out, "w") as f:                       # rewritten as it goes: a cut-off run keeps what it has
            json.dump(result, f, indent=1)

    with sage.Context(stream=stream) as ctx:
        info = ctx.query()
        n = info.blocks * info.threads
        result.update({"blocks": info.blocks, "threads": info.threads, "threads_total": n})
        pw = torch.zeros(n // 32, dtype=torch.int64, device=dev)
        for R, count in zip(rounds_list, counts):
            ns = nonces(first + count, master_seed=0xC4000000 + R)[first:]
            for k in range(3):                                   # warm-up
                ctx.attest(ns[k] ^ 0xFFFF, region, R)
            el, dv, cyc, samples, sum_ok = [], [], [], [], 0
            clk = ClockSampler(torch.cuda.current_device()).start()
            t_start = time.time()
            for k, nonce in enumerate(ns):
                res = ctx.attest_debug(nonce, region, R, pw)
                el.append(res.elapsed_ns / 1e9)
                dv.append(res.device_ns / 1e9)
                cyc.append(res.cycles)
                parts = pw.cpu().tolist()
                sum_ok += (sum(int(v) & M64 for v in parts) & M64) == res.checksum
                if k < samples_per_r:
                    w = (nonce >> 17) % (n // 32)
                    samples.append({"nonce": nonce, "checksum": res.checksum, "warp": int(w),
                                    "warp_partial": int(parts[w]) & M64, "region_va": region.data_ptr()})
                if R >= 1_000_000 and (k + 1) % 20 == 0:         # long round counts: keep partial progress
                    result["partial"] = {"rounds": R, "n_attest": len(el), "sum_of_partials_ok": sum_ok,
                                         "samples": samples, "elapsed_ns_all": [int(round(x * 1e9)) for x in el],
                                         "device_ns_all": [int(round(x * 1e9)) for x in dv], "cycles_all": cyc}
                    dump()
            wall_s = time.time() - t_start
            entry = summarize(R, n, el, dv, cyc, samples, sum_ok, wall_s, clk.stop())
            entry["first_nonce_index"] = first
            result.pop("partial", None)
            result["per_R"].append(entry)
            dump()
            print(json.dumps({k: v for k, v in entry.items() if k not in BIG}), flush=True)


def merge(paths, out):
    """Concatenate the per-R raw arrays of several captures (nonce slices of the same
    streams, possibly partial) in nonce order and recompute the statistics."""
    caps = [json.load(open(p)) for p in paths]
    base = caps[0]
    assert all(c["region_hex"] == base["region_hex"] and c["threads_total"] == base["threads_total"] for c in caps)
    chunks = {}
    for c in caps:
        ents = list(c["per_R"]) + ([dict(c["partial"], partial=True)] if "partial" in c else [])
        for e in ents:
            first = e.get("first_nonce_index", c.get("first_nonce_index", 0))
            samples = [dict(s, region_va=s.get("region_va", c["region_va"])) for s in e["samples"]]
            chunks.setdefault(e["rounds"], []).append(
                (first, e, samples, {"gpu_uuid": c.get("gpu_uuid"), "first_nonce_index": first,
                                     "n_attest": e["n_attest"], "partial": bool(e.get("partial")),
                                     "clocks": e.get("clocks"), "region_va": c["region_va"],
                                     "p50_s": verifier.percentile([x / 1e9 for x in e["elapsed_ns_all"]], 50)}))
    result = {k: v for k, v in base.items() if k not in ("per_R", "partial", "first_nonce_index")}
    result["merged_from"] = [os.path.basename(p) for p in paths]
    result["per_R"] = []
    n = base["threads_total"]
    for R in sorted(chunks):
        parts = sorted(chunks[R], key=lambda t: t[0])
        el, dv, cyc, samples, sum_ok, wall = [], [], [], [], 0, 0.0
        for _, e, smp, _ in parts:
            el += [x / 1e9 for x in e["elapsed_ns_all"]]
            dv += [x / 1e9 for x in e["device_ns_all"]]
            cyc += e["cycles_all"]
            samples += smp
            sum_ok += e["sum_of_partials_ok"]
            wall += e.get("wall_s", 0.0)
        entry = summarize(R, n, el, dv, cyc, samples, sum_ok, wall, [m["clocks"] for _, _, _, m in parts])
        entry["chunks"] = [m for _, _, _, m in parts]
        result["per_R"].append(entry)
        print(json.dumps({k: v for k, v in entry.items() if k not in BIG}), flush=True)
    with open(out, "w") as f:
        json.dump(result, f, indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", default="10000,100000,1000000,10000000")
    ap.add_argument("--counts", default="1000,1000,100,20")
    ap.add_argument("--samples", type=int, default=4)
    ap.add_argument("--first", type=int, default=0, help="index of the first nonce of each stream")
    ap.add_argument("--merge", nargs="+", help="merge these captures (nonce slices) instead of running")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "c4_timing.json"))
    a = ap.parse_args()
    if a.merge:
        merge(a.merge, a.out)
    else:
        run([int(float(x)) for x in a.rounds.split(",")], [int(x) for x in a.counts.split(",")], a.samples, a.out,
            a.first)
