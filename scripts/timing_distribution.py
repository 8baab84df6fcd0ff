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


def run(rounds_list, counts, samples_per_r, out):
    dev = torch.device("cuda:0")
    region_np = make_region(8192, prefix=launched_kernel_prefix(8192))
    region = torch.from_numpy(region_np).to(dev)
    stream = torch.cuda.Stream()
    result = {"what": "SAGE attestation-time distribution (config 4)", "gpu": torch.cuda.get_device_name(0),
              "region_hex": region_np.tobytes().hex(), "region_va": region.data_ptr(), "P": 1, "per_R": []}
    with sage.Context(stream=stream) as ctx:
        info = ctx.query()
        n = info.blocks * info.threads
        result.update({"blocks": info.blocks, "threads": info.threads, "threads_total": n})
        pw = torch.zeros(n // 32, dtype=torch.int64, device=dev)
        for R, count in zip(rounds_list, counts):
            ns = nonces(count, master_seed=0xC4000000 + R)
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
                                    "warp_partial": int(parts[w]) & M64})
            wall_s = time.time() - t_start
            clocks = clk.stop()
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
            entry = {"rounds": R, "n_attest": len(el), "wall_s": wall_s, "clocks": clocks,
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
            result["per_R"].append(entry)
            with open(out, "w") as f:                           # after every R: a cut-off run keeps what it has
                json.dump(result, f, indent=1)
            print(json.dumps({k: v for k, v in entry.items() if k not in ("samples", "elapsed_ns_all", "device_ns_all", "cycles_all")}), flush=True)
    with open(out, "w") as f:
        json.dump(result, f, indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", default="10000,100000,1000000,10000000")
    ap.add_argument("--counts", default="1000,1000,100,20")
    ap.add_argument("--samples", type=int, default=4)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "c4_timing.json"))
    a = ap.parse_args()
    run([int(float(x)) for x in a.rounds.split(",")], [int(x) for x in a.counts.split(",")], a.samples, a.out)
