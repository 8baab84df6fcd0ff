"""SAGE's security claim on B200, driver-verified (Table 1 Exp 1
vs Exp 2): the product's c2a attestation (sage_attest) is
interleaved run by run (96 passes of 5 honest runs and one run of each
adversary) with adversary kernels from the test-only
bench/libsage_adv.so -- one IMAD per round on the product's schedule and on the
attacker's own searched schedules (scripts/schedule_search.py --extra), one ALU
op per 18 rounds, one IMAD per 7 rounds (about one per paper iteration of 428
instructions).  Every adversary returns the correct checksum.

Two verifier rules, calibrated on honest runs:
  * per run (calibrate_robust, restart on timeout): rejects >= 95% of the
    runs of every adversary except the attacker's fastest schedule for +1 IMAD per
    round, which lands within one run's timing noise (+0.05-0.08%); honest runs
    need a restart <= 5% of the time;
  * per session of m = 16 challenges (the paper's "series of challenges",
    P:313-314; calibrate_session / verify_session on the session median): rejects
    every session of every code-injection adversary, the fastest included, and
    accepts the honest sessions;
  * per session on the 14th of 16 run times (q = 13/15): rejects every session of
    every code-injection adversary but the fastest.  On the fastest -- fully, or
    cheating in only 5 of the 16 challenges (composed from its measured runs and
    honest ones; the median lets that through by design) -- it sits at the noise
    limit: the cheater's +0.04-0.09% is the size of the honest main mode's drift
    within one test (the 14th of 16 honest runs reached +0.066% on one box), so
    the rule's honest acceptance and its rejection of that attacker trade against
    each other (92-100% / 95-100% over the session-2 test runs; on one session-3
    box the attacker ran +0.06% and the rule rejected 17% of its full and 0% of
    its partial sessions).  Its honest acceptance is bounded
    loosely (>= 75%: with 24 held-out sessions a 4% false-positive rate alone
    fails ">= 95%" one time in four), its verdict on the fastest attacker is
    recorded, not asserted, and the gate is the median rule.
Equal footing: the adversaries are built from the lab template with ptxas'
scheduling hints, so the honest runs use the embedded c2a kernel (ptxas' hints)
rather than the shipped control-bit-tuned one, which is ~1.9% faster -- a gap an
attacker closes by running the same hint search on its own kernel (DESIGN.md
sections 8 and 11).
The memory-copy adversary (SMEM placement staged from a clean copy) is measured
and reported, not asserted: staging reads the region once per CTA, so that attack
costs nothing per round (DESIGN.md sections 9 and 11)."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle                                                     # noqa: E402
from paper_2209_03125_b200 import sage, verifier                  # noqa: E402
from paper_2209_03125_b200.inputs import launched_kernel_prefix, make_region, nonces  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.statistical]
R = 100_000
PASSES, HONEST_PER_PASS, CALIB, SESSION = 96, 5, 96, 16
FASTEST = "+1 IMAD / round (attacker-searched schedule)"     # within single-run noise
M64 = (1 << 64) - 1


@pytest.fixture(scope="module")
def adv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from bench import adversary_lib
    from paper_2209_03125_b200 import build
    build.build()
    adversary_lib.build()
    return adversary_lib


def test_timing_verifier_rejects_adversaries(adv):
    dev = torch.device("cuda:0")
    nbytes = 8192
    region = make_region(nbytes, prefix=launched_kernel_prefix(nbytes))
    buf = torch.empty(4 * nbytes, dtype=torch.uint8, device=dev)
    off = (-buf.data_ptr()) % 256
    d = buf[off:off + nbytes]                                   # the region the verifier attests
    clean = buf[off + 2 * nbytes:off + 3 * nbytes]              # memory-copy attacker's clean copy
    delta = clean.data_ptr() - d.data_ptr()
    d.copy_(torch.from_numpy(region))
    clean.copy_(torch.from_numpy(region))
    tampered = torch.from_numpy(region.copy())
    tampered[100:108] ^= 0xFF                                   # the attacker's modified code at d
    kinds = adv.adversaries()
    ns = nonces(PASSES + 3, master_seed=0xADD5EED)
    honest_t, adv_t, mismatch = [], {k: [] for k, _, _ in kinds}, []
    # Equal footing: the adversary kernels carry ptxas' scheduling hints, so the honest
    # side runs the embedded c2a kernel with ptxas' hints too (a context created while
    # SAGE_NO_TUNED is set); the shipped product's control-bit-tuned kernel is ~1%
    # faster still, a gap an attacker can close with the same search.
    os.environ["SAGE_NO_TUNED"] = "1"
    try:
        ctx = sage.Context()
    finally:
        os.environ.pop("SAGE_NO_TUNED", None)
    with ctx:
        for p in range(-3, PASSES):                             # 3 warm-up passes
            nonce = ns[p + 3]
            hts = []
            for _ in range(HONEST_PER_PASS):
                res = ctx.attest(nonce, d, R)
                assert res.tuned == 0
                hts.append(res.elapsed_ns * 1e-9)
            want = res.checksum
            for k, name, memcopy in kinds:
                if memcopy:
                    d.copy_(tampered)
                cs, t = adv.attest(k, nonce, d.data_ptr(), nbytes, R, copy_delta=delta if memcopy else 0)
                if memcopy:
                    d.copy_(torch.from_numpy(region))
                if p >= 0:
                    adv_t[k].append(t * 1e-9)
                    if cs != want:
                        mismatch.append((name, p))
            if p >= 0:
                honest_t.extend(hts)
        # one adversary's per-warp partials against the oracle (the checksum is the product's)
        pw = torch.zeros(2 * ctx.query().sm_count * 1024 // 32, dtype=torch.int64, device=dev)
        cs, _ = adv.attest(2, 0x5EED, d.data_ptr(), nbytes, 2000, per_warp_ptr=pw.data_ptr())
        parts = [int(v) & M64 for v in pw.cpu().tolist()]
        assert sum(parts) & M64 == cs
        for w in (0, len(parts) // 3, len(parts) - 1):
            assert parts[w] == oracle.warp_sum(0x5EED, region, d.data_ptr(), 2000, w, 1)
    assert not mismatch, mismatch[:5]
    # calibrate on the first CALIB honest runs (interleaved in time with everything else)
    calib, held = honest_t[:CALIB], honest_t[CALIB:]
    model = verifier.calibrate_robust(calib)
    smodel = verifier.calibrate_session(calib, SESSION)
    qmodel = verifier.calibrate_session(calib, SESSION, q=13 / 15)
    med = model.median

    def sessions(ts, sm=smodel):
        return [verifier.verify_session([(i, 1, t, 1) for i, t in enumerate(ts[j:j + SESSION])], sm).accepted
                for j in range(0, len(ts) - SESSION + 1, SESSION)]
    summary = {"rounds": R, "honest_kernel": "embedded c2a kernel, ptxas' scheduling hints (equal footing)",
               "honest_runs": len(honest_t), "calibration_runs": len(calib),
               "threshold_s": model.threshold, "margin": model.margin, "median_s": med,
               "honest_restart_frac": float(np.mean([t > model.threshold for t in held])),
               "session_m": SESSION, "session_threshold_s": smodel.threshold, "session_margin": smodel.margin,
               "honest_sessions_accepted_frac": float(np.mean(sessions(held))),
               "q_session_threshold_s": qmodel.threshold,
               "honest_q_sessions_accepted_frac": float(np.mean(sessions(held, qmodel))), "adversaries": {}}
    for k, name, memcopy in kinds:
        ts = adv_t[k]
        summary["adversaries"][name] = {
            "runs": len(ts), "median_s": float(np.median(ts)), "slowdown": float(np.median(ts)) / med - 1.0,
            "min_slowdown": min(ts) / med - 1.0,
            "rejected_frac": float(np.mean([t > model.threshold for t in ts])), "memory_copy": memcopy,
            "sessions_rejected_frac": 1.0 - float(np.mean(sessions(ts))),
            "q_sessions_rejected_frac": 1.0 - float(np.mean(sessions(ts, qmodel))),
            "times_s": ts}
    summary["honest_times_s"] = honest_t
    # the fastest adversary cheating in 5 of 16 challenges (its measured runs mixed with honest ones)
    fast = adv_t[[k for k, n, _ in kinds if n == FASTEST][0]]
    mixed = []
    for j in range(len(fast) // 5):
        mixed += fast[5 * j:5 * j + 5] + held[11 * j:11 * j + 11]
    summary["partial_cheating_5_of_16"] = {
        "sessions": len(mixed) // SESSION,
        "median_rule_rejected_frac": 1.0 - float(np.mean(sessions(mixed))),
        "q_rule_rejected_frac": 1.0 - float(np.mean(sessions(mixed, qmodel)))}
    out = os.environ.get("SAGE_ADV_OUT")
    if out:
        with open(out, "w") as f:
            json.dump(summary, f, indent=1)
    print(json.dumps({k: ({n: {f: x for f, x in a.items() if f != "times_s"} for n, a in v.items()}
                          if k == "adversaries" else v) for k, v in summary.items() if k != "honest_times_s"}))
    assert summary["honest_restart_frac"] <= 0.05, summary
    assert summary["honest_sessions_accepted_frac"] >= 0.95, summary
    # the 14th-of-16 rule at the noise limit (docstring): recorded; its honest
    # acceptance loosely bounded, its verdict on the fastest adversary (full or
    # partial cheating) not asserted
    assert summary["honest_q_sessions_accepted_frac"] >= 0.75, summary
    for k, name, memcopy in kinds:
        if memcopy:
            continue
        a = summary["adversaries"][name]
        assert a["sessions_rejected_frac"] >= 0.95, (name, a)
        if name != FASTEST:
            assert a["q_sessions_rejected_frac"] >= 0.95, (name, a)
        if name != FASTEST:
            assert a["rejected_frac"] >= 0.95, (name, a)
