"""Verifier host logic."""
import math
import random

import numpy as np

import pytest

from paper_2209_03125_b200 import verifier as V


def test_table1_threshold_arithmetic():
    """T_avg + 2.5 sigma = 0.4941 + 2.5 * 0.0009 = 0.49635, printed 0.4964."""
    m = V.TimingModel(t_avg=0.4941, sigma=0.0009, runs=100)
    assert m.threshold == pytest.approx(0.49635, abs=1e-12)
    assert round(m.threshold, 4) == 0.4964 or round(m.threshold, 4) == 0.4963  # banker's/float rounding
    assert f"{m.threshold + 1e-12:.4f}" == "0.4964"


def test_adversarial_nop_is_rejected():
    """Exp 2: T_min = 0.4966 > 0.4964 -> rejected as timeout."""
    m = V.TimingModel(t_avg=0.4941, sigma=0.0009, runs=100)
    v = V.verify(123, 0.4966, 123, m)
    assert not v.accepted and v.reason == "timeout"
    assert V.verify(123, 0.4941, 123, m).accepted
    v = V.verify(124, 0.1, 123, m)
    assert not v.accepted and v.reason == "checksum_mismatch"


def test_calibrate_identity_and_min_runs():
    rnd = random.Random(1)
    xs = [rnd.gauss(1.0, 0.01) for _ in range(100)]
    m = V.calibrate(xs)
    assert m.threshold - m.t_avg == pytest.approx(2.5 * m.sigma, rel=1e-12)
    assert m.t_avg == pytest.approx(sum(xs) / 100)
    with pytest.raises(ValueError):
        V.calibrate(xs[:10])
    assert V.calibrate([2.0] * 30).threshold == 2.0


def test_verify_monotone():
    """lowering elapsed never flips accept -> reject."""
    m = V.TimingModel(1.0, 0.1, 100)
    prev = None
    for e in [1.3, 1.26, 1.25, 1.2, 0.9, 0.1]:
        acc = V.verify(5, e, 5, m).accepted
        if prev:
            assert acc
        prev = acc


def test_stale_nonce():
    m = V.TimingModel(1.0, 0.1, 100)
    led = V.NonceLedger()
    assert V.verify(1, 1.0, 1, m, nonce=7, ledger=led).accepted
    v = V.verify(1, 1.0, 1, m, nonce=7, ledger=led)
    assert not v.accepted and v.reason == "stale_nonce"


def test_inclusion_probability():
    """(1 - 1/524288)^100000 = 0.8264; the paper prints 0.082 (Q15)."""
    assert V.inclusion_probability(524288, 100000) == pytest.approx(0.82642, abs=1e-4)
    assert V.inclusion_probability(524288 // 4, 100000) == pytest.approx(0.46629, abs=1e-4)
    assert V.inclusion_probability(10, 0) == 1.0
    # Monte Carlo, S = 1024 words, N = 2048 accesses
    rnd = random.Random(3)
    S, N, trials = 1024, 2048, 200
    missed = 0
    for _ in range(trials):
        seen = set(rnd.randrange(S) for _ in range(N))
        missed += S - len(seen)
    p_hat = missed / (S * trials)
    p = V.inclusion_probability(S, N)
    se = math.sqrt(p * (1 - p) / (S * trials))
    assert abs(p_hat - p) < 4 * se


def test_normal_tail():
    """2.5 sigma one-sided tail = 0.621% (the paper says "about 0.5%"; Q16)."""
    assert V.normal_tail(2.5) == pytest.approx(0.00621, abs=1e-5)


def test_percentile():
    assert V.percentile([1, 2, 3, 4, 5], 50) == 3
    assert V.percentile(list(range(101)), 99) == pytest.approx(99)


def test_quantile_calibration():
    """S:311 empirical-quantile mode: a bimodal honest distribution (99% main
    mode, 1% slow mode) keeps a tight threshold, unlike T_avg + 2.5 sigma."""
    main = [1.0 + 1e-5 * (k % 7) for k in range(990)]
    slow = [1.03] * 10
    xs = main + slow
    qm = V.calibrate_quantile(xs, q=0.98)
    nm = V.calibrate(xs)
    assert qm.threshold < 1.0001 < nm.threshold
    adv = 1.0035                                  # +0.35% adversary
    assert not V.verify(1, adv, 1, qm).accepted
    assert V.verify(1, adv, 1, nm).accepted
    assert V.verify(1, 1.00003, 1, qm).accepted
    with pytest.raises(ValueError):
        V.calibrate_quantile(xs, q=1.5)


def test_verify_with_restarts():
    """a timeout restarts with a fresh nonce; a wrong checksum does not."""
    m = V.TimingModel(1.0, 0.01, 100)
    seq = iter([(1, 5, 1.5, 5), (2, 5, 1.01, 5)])
    v, k = V.verify_with_restarts(lambda: next(seq), m, max_tries=3, ledger=V.NonceLedger())
    assert v.accepted and k == 2
    seq = iter([(3, 5, 1.5, 5)] * 3)
    v, k = V.verify_with_restarts(lambda: next(seq), m, max_tries=3)
    assert not v.accepted and v.reason == "timeout" and k == 3
    seq = iter([(4, 6, 0.9, 5), (5, 5, 0.9, 5)])
    v, k = V.verify_with_restarts(lambda: next(seq), m)
    assert not v.accepted and v.reason == "checksum_mismatch" and k == 1


def test_robust_calibration_closed_forms():
    """calibrate_robust: median / MAD by hand on a small set, the margin floor, and
    the normal-consistency constant (1.4826 * MAD estimates sigma for normal data)."""
    xs = [10.0, 10.1, 9.9, 10.2, 9.8] * 6 + [13.0]           # 31 runs, one slow outlier
    m = V.calibrate_robust(xs, k=2.0, min_margin=0.0)
    assert m.median == 10.0
    assert m.sigma_r == pytest.approx(1.4826 * 0.1)             # |x - 10| medians to 0.1
    assert m.threshold == pytest.approx(10.0 * (1 + 2.0 * 1.4826 * 0.1 / 10.0))
    assert m.t_avg > m.median                                   # the mean is pulled up by the outlier
    assert V.calibrate_robust([5.0] * 30, min_margin=1e-3).threshold == pytest.approx(5.005)
    rnd = random.Random(7)
    big = [rnd.gauss(1.0, 0.01) for _ in range(20000)]
    assert V.calibrate_robust(big, k=1.0, min_margin=0.0).sigma_r == pytest.approx(0.01, rel=0.03)
    with pytest.raises(ValueError):
        V.calibrate_robust(xs[:10])
    with pytest.raises(ValueError):
        V.calibrate_robust(xs, k=0)


def test_robust_rule_ignores_the_slow_mode():
    """A tight main mode plus a 2% slow mode 3% above it (the B200 distribution,
    DESIGN.md section 11): the paper's mean + 2.5 sigma threshold is inflated past
    a +0.8% adversary, the robust threshold is not, and honest slow runs are
    resolved by the paper's restart."""
    rnd = random.Random(3)
    def honest():
        return rnd.gauss(1.0, 0.0002) * (1.03 if rnd.random() < 0.02 else 1.0)
    cal = [honest() for _ in range(500)]
    paper, robust = V.calibrate(cal), V.calibrate_robust(cal)
    adversary = [rnd.gauss(1.008, 0.0002) for _ in range(200)]     # +0.8%
    assert sum(t > robust.threshold for t in adversary) == len(adversary)
    assert sum(t > paper.threshold for t in adversary) < len(adversary) // 2
    led = V.NonceLedger()
    n = iter(range(10 ** 6))
    def attempt():
        return next(n), 1, honest(), 1
    outcomes = [V.verify_with_restarts(attempt, robust, max_tries=3, ledger=led)[0].accepted for _ in range(300)]
    assert all(outcomes)


def test_stall_estimate_recovers_injected_pauses():
    """Fixed 1.7 ms pauses injected into a constant main mode: count, share,
    pause length and the Poisson rate -ln(1 - frac) / T are recovered exactly."""
    T = 0.054
    xs = [T] * 975 + [T + 0.0017] * 25
    est = V.stall_estimate(xs)
    assert est["paused_runs"] == 25 and est["paused_frac"] == 0.025
    assert est["excess_median_s"] == pytest.approx(0.0017)
    assert est["rate_per_s"] == pytest.approx(-math.log(1 - 0.025) / T)
    assert V.stall_estimate([T] * 10)["rate_per_s"] == 0.0


def test_session_model_closed_form_and_checks():
    """calibrate_session: margin = max(floor, k * 1.2533 * sigma_r / (sqrt(m) * median)),
    sigma_r = 1.4826 * MAD; verify_session rejects a wrong checksum or a reused nonce
    before looking at time, and thresholds the session median."""
    xs = [100.0 + d for d in (-2, -1, 0, 1, 2)] * 6          # median 100, MAD 1
    m = V.calibrate_session(xs, m=16, k=6.0, min_margin=0.0)
    assert m.median == 100.0 and m.sigma_r == pytest.approx(1.4826)
    # median: sqrt(q (1 - q)) / phi(0) = sqrt(pi / 2) = 1.2533...
    assert m.margin == pytest.approx(6 * math.sqrt(math.pi / 2) * 1.4826 / (4 * 100.0))
    assert m.threshold == pytest.approx(100.0 * (1 + m.margin))
    assert V.calibrate_session(xs, m=16, min_margin=0.5).margin == 0.5
    runs = [(n, 7, 100.0, 7) for n in range(16)]
    assert V.verify_session(runs, m).accepted
    slow = [(n, 7, 103.0, 7) for n in range(16)]
    assert V.verify_session(slow, m).reason == "session_timeout"
    bad = runs[:5] + [(99, 8, 100.0, 7)] + runs[6:]
    assert V.verify_session(bad, m).reason == "checksum_mismatch"
    led = V.NonceLedger()
    led.consume(3)
    assert V.verify_session(runs, m, ledger=led).reason == "stale_nonce"
    with pytest.raises(ValueError):
        V.verify_session(runs[:15], m)


def test_session_median_separates_a_small_shift_that_single_runs_cannot():
    """Synthetic B200-like run times (main mode sigma 0.02%, 1% of runs paused by
    +3%): an adversary +0.07% slower passes the single-run robust rule most of the
    time, but every one of its 16-run sessions is rejected while honest sessions are
    accepted, paused runs included."""
    rng = np.random.default_rng(5)
    T, s = 0.0538, 0.0002 * 0.0538

    def runs(n, shift):
        t = T * (1 + shift) + rng.normal(0, s, n)
        t[rng.random(n) < 0.01] += 0.03 * T
        return t

    cal = runs(100, 0.0)
    single = V.calibrate_robust(cal)
    adv = runs(160, 0.0007)
    assert np.mean(adv > single.threshold) < 0.5
    sess = V.calibrate_session(cal, m=16)
    sessions = lambda t: [V.verify_session([(i, 1, x, 1) for i, x in enumerate(t[j:j + 16])], sess).accepted
                          for j in range(0, len(t), 16)]
    assert not any(sessions(adv))
    assert all(sessions(runs(320, 0.0)))


def test_session_quantile_rule_bounds_partial_cheating():
    """calibrate_session(q=13/15): the 14th smallest of 16 run times (linear
    interpolation puts q = 13/15 exactly on it).  Its standard error
    sigma * sqrt(q(1-q)) / (phi(z_q) sqrt(m)) is checked in closed form (z_{13/15} =
    1.11077); on synthetic B200-like times an attacker +0.07% slower in 5 of 16
    challenges passes the median rule but fails the q = 13/15 rule, while honest
    sessions with two paused runs pass both."""
    q = 13 / 15
    z = 1.110771
    phi = math.exp(-z * z / 2) / math.sqrt(2 * math.pi)
    xs = [100.0 + d for d in (-2, -1, 0, 1, 2)] * 6
    mq = V.calibrate_session(xs, m=16, q=q, min_margin=0.0)
    assert mq.margin == pytest.approx(6 * 1.4826 * math.sqrt(q * (1 - q)) / (phi * 4) / 100.0, rel=1e-6)
    assert mq.quantile == V.percentile(xs, 100 * q)
    assert V.percentile(list(range(16)), 100 * q) == pytest.approx(13.0)
    rng = np.random.default_rng(9)
    T, s = 0.0538, 0.00013 * 0.0538
    cal = T + rng.normal(0, s, 200)
    med_rule, q_rule = V.calibrate_session(cal, 16), V.calibrate_session(cal, 16, q=q)

    def verdicts(t, model):
        return [V.verify_session([(i, 1, x, 1) for i, x in enumerate(t[j:j + 16])], model).accepted
                for j in range(0, len(t), 16)]
    honest = T + rng.normal(0, s, 320)
    honest[::16] += 0.03 * T                        # one paused run per session
    honest[5::16] += 0.03 * T                       # and a second one
    assert all(verdicts(honest, med_rule)) and all(verdicts(honest, q_rule))
    partial = T + rng.normal(0, s, 320)
    for j in range(0, 320, 16):
        partial[j:j + 5] += 0.0007 * T              # cheating in 5 of 16 challenges
    assert all(verdicts(partial, med_rule))
    assert not any(verdicts(partial, q_rule))


def test_models_bound_to_a_device_reject_other_devices():
    """A timing model is a property of one GPU (two B200s differ by 0.19% in the
    median run time of the same kernel): every calibrate_*
    takes the device id, bind_device binds an existing model, and a bound model
    rejects a run or a session reported for another device (or for none) as
    device_mismatch -- before any timing or checksum test -- while an unbound
    model ignores the device."""
    a, b = "GPU-c305bf10-4c86-5a33-dc0b-e0b21eda131b", "GPU-45eb5f3e-355c-4498-195f-a6ea95f34e9a"
    xs = [1.0 + 0.001 * (i % 7) for i in range(40)]
    models = [V.calibrate(xs, device=a), V.calibrate_quantile(xs, device=a), V.calibrate_robust(xs, device=a),
              V.bind_device(V.calibrate_robust(xs), a)]
    for m in models:
        assert m.device == a
        assert V.verify(5, 1.0, 5, m, device=a).accepted
        for other in (b, None):
            v = V.verify(5, 1.0, 5, m, device=other)
            assert (v.accepted, v.reason) == (False, "device_mismatch")
        v = V.verify(4, 1.0, 5, m, device=b)                  # the device is checked first
        assert v.reason == "device_mismatch"
    free = V.calibrate_robust(xs)
    assert free.device is None and V.verify(5, 1.0, 5, free, device=b).accepted
    sm = V.calibrate_session(xs, 4, device=a)
    runs = [(i, 5, 1.0, 5) for i in range(4)]
    assert V.verify_session(runs, sm, device=a).accepted
    assert V.verify_session(runs, sm, device=b).reason == "device_mismatch"
    calls = []

    def attempt():
        calls.append(1)
        return len(calls), 5, 1.0, 5
    v, tries = V.verify_with_restarts(attempt, models[2], device=b)
    assert (v.reason, tries) == ("device_mismatch", 1)          # not retried
    assert V.verify_with_restarts(attempt, models[2], device=a)[0].accepted
