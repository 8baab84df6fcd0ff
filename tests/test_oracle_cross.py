"""The C oracle against the independent pure-Python oracle (oracle/ref.py), the
frozen golden vector, and order-sensitivity mutants of SCS-2.

Mutants live in this test file only: each is a copy of oracle/ref.py's round
with one plausible mistake ("strong ordering").  Each must
change the result, which shows both that the definition is order-sensitive and
that the cross-check would catch that mistake in either oracle.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import ref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "c1_checksum.json")


def test_c_oracle_equals_python_oracle_random_small():
    rng = np.random.default_rng(2209)
    for _ in range(120):
        P = int(rng.choice([1, 4, 8]))
        nc = 1 << int(rng.integers(0, 7))
        region = rng.integers(0, 256, 4 * P * nc, dtype=np.uint8)
        base = int(rng.integers(0, 2**47)) & ~0x1F
        if rng.random() < 0.2:                    # chunk addresses straddle 2^32
            base = (int(rng.integers(1, 2**15)) << 32) - 32 * int(rng.integers(0, nc + 1))
        nonce = int(rng.integers(0, 2**64, dtype=np.uint64))
        rounds = int(rng.integers(0, 40))
        nthreads = 32 * int(rng.integers(1, 3))
        want = ref.attest(nonce, region.tobytes(), base, rounds, nthreads, P)
        got = oracle.attest(nonce, region, base, rounds, 1, nthreads, P)
        assert got == want, (P, nc, base, nonce, rounds, nthreads)


def test_golden_c1():
    """Config 1 checksum frozen by scripts/make_golden.py (calls oracle/ only).
    Self-generated, not an independent fact: it guards against oracle drift."""
    with open(GOLDEN) as f:
        g = json.load(f)
    from paper_2209_03125_b200.inputs import make_region
    region = make_region(g["region_bytes"], g["fill_seed"])
    got = oracle.attest(int(g["nonce"], 16), region, int(g["base"], 16), g["rounds"], g["blocks"],
                        g["threads"], g["P"])
    assert got == int(g["checksum"], 16)
    assert ref.attest(int(g["nonce"], 16), region.tobytes(), int(g["base"], 16), 300, 32, 1) == \
        int(g["checksum_r300"], 16)


# ------------------------------------------------------------------ mutants
def _mut_round(kind):
    def one_round(A, X, r, words, nchunks, base, P):
        ts = []
        for lane in range(32):
            a = A[lane]
            X[lane] = ref.xorshift_step(X[lane])
            y = (X[lane] * ref.XS_MULT) & ref.MASK64
            C = a[15]
            i = ((y >> 32) ^ C) & (nchunks - 1)
            d = [words[P * i + q] for q in range(P)]
            if kind == "reverse_words":
                d = d[::-1]
            dp = (base + 4 * P * i) & ref.MASK64
            if kind == "drop_dp":
                dp = 0
            rr = r + 1 if kind == "round_shift" else r
            t = ((y & ref.MASK32) + rr * ref.KR + (dp & ref.MASK32) + (dp >> 32) * ref.KH) & ref.MASK32
            for q in range(P):
                t = (ref.rotl(t, 5) + d[q]) & ref.MASK32
            order = list(range(16))
            if kind == "swap_chain":
                order[6], order[7] = order[7], order[6]
            for j in order:
                a[j] = (a[j] * ((1 << ref.MULT_EXP[j]) + 1) + t) & ref.MASK32
                t = (a[j] + ref.rotl(t, ref.ROT[j])) & ref.MASK32
            if kind != "no_smc":
                t = (t + (t >> (C % 32))) & ref.MASK32
            ts.append(t)
        for lane in range(32):
            if kind == "no_exchange":
                continue
            if kind == "scs1_xor":               # the superseded SCS-1 exchange
                A[lane][15] ^= ts[(lane + 1) % 32]
                continue
            src = (lane - 1) % 32 if kind == "left_neighbour" else (lane + 1) % 32
            A[lane][15] = (A[lane][15] * ref.KX + ts[src]) & ref.MASK32
    return one_round


@pytest.mark.parametrize("kind", ["reverse_words", "drop_dp", "round_shift", "swap_chain", "no_smc",
                                  "no_exchange", "left_neighbour", "scs1_xor"])
def test_mutant_changes_result(kind, monkeypatch):
    rng = np.random.default_rng(99)
    P = 4 if kind == "reverse_words" else 1
    region = rng.integers(0, 256, 4 * P * 64, dtype=np.uint8).tobytes()
    base = 0x7F00_1234_5600
    want = oracle.attest(0x5EED, np.frombuffer(region, dtype=np.uint8), base, 20, 1, 32, P)
    assert ref.attest(0x5EED, region, base, 20, 32, P) == want
    monkeypatch.setattr(ref, "one_round", _mut_round(kind))
    assert ref.attest(0x5EED, region, base, 20, 32, P) != want
