"""Pins for the CPU oracle (oracle/sage_oracle.c) against facts fixed outside it.

Each test states what it pins and where the fact comes from.  Expected values
are published constants, hand-derived values for degenerate inputs, algebraic
invariants of SCS-2, statistics the paper's design fixes,
or brute force on tiny inputs -- never the oracle's own output.  P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
import numpy as np
import pytest

import oracle

M32 = (1 << 32) - 1
M64 = (1 << 64) - 1
XS_MULT_DEC = 2685821657736338717          # S:241 as printed (decimal)
GAMMA = 0x9E3779B97F4A7C15
L_TAB = (5, 11, 3, 17, 9, 23, 7, 13, 29, 2, 19, 6, 15, 27, 4, 21)
S_TAB = (7, 13, 19, 3, 25, 9, 17, 5, 11, 29, 2, 23, 14, 6, 27, 18)
KR, KH, KX = 0x9E3779B1, 0x85EBCA77, 0xC2B2AE3D      # SCS-2 R6/R9 constants


def rotl(v, s):
    return ((v << s) | (v >> (32 - s))) & M32


# ---------------------------------------------------------------- I1 SplitMix64
def test_splitmix64_published_outputs():
    """Pins I1's mixer and increment: the first outputs of SplitMix64 seeded with 0
    are 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F (Vigna,
    splitmix64.c reference outputs; SURVEY 8(c) pin table)."""
    published = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    for k, want in enumerate(published, start=1):
        assert oracle.splitmix_mix((k * GAMMA) & M64) == want


def test_seed_uses_g_plus_one_th_output():
    """I1: thread g with nonce 0 starts from SplitMix64 output #(g+1); thread 0's
    first accumulator is the high half of xs(0xE220A8397B1DCDAF) times M64."""
    a, _ = oracle.thread_init(0, 0)
    x1 = oracle.xs(0xE220A8397B1DCDAF)
    assert a[0] == ((x1 * XS_MULT_DEC) & M64) >> 32
    a1, _ = oracle.thread_init(0, 1)
    assert a1[0] == ((oracle.xs(0x6E789E6AA1B965F4) * XS_MULT_DEC) & M64) >> 32


def test_seed_distinct_for_distinct_threads():
    """SplitMix64's finaliser is a bijection, so distinct g give distinct seeds
    (exhaustive over a small range through the public init)."""
    xs_seen = {oracle.thread_init(0xABCDEF, g)[1] for g in range(4096)}
    assert len(xs_seen) == 4096


# ---------------------------------------------------------------- R1 xorshift64*
def test_xorshift_hand_values():
    """Pins the shift triple and directions (>>12, <<25, >>27) with values
    worked by hand: xs(1) = 2^25+1; xs(2^63) = 2^63+2^51+2^36+2^24;
    xs(2^40) = 2^53+2^40+2^28+2^26+2^13+2^1."""
    assert oracle.xs(1) == (1 << 25) | 1
    assert oracle.xs(1 << 63) == (1 << 63) | (1 << 51) | (1 << 36) | (1 << 24)
    assert oracle.xs(1 << 40) == (1 << 53) | (1 << 40) | (1 << 28) | (1 << 26) | (1 << 13) | (1 << 1)


def _gf2_matrix():
    # column k = xs(e_k); xs is linear over GF(2)
    M = np.zeros((64, 64), dtype=np.uint8)
    for k in range(64):
        v = oracle.xs(1 << k)
        for b in range(64):
            M[b, k] = (v >> b) & 1
    return M


def _gf2_pow(M, e):
    R = np.eye(64, dtype=np.int64)
    B = M.astype(np.int64)
    while e:
        if e & 1:
            R = (R @ B) % 2
        B = (B @ B) % 2
        e >>= 1
    return R


def test_xorshift_full_period():
    """xorshift64 with (12,25,27) has period 2^64-1 (Marsaglia 2003; Vigna 2016):
    its GF(2) transition matrix has multiplicative order exactly 2^64-1."""
    factors = [3, 5, 17, 257, 641, 65537, 6700417]
    assert np.prod([np.uint64(f) for f in factors], dtype=object) == (1 << 64) - 1
    M = _gf2_matrix()
    I = np.eye(64, dtype=np.int64)
    assert np.array_equal(_gf2_pow(M, (1 << 64) - 1), I)
    for p in factors:
        assert not np.array_equal(_gf2_pow(M, ((1 << 64) - 1) // p), I)


# ------------------------------------------------- one injected round (R1-R9)
def _zero_state():
    return np.zeros((32, 16), dtype=np.uint32), np.ones(32, dtype=np.uint64)


def test_round_reveals_prng_output():
    """R1 + R6 + R7[0] on a degenerate state: a = 0, x = 1, one-chunk zero region,
    base 0, r 0.  Then xs(1) = 0x2000001, i = 0, dp = 0, t = rotl(lo32(y), 5) and
    a[0]' = 0*MUL + t.  Pins y = xs(x) * M64 and its low half feeding t."""
    A, X = _zero_state()
    region = np.zeros(4, dtype=np.uint8)
    A2, X2 = oracle.warp_rounds(A, X, region, 0, 0, 1, P=1)
    y = (0x2000001 * XS_MULT_DEC) & M64
    assert int(X2[0]) == 0x2000001
    assert int(A2[5, 0]) == rotl(y & M32, 5)


def test_round_index_and_data_pointer_fold():
    """R5-R6: t = lo32(y) + r*KR + lo32(dp) + hi32(dp)*KH then
    rotl(t,5) + d.  Degenerate state a = 0 so a[0]' = t; one chunk so dp = base."""
    A, X = _zero_state()
    word = 0xDEADBEEF
    region = np.frombuffer(word.to_bytes(4, "little"), dtype=np.uint8)
    base = 0x0000_7F12_3456_7890 & ~0xF
    r = 12345
    A2, _ = oracle.warp_rounds(A, X, region, base, r, r + 1, P=1)
    y = (0x2000001 * XS_MULT_DEC) & M64
    t = ((y & M32) + r * KR + (base & M32) + (base >> 32) * KH) & M32
    assert int(A2[0, 0]) == (rotl(t, 5) + word) & M32
    # each of the three terms is a bijective summand: moving r by one moves t by KR
    A3, _ = oracle.warp_rounds(A, X, region, base, r + 1, r + 2, P=1)
    t2 = ((y & M32) + (r + 1) * KR + (base & M32) + (base >> 32) * KH) & M32
    assert int(A3[0, 0]) == (rotl(t2, 5) + word) & M32


def test_pick_index_formula():
    """R3 (Q1/Q2): i = (hi32(y) ^ C) & (Nc-1).  Region word k holds k,
    base 0, so with a = 0 except a[15] = C: a[0]' = rotl(lo32(y) + 4i, 5) + i."""
    nc = 1024
    region = np.arange(nc, dtype=np.uint32).view(np.uint8)
    for C in (0, 0x2A, 0xFFFFFFFF, 0x12345678):
        A, X = _zero_state()
        A[:, 15] = C
        A2, _ = oracle.warp_rounds(A, X, region, 0, 0, 1, P=1)
        y = (0x2000001 * XS_MULT_DEC) & M64
        i = ((y >> 32) ^ C) & (nc - 1)
        t = ((y & M32) + 4 * i) & M32
        assert int(A2[0, 0]) == (rotl(t, 5) + i) & M32


def test_multi_word_pick_order():
    """R4/R6 with P = 4 and 8: the P words of a chunk are folded in ascending
    address order, t = rotl(t,5) + d[q] (Q19)."""
    for P in (4, 8):
        words = [0x11111111 * (q + 1) & M32 for q in range(P)]
        region = np.array(words, dtype=np.uint32).view(np.uint8)
        A, X = _zero_state()
        A2, _ = oracle.warp_rounds(A, X, region, 0, 0, 1, P=P)
        y = (0x2000001 * XS_MULT_DEC) & M64
        t = y & M32
        for q in range(P):
            t = (rotl(t, 5) + words[q]) & M32
        assert int(A2[0, 0]) == t


def test_chain_multipliers_and_order():
    """R7: a[j] <- a[j]*(2^L[j]+1) + t with t independent of the
    old a[j], so raising a[j] by delta raises a[j]' by exactly MUL[j]*delta and
    leaves a[0..j-1]' unchanged, while every later accumulator changes
    (strong ordering)."""
    rng = np.random.default_rng(7)
    region = rng.integers(0, 256, 256, dtype=np.uint8)
    A0 = rng.integers(0, 2**32, (32, 16), dtype=np.uint64).astype(np.uint32)
    X0 = rng.integers(1, 2**63, 32, dtype=np.uint64)
    A0[:, 15] = 0   # keep C fixed (0) so the pick index does not move
    ref, _ = oracle.warp_rounds(A0, X0, region, 0, 0, 1, P=1)
    for j in range(15):
        for delta in (1, 0x80000000, 0x12345):
            A = A0.copy()
            A[3, j] = (int(A[3, j]) + delta) & M32
            out, _ = oracle.warp_rounds(A, X0, region, 0, 0, 1, P=1)
            mul = (1 << L_TAB[j]) + 1
            assert (int(out[3, j]) - int(ref[3, j])) & M32 == (mul * delta) & M32
            assert np.array_equal(out[3, :j], ref[3, :j])
            assert all(out[3, k] != ref[3, k] for k in range(j + 1, 15))


def test_chain_rotations_on_zero_state():
    """R7 rotate-add amounts S[j]: with a = 0 the chain reduces to
    a[j]' = t_j, t_{j+1} = t_j + rotl(t_j, S[j]); R8 with C = 0 doubles t;
    R9 gives a[15]' = t_15*KX + (neighbour's final t).  All lanes share x, so all
    lanes have the same t and a[15]' = t_15*KX + 2*t_16."""
    A, X = _zero_state()
    region = np.zeros(4, dtype=np.uint8)
    A2, _ = oracle.warp_rounds(A, X, region, 0, 0, 1, P=1)
    y = (0x2000001 * XS_MULT_DEC) & M64
    t = rotl(y & M32, 5)
    expect = []
    for j in range(16):
        expect.append(t)
        t = (t + rotl(t, S_TAB[j])) & M32
    final_t = (t + t) & M32            # R8, N = 0
    expect[15] = (expect[15] * KX + final_t) & M32      # R9
    assert [int(v) for v in A2[0]] == expect


def test_self_modify_shift_examples():
    """R8: N = C mod 32, so C = 0 -> N = 0, C = 0x2A -> N = 10.
    Lane 1 carries C; lane 0 receives lane 1's t, so lane 0's a[15] exposes it."""
    region = np.zeros(4, dtype=np.uint8)
    for C, N in ((0, 0), (0x2A, 10), (0xFFFFFFE0, 0), (31, 31)):
        A, X = _zero_state()
        A[1, 15] = C
        A2, _ = oracle.warp_rounds(A, X, region, 0, 0, 1, P=1)
        # lane 1's chain with a = 0 except a[15] = C
        y = (0x2000001 * XS_MULT_DEC) & M64
        t = rotl(y & M32, 5)
        for j in range(15):
            t = (t + rotl(t, S_TAB[j])) & M32
        a15 = (C * ((1 << L_TAB[15]) + 1) + t) & M32
        t = (a15 + rotl(t, S_TAB[15])) & M32
        t1 = (t + (t >> N)) & M32
        # lane 0 (C = 0) has a[15]' = its own t_15 * KX + t1
        t0 = rotl(y & M32, 5)
        for j in range(15):
            t0 = (t0 + rotl(t0, S_TAB[j])) & M32
        assert int(A2[0, 15]) == (t0 * KX + t1) & M32


def test_neighbour_exchange_direction():
    """R9 (north_star, Q13): lane l folds lane (l+1) mod 32's t into a[15] only
    (SCS-2: a[15] <- a[15]*KX + t_{l+1}).
    Perturbing lane k changes lane k's state and only a[15] of lane k-1."""
    rng = np.random.default_rng(3)
    region = rng.integers(0, 256, 1024, dtype=np.uint8)
    A0 = rng.integers(0, 2**32, (32, 16), dtype=np.uint64).astype(np.uint32)
    X0 = rng.integers(1, 2**63, 32, dtype=np.uint64)
    ref, refx = oracle.warp_rounds(A0, X0, region, 0x1000, 5, 6, P=1)
    for k in (0, 1, 17, 31):
        A = A0.copy()
        A[k, 4] ^= 1
        out, outx = oracle.warp_rounds(A, X0, region, 0x1000, 5, 6, P=1)
        src = (k - 1) % 32
        for lane in range(32):
            if lane == k:
                assert not np.array_equal(out[lane, 4:], ref[lane, 4:])
            elif lane == src:
                assert np.array_equal(out[lane, :15], ref[lane, :15])
                assert out[lane, 15] != ref[lane, 15]
            else:
                assert np.array_equal(out[lane], ref[lane])
        assert np.array_equal(outx, refx)


# ---------------------------------------------------------------- F1-F2 fold
def test_fold_hand_example():
    """F1-F2: e = XOR of even accumulators, o = XOR of odd ones,
    f = (o << 32 | e) ^ x.  With a[j] = 2^j: e = 0x5555, o = 0xAAAA."""
    a = [1 << j for j in range(16)]
    assert oracle.fold(a, 0) == (0xAAAA << 32) | 0x5555
    assert oracle.fold(a, M64) == ((0xAAAA << 32) | 0x5555) ^ M64
    assert oracle.fold([0] * 16, 0x0123456789ABCDEF) == 0x0123456789ABCDEF


# ---------------------------------------------------------------- sum / epilog
def test_zero_rounds_closed_form_and_geometry():
    """R = 0: checksum = sum over g of F(I1-I3(nonce, g)) mod 2^64;
    it depends on the thread count only, not on how it is split into blocks
    (tree sum = flat modular sum)."""
    region = np.zeros(64, dtype=np.uint8)
    nonce = 0xFEEDFACECAFEBEEF
    flat = 0
    for g in range(256):
        a, x = oracle.thread_init(nonce, g)
        flat += oracle.fold(a, x)
    flat &= M64
    assert flat != sum(oracle.fold(*oracle.thread_init(nonce, g)) for g in range(256))  # it wrapped
    for blocks, threads in ((1, 256), (2, 128), (8, 32)):
        assert oracle.attest(nonce, region, 0, 0, blocks, threads) == flat


# ------------------------------------------------------ brute force, tiny inputs
def test_every_bit_of_small_region_is_covered():
    """Self-verification: flipping any single bit of a 64-word
    region changes the checksum.  32 threads x 64 rounds = 2048 picks over
    64 words, so each word is read with probability 1 - e^-32."""
    rng = np.random.default_rng(11)
    region = rng.integers(0, 256, 256, dtype=np.uint8)
    base = 0x7F00_0000_0000
    ref = oracle.attest(0x1111, region, base, 64, 1, 32)
    for bit in range(256 * 8):
        r2 = region.copy()
        r2[bit // 8] ^= 1 << (bit % 8)
        assert oracle.attest(0x1111, r2, base, 64, 1, 32) != ref, bit


def test_inputs_each_change_result():
    """Challenge dependence, DP binding, round count and
    geometry all enter the result."""
    rng = np.random.default_rng(5)
    region = rng.integers(0, 256, 4096, dtype=np.uint8)
    base = 0x7F00_0000_1000
    ref = oracle.attest(42, region, base, 100, 1, 32)
    assert oracle.attest(43, region, base, 100, 1, 32) != ref
    assert oracle.attest(42, region, base + 16, 100, 1, 32) != ref
    assert oracle.attest(42, region, base, 101, 1, 32) != ref
    assert oracle.attest(42, region, base, 100, 1, 64) != ref
    assert oracle.attest(42, region, base, 100, 1, 32, P=4) != ref


def test_challenge_collisions():
    """Distinct challenges give distinct checksums: 2000 nonces, tiny config."""
    region = np.arange(64, dtype=np.uint32).view(np.uint8)
    seen = {oracle.attest(n, region, 0, 4, 1, 32) for n in range(2000)}
    assert len(seen) == 2000


def test_argument_rejection():
    """Q1: non-power-of-two chunk counts, misaligned base, unknown P, R >= 2^32."""
    region = np.zeros(4096, dtype=np.uint8)
    with pytest.raises(ValueError):
        oracle.attest(0, region[:12], 0, 1, 1, 32)
    with pytest.raises(ValueError):
        oracle.attest(0, region, 8, 1, 1, 32)
    with pytest.raises(ValueError):
        oracle.attest(0, region, 0, 1, 1, 32, P=2)
    with pytest.raises(ValueError):
        oracle.attest(0, region, 0, 1 << 32, 1, 32)
    with pytest.raises(ValueError):
        oracle.attest(0, region, 16, 1, 1, 32, P=8)   # P=8 needs 32-B alignment


def test_address_formula_identity():
    """Q1 (P:646 vs S:240): for W = data_size/4 words, (4C) mod (4W) = 4 (C mod W),
    and for W a power of two C mod W = C & (W-1)."""
    rng = np.random.default_rng(0)
    for _ in range(1000):
        C = int(rng.integers(0, 2**32))
        W = 1 << int(rng.integers(0, 20))
        assert (4 * C) % (4 * W) == 4 * (C % W) == 4 * (C & (W - 1))


def test_nonce_is_added_to_the_splitmix_counter():
    """I1 adds the nonce to the counter (g+1)*G: nonce = G makes thread 0 start
    from SplitMix64 output #2 of seed 0, 0x6E789E6AA1B965F4 (published); an XOR
    would give sm(0) instead."""
    a, _ = oracle.thread_init(GAMMA, 0)
    assert a[0] == ((oracle.xs(0x6E789E6AA1B965F4) * XS_MULT_DEC) & M64) >> 32


def test_zero_seed_maps_to_gamma():
    """I2: the only zero SplitMix64 output is sm(0) = 0 (the finaliser fixes 0),
    reached for nonce = -(g+1)*G; the xorshift state then starts at G."""
    assert oracle.splitmix_mix(0) == 0
    nonce = (-GAMMA) & M64                      # thread g = 0
    a, x = oracle.thread_init(nonce, 0)
    xs = GAMMA
    for j in range(16):
        xs = oracle.xs(xs)
        assert a[j] == ((xs * XS_MULT_DEC) & M64) >> 32
    assert x == xs


def test_all_sixteen_seed_words():
    """I3: a[j] = hi32(x_j * M64) for the j-th xorshift state after the seed."""
    a, x = oracle.thread_init(0, 5)            # thread 5: SplitMix64 output #6 of seed 0
    s = oracle.splitmix_mix((6 * GAMMA) & M64)
    for j in range(16):
        s = oracle.xs(s)
        assert a[j] == ((s * XS_MULT_DEC) & M64) >> 32
    assert x == s


def test_data_pointer_scales_with_pick_words():
    """R5: dp = base + 4*P*i.  Region chunk k holds word value k in every word;
    a = 0 except a[15] = C fixes i, base 0: a[0]' = R6 fold of t0 = lo32(y) + 4*P*i."""
    for P in (4, 8):
        nc = 64
        words = np.repeat(np.arange(nc, dtype=np.uint32), P)
        region = words.view(np.uint8)
        for C in (0, 0x1234567, 0xFFFFFFFF):
            A, X = _zero_state()
            A[:, 15] = C
            A2, _ = oracle.warp_rounds(A, X, region, 0, 0, 1, P=P)
            y = (0x2000001 * XS_MULT_DEC) & M64
            i = ((y >> 32) ^ C) & (nc - 1)
            t = ((y & M32) + 4 * P * i) & M32
            for _ in range(P):
                t = (rotl(t, 5) + i) & M32
            assert int(A2[0, 0]) == t, (P, C)


# ------------------------------------------- R4-R7 injectivity, exhaustive at R = 1
def _picks_by_formula(A, X, nc):
    """R1-R3 written out independently: lane l's chunk index for one round."""
    out = []
    for lane in range(32):
        x = int(X[lane])
        x ^= x >> 12
        x ^= (x << 25) & M64
        x ^= x >> 27
        y = (x * XS_MULT_DEC) & M64
        out.append(((y >> 32) ^ int(A[lane, 15])) & (nc - 1))
    return out


@pytest.mark.parametrize("P", [1, 4, 8])
def test_single_round_injectivity_exhaustive(P):
    """SURVEY 8(c) R6-R7 pin, exhaustive over a 64-word region at R = 1: for a fixed
    pre-round state and pick, t after R6 is a bijection of each loaded word (rotl
    then add), and a[0] <- a[0]*MUL[0] + t a bijection of t.  So for EVERY one of
    the 64 x 32 single-bit flips of the region, a[0] changes in exactly the lanes
    whose pick contained the flipped word -- deterministically, after one round --
    and in no other lane; every other lane keeps its whole state except a[15] of
    the lane to the left of a picking lane (R9 takes its neighbour's t).  The
    picking lanes come from R1-R3 retyped here, and every lane must pick exactly
    one chunk (the flips reaching it all lie in one P-word chunk)."""
    rng = np.random.default_rng(100 + P)
    nwords = 64
    nc = nwords // P
    region = rng.integers(0, 256, 4 * nwords, dtype=np.uint8)
    base = 0x7F3A_0000_2000
    A0 = rng.integers(0, 2**32, (32, 16), dtype=np.uint64).astype(np.uint32)
    X0 = rng.integers(1, 2**64 - 1, 32, dtype=np.uint64)
    r = 77
    ref, refx = oracle.warp_rounds(A0, X0, region, base, r, r + 1, P=P)
    picks = _picks_by_formula(A0, X0, nc)
    reached = {lane: set() for lane in range(32)}
    for bit in range(32 * nwords):
        k = bit // 32
        reg = region.copy()
        reg[4 * k + (bit % 32) // 8] ^= 1 << (bit % 8)
        out, outx = oracle.warp_rounds(A0, X0, reg, base, r, r + 1, P=P)
        assert np.array_equal(outx, refx)
        pickers = {lane for lane in range(32) if picks[lane] == k // P}
        changed = {lane for lane in range(32) if out[lane, 0] != ref[lane, 0]}
        assert changed == pickers, (bit, sorted(changed), sorted(pickers))
        left = {(lane - 1) % 32 for lane in pickers}
        for lane in range(32):
            if lane in pickers:
                reached[lane].add(k // P)
            elif lane in left:
                assert np.array_equal(out[lane, :15], ref[lane, :15]) and out[lane, 15] != ref[lane, 15]
            else:
                assert np.array_equal(out[lane], ref[lane])
    assert all(len(v) == 1 for v in reached.values())


# --------------------------------------------------- R8 shift amount uniformity
def test_self_modify_shift_amount_is_uniform():
    """S:228-230 (R8): N = C mod 32 with C the round-start a[15] is uniform over
    0..31: chi-square over 10^5 (lane, round) samples of a seeded warp, 31 degrees of
    freedom, below the 0.1% critical value 61.1; every value of N occurs."""
    rng = np.random.default_rng(8)
    region = rng.integers(0, 256, 4096, dtype=np.uint8)
    A, X = [], []
    for lane in range(32):
        a, x = oracle.thread_init(0x5EED, lane)
        A.append(a)
        X.append(x)
    A = np.array(A, dtype=np.uint32)
    X = np.array(X, dtype=np.uint64)
    counts = np.zeros(32, dtype=np.int64)
    rounds = 100_000 // 32 + 1
    for r in range(rounds):
        counts += np.bincount(A[:, 15] & 31, minlength=32)
        A, X = oracle.warp_rounds(A, X, region, 0x10000, r, r + 1, P=1)
    n = counts.sum()
    assert n >= 100_000
    chi2 = float((((counts - n / 32) ** 2) / (n / 32)).sum())
    assert chi2 < 61.1 and counts.min() > 0, (chi2, counts)


# ------------------------------- SCS-2's odd multipliers KR, KH, KX are permutations
class _FastRound:
    """One-round oracle calls with preallocated ctypes buffers (2^20 of them per test)."""

    def __init__(self, region):
        import ctypes
        self.ct = ctypes
        self.L = oracle.lib()
        self.region = np.ascontiguousarray(region, dtype=np.uint8)
        self.A = np.zeros((32, 16), dtype=np.uint32)
        self.X = np.zeros(32, dtype=np.uint64)
        self.pa = self.A.ctypes.data_as(ctypes.c_void_p)
        self.px = self.X.ctypes.data_as(ctypes.c_void_p)
        self.pr = self.region.ctypes.data_as(ctypes.c_void_p)

    def __call__(self, A0, X0, base, r):
        self.A[:] = A0
        self.X[:] = X0
        rc = self.L.sage_oracle_warp_rounds(self.pa, self.px, self.pr, self.region.nbytes, base, r, r + 1, 1)
        assert rc == 0
        return self.A


def _rotr(v, s):
    return ((v >> s) | (v << (32 - s))) & M32


def test_odd_multipliers_are_permutations_of_z_2_32():
    """KR, KH, KX (and MUL[15] = 2^21 + 1) are odd, hence units of Z/2^32: v -> v*K mod 2^32
    is a permutation.  Exhaustive on 2^20 inputs: the images are distinct, and the
    modular inverse K^-1 (K * K^-1 = 1 mod 2^32) maps every image back to its input."""
    v = np.arange(1 << 20, dtype=np.uint64)
    for K in (KR, KH, KX, (1 << L_TAB[15]) + 1):
        assert K % 2 == 1
        Kinv = pow(K, -1, 1 << 32)
        assert (K * Kinv) & M32 == 1
        img = (v * np.uint64(K)) & np.uint64(M32)
        assert np.unique(img).size == v.size
        assert np.array_equal((img * np.uint64(Kinv)) & np.uint64(M32), v)


def test_round_index_enters_as_a_permutation():
    """R6 (Q10): the round index enters t as r*KR.  On a degenerate warp
    (a = 0, one-chunk region, so a[0]' = rotl(t, 5) + w) the difference
    rotr(a[0]'(r) - w, 5) - rotr(a[0]'(0) - w, 5) decoded with KR^-1 returns r for
    every r < 2^20: the oracle's r -> a[0]' map is injective, exactly r*KR + const."""
    w = 0x6A09E667
    region = np.frombuffer(w.to_bytes(4, "little"), dtype=np.uint8)
    run = _FastRound(region)
    A0, X0 = _zero_state()
    Kinv = pow(KR, -1, 1 << 32)
    t0 = _rotr((int(run(A0, X0, 0, 0)[0, 0]) - w) & M32, 5)
    for r in range(1, 1 << 20):
        t = _rotr((int(run(A0, X0, 0, r)[0, 0]) - w) & M32, 5)
        assert ((t - t0) * Kinv) & M32 == r, r


def test_data_pointer_high_word_enters_as_a_permutation():
    """R5-R6 (Q9): hi32(dp) enters t as hi32(dp)*KH.  With base = h << 32
    (one chunk, so dp = base) the difference against h = 0 decoded with KH^-1 returns h
    for every h < 2^20."""
    w = 0xBB67AE85
    region = np.frombuffer(w.to_bytes(4, "little"), dtype=np.uint8)
    run = _FastRound(region)
    A0, X0 = _zero_state()
    Kinv = pow(KH, -1, 1 << 32)
    t0 = _rotr((int(run(A0, X0, 0, 5)[0, 0]) - w) & M32, 5)
    for h in range(1, 1 << 20):
        t = _rotr((int(run(A0, X0, h << 32, 5)[0, 0]) - w) & M32, 5)
        assert ((t - t0) * Kinv) & M32 == h, h


def test_exchange_multiplier_is_a_permutation():
    """R7[15] + R9 (Q13): lane 0's a[15]' = (a[15]*MUL[15] + t_15)*KX + t_{lane 1}, and
    lane 1 does not depend on lane 0, so changing lane 0's a[15] by v changes its
    a[15]' by v*MUL[15]*KX.  With a one-chunk region (the pick cannot move) the
    difference decoded with (MUL[15]*KX)^-1 returns v for every v < 2^20 (all 32-bit
    residues of the form covered: the map is a permutation)."""
    rng = np.random.default_rng(15)
    region = rng.integers(0, 256, 4, dtype=np.uint8)
    run = _FastRound(region)
    A0 = rng.integers(0, 2**32, (32, 16), dtype=np.uint64).astype(np.uint32)
    X0 = rng.integers(1, 2**63, 32, dtype=np.uint64)
    A0[0, 15] = 0
    Kinv = pow(((1 << L_TAB[15]) + 1) * KX, -1, 1 << 32)
    ref = int(run(A0, X0, 0x4000, 9)[0, 15])
    A = A0.copy()
    for v in range(1, 1 << 20):
        A[0, 15] = v
        out = int(run(A, X0, 0x4000, 9)[0, 15])
        assert ((out - ref) * Kinv) & M32 == v, v


# ------------------------------------------------ R3 read-count instrumentation
def test_pick_counts_config1_read_every_word():
    """SURVEY 8(c) R3 pin: at config 1 (1 x 32 threads, 1,024 words, 10^4 rounds =
    3.2 x 10^5 picks) every word is read -- under uniform picks each word is missed
    with probability (1 - 1/1024)^320000 ~ e^-312.5 -- the counts add up to the
    number of picks, and instrumenting does not change the checksum."""
    region = np.random.default_rng(1).integers(0, 256, 4096, dtype=np.uint8)
    cs, counts = oracle.attest_counts(0x0123456789ABCDEF, region, 0x7F00_0000_0000, 10_000, 1, 32, 1)
    assert cs == oracle.attest(0x0123456789ABCDEF, region, 0x7F00_0000_0000, 10_000, 1, 32, 1)
    assert int(counts.sum()) == 32 * 10_000 and int(counts.min()) > 0
    # uniform picks: each count is Binomial(N, 1/1024); chi-square over the 1,024 words
    e = 32 * 10_000 / 1024
    chi2 = float(((counts - e) ** 2 / e).sum())
    assert chi2 < 1023 + 6 * (2 * 1023) ** 0.5, chi2


def test_pick_counts_follow_the_inclusion_formula():
    """P:747-749 with the formula of S:302: N = 100,000 picks over S = 131,072 words
    leave a fraction (1 - 1/S)^N = 0.4663 unread (within 6 standard errors)."""
    S, rounds = 131072, 3125
    region = np.random.default_rng(2).integers(0, 256, 4 * S, dtype=np.uint8)
    _, counts = oracle.attest_counts(77, region, 0x10000, rounds, 1, 32, 1)
    N = 32 * rounds
    p = (1 - 1 / S) ** N
    unread = float((counts == 0).mean())
    assert abs(p - 0.46629) < 1e-4
    assert abs(unread - p) < 6 * (p * (1 - p) / S) ** 0.5, (unread, p)
