"""Second, pure-Python oracle for SCS-2 (tiny inputs only).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  Written independently of
sage_oracle.c from the SCS-2 text in DESIGN.md section 3; used
to cross-check the C oracle on small random configurations.  Python ints with
explicit masking, one step per line in definition order.

Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.
"""

MASK32 = (1 << 32) - 1
MASK64 = (1 << 64) - 1

XS_MULT = 2685821657736338717          # S:241, written in decimal on purpose
SPLITMIX_GAMMA = 0x9E3779B97F4A7C15
MULT_EXP = (5, 11, 3, 17, 9, 23, 7, 13, 29, 2, 19, 6, 15, 27, 4, 21)   # L[j]
ROT = (7, 13, 19, 3, 25, 9, 17, 5, 11, 29, 2, 23, 14, 6, 27, 18)        # S[j]
KR, KH, KX = 0x9E3779B1, 0x85EBCA77, 0xC2B2AE3D                         # SCS-2 R6 / R9


def splitmix_mix(z):
    """SplitMix64 output function (Vigna, splitmix64.c)."""
    z &= MASK64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & MASK64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & MASK64
    z ^= z >> 31
    return z


def xorshift_step(x):
    """xorshift64 (12, 25, 27) state transition."""
    x ^= x >> 12
    x ^= (x << 25) & MASK64
    x ^= x >> 27
    return x


def rotl(v, s):
    return ((v << s) | (v >> (32 - s))) & MASK32


def seed_thread(nonce, g):
    """I1-I3: returns (a[16], x)."""
    s = splitmix_mix(nonce + (g + 1) * SPLITMIX_GAMMA)
    x = s if s != 0 else SPLITMIX_GAMMA
    a = []
    for _ in range(16):
        x = xorshift_step(x)
        a.append(((x * XS_MULT) & MASK64) >> 32)
    return a, x


def fold(a, x):
    """F1-F2."""
    e = 0
    o = 0
    for j in range(0, 16, 2):
        e ^= a[j]
    for j in range(1, 16, 2):
        o ^= a[j]
    return ((o << 32) | e) ^ x


def one_round(A, X, r, words, nchunks, base, P):
    """R1-R9 for a warp: A is a list of 32 lists of 16 ints, X a list of 32 ints."""
    ts = []
    for lane in range(32):
        a = A[lane]
        X[lane] = xorshift_step(X[lane])                 # R1
        y = (X[lane] * XS_MULT) & MASK64
        C = a[15]                                        # R2
        i = ((y >> 32) ^ C) & (nchunks - 1)              # R3
        d = [words[P * i + q] for q in range(P)]         # R4
        dp = (base + 4 * P * i) & MASK64                 # R5
        t = ((y & MASK32) + r * KR + (dp & MASK32) + (dp >> 32) * KH) & MASK32   # R6
        for q in range(P):
            t = (rotl(t, 5) + d[q]) & MASK32
        for j in range(16):                              # R7
            a[j] = (a[j] * ((1 << MULT_EXP[j]) + 1) + t) & MASK32
            t = (a[j] + rotl(t, ROT[j])) & MASK32
        t = (t + (t >> (C % 32))) & MASK32               # R8
        ts.append(t)
    for lane in range(32):                               # R9
        A[lane][15] = (A[lane][15] * KX + ts[(lane + 1) % 32]) & MASK32


def words_of(region):
    b = bytes(region)
    return [int.from_bytes(b[4 * k:4 * k + 4], "little") for k in range(len(b) // 4)]


def warp_sum(nonce, region, base, rounds, w, P=1):
    words = words_of(region)
    nchunks = len(words) // P
    A, X = [], []
    for lane in range(32):
        a, x = seed_thread(nonce, 32 * w + lane)
        A.append(a)
        X.append(x)
    for r in range(rounds):
        one_round(A, X, r, words, nchunks, base, P)
    return sum(fold(A[lane], X[lane]) for lane in range(32)) & MASK64


def attest(nonce, region, base, rounds, n_threads, P=1):
    assert n_threads % 32 == 0
    total = 0
    for w in range(n_threads // 32):
        total += warp_sum(nonce, region, base, rounds, w, P)
    return total & MASK64
