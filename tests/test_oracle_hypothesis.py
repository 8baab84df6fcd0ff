"""Property-based cross-check of the two oracles at the level of one round from
arbitrary injected warp states (hypothesis): the C oracle's warp_rounds and the
pure-Python ref.one_round must agree on every accumulator and PRNG state, for
any state, round index, base address and region."""
import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle
from oracle import ref

u32 = st.integers(min_value=0, max_value=2**32 - 1)
u64nz = st.integers(min_value=1, max_value=2**64 - 1)


@settings(max_examples=60, deadline=None)
@given(st.lists(st.lists(u32, min_size=16, max_size=16), min_size=32, max_size=32),
       st.lists(u64nz, min_size=32, max_size=32),
       st.integers(min_value=0, max_value=2**32 - 2),      # round index (r_end = r + 1 < 2^32)
       st.integers(min_value=0, max_value=2**15 - 1),
       st.sampled_from([1, 4, 8]),
       st.integers(min_value=0, max_value=6),
       st.integers(min_value=0, max_value=2**31))
def test_one_round_c_equals_python(A, X, r, base_hi, P, log_nc, seed):
    nc = 1 << log_nc
    region = np.random.default_rng(seed).integers(0, 256, 4 * P * nc, dtype=np.uint8)
    base = (base_hi << 32) | (seed * 32 & 0xFFFFFFE0)
    A_c, X_c = oracle.warp_rounds(np.array(A, dtype=np.uint32), np.array(X, dtype=np.uint64), region, base, r,
                                  r + 1, P)
    A_p = [list(a) for a in A]
    X_p = list(X)
    ref.one_round(A_p, X_p, r, ref.words_of(region.tobytes()), nc, base, P)
    assert [[int(v) for v in row] for row in A_c] == A_p
    assert [int(v) for v in X_c] == X_p
