"""Pins for the SHA-256 oracle (oracle/sha256_oracle.c) used by the kernel-hash
row h = H(r || code) (SAGE Eq. (9)): FIPS 180-4 / NIST example
vectors, the SPEC example, and padding-boundary lengths against
hashlib (a library SHA-256, as an independent implementation)."""
import hashlib

import numpy as np

import oracle


def H(r, code=b""):
    return oracle.sha256(r, code).hex()


def test_fips_vectors():
    assert H(b"abc") == "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
    assert H(b"") == "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"
    assert H(b"abcdbcdecdefdefgefghfghighijhijkijkljklmklmnlmnomnopnopq") == \
        "248d6a61d20638b8e5c026930c3e6039a33ce45964ff2167f6ecedd419db06c1"
    assert H(b"a" * 1_000_000) == "cdc76e5c9914fb9281a1c7e284d73e67f1809a48a497200e046d39ccc7112cd0"


def test_spec_example_and_concatenation():
    """r = 32 zero bytes, empty code -> 66687aad...2925; the split between
    r and code does not matter (it is one message r || code)."""
    assert H(bytes(32)) == "66687aadf862bd776c8fc18b8e9f8e20089714856ee233b3902a591d0d5f2925"
    msg = bytes(range(200))
    for k in (0, 1, 31, 32, 55, 56, 63, 64, 65, 199, 200):
        assert H(msg[:k], msg[k:]) == H(msg)


def test_padding_boundaries_against_hashlib():
    rng = np.random.default_rng(1)
    for n in list(range(0, 130)) + [447, 448, 511, 512, 4095, 4096, 65537]:
        m = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert H(m[: n // 3], m[n // 3:]) == hashlib.sha256(m).hexdigest(), n
