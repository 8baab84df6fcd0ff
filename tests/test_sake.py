"""Modified SAKE (Eqs. (1)-(8)) on the host with
injected device primitives (the checksum from the CPU oracle, SHA-256 from
hashlib); tests/test_gpu_sake.py runs the device role on the GPU."""
import hashlib
import random

import mpmath
import numpy as np
import pytest

import oracle
from paper_2209_03125_b200 import sake
from paper_2209_03125_b200.inputs import make_region

REGION = make_region(1024, fill_seed=5)
BASE = 0x7F00_0000_0000


def cpu_checksum(nonce):
    return oracle.attest(nonce, REGION, BASE, 20, 1, 32)


def sha(x):
    return hashlib.sha256(x).digest()


def det_rng(seed):
    r = random.Random(seed)
    return lambda n: bytes(r.getrandbits(8) for _ in range(n))


def sessions(group=sake.TEST_GROUP, a=None, b=None, threshold=10.0, seed=1):
    v = sake.VerifierSession(group=group, expected_checksum=cpu_checksum, threshold_s=threshold,
                             rng=det_rng(seed), fixed_secret=a)
    d = sake.DeviceSession(group=group, checksum=cpu_checksum, hash=sha, rng=det_rng(seed + 1), fixed_secret=b)
    return v, d


def test_modp2048_constant_from_its_definition():
    """RFC 3526 group 14: p = 2^2048 - 2^1984 - 1 + 2^64 (floor(2^1918 pi) + 124476)."""
    mpmath.mp.prec = 2200
    p = 2**2048 - 2**1984 - 1 + 2**64 * (int(mpmath.floor(mpmath.mpf(2) ** 1918 * mpmath.pi)) + 124476)
    assert p == sake.MODP2048_P and sake.MODP2048.g == 2


RFC4493_KEY = bytes.fromhex("2b7e151628aed2a6abf7158809cf4f3c")
RFC4493_MSG = bytes.fromhex("6bc1bee22e409f96e93d7e117393172aae2d8a571e03ac9c9eb76fac45af8e51"
                            "30c81c46a35ce411e5fbc1191a0a52eff69f2445df4f9b17ad2b417be66c3710")


@pytest.mark.parametrize("mlen,tag", [(0, "bb1d6929e95937287fa37d129b756746"),
                                      (16, "070a16b46b4d4144f79bdd9dd04a287c"),
                                      (40, "dfa66747de9ae63030ca32611497c827"),
                                      (64, "51f0bebf7e3b9d92fc49741779363cfe")])
def test_rfc4493_cmac_vectors(mlen, tag):
    """S:358 / RFC 4493 section 4: AES-CMAC examples 1-4 under K = 2b7e1516..., through
    the MAC primitive sake.mac uses (empty, one block, a partial last block, four blocks)."""
    assert sake.cmac_aes128(RFC4493_KEY, RFC4493_MSG[:mlen]).hex() == tag


def test_sake_mac_key_derivation_and_check():
    """sake.mac(km, m) is AES-CMAC under SHA-256(km)[0:16]: the derived key is the
    hashlib digest prefix, the tag equals the RFC 4493 primitive's under that key, mac_ok
    accepts it and rejects any single-bit change of tag, message or key material."""
    km, m = b"session key material", RFC4493_MSG[:40]
    assert sake.mac_key(km) == hashlib.sha256(km).digest()[:16]
    tag = sake.mac(km, m)
    assert tag == sake.cmac_aes128(hashlib.sha256(km).digest()[:16], m)
    assert sake.mac_ok(km, m, tag)
    for bit in range(0, 128, 7):
        bad = bytearray(tag)
        bad[bit // 8] ^= 1 << (bit % 8)
        assert not sake.mac_ok(km, m, bytes(bad))
    assert not sake.mac_ok(km, m[:-1] + bytes([m[-1] ^ 1]), tag)
    assert not sake.mac_ok(km + b"!", m, tag)


def test_toy_group_key_agreement():
    """p=23, g=5, a=6 -> v0 = 8; b=15 -> shared key 2."""
    v, d = sessions(a=6, b=15)
    sk_v, sk_d = sake.run_protocol(v, d)
    assert int.from_bytes(v.v[0], "big") == 8
    assert sk_v == sk_d == 2


def test_modp_key_agreement_random():
    for seed in range(3):
        v, d = sessions(group=sake.MODP2048, seed=10 + seed)
        sk_v, sk_d = sake.run_protocol(v, d)
        assert sk_v == sk_d and sk_v > 1


@pytest.mark.parametrize("msg", ["v2", "w2", "mac_c_w2", "v1", "w1", "k", "mac_w2_k", "v0", "w0"])
def test_any_single_bit_tamper_aborts(msg):
    """tampering with any protocol message field yields an abort."""
    rnd = random.Random(hash(msg) & 0xFFFF)
    for _ in range(8):
        v, d = sessions(group=sake.MODP2048, seed=rnd.randrange(1 << 30))

        def tamper(name, val):
            if name != msg:
                return val
            if isinstance(val, int):
                return val ^ (1 << rnd.randrange(val.bit_length()))
            b = bytearray(val)
            b[rnd.randrange(len(b))] ^= 1 << rnd.randrange(8)
            return bytes(b)
        with pytest.raises(sake.SakeAbort):
            sake.run_protocol(v, d, tamper)


def test_timing_abort_and_state_machine():
    v, d = sessions(threshold=0.0)
    v2 = v.start()
    w2, tag = d.on_v2(v2)
    with pytest.raises(sake.AbortTiming):
        v.on_w2(w2, tag, t1=v.t0 + 1e-3)
    v, d = sessions()
    with pytest.raises(sake.AbortState):
        d.on_v1(b"\0" * 32)                   # reveal before commit
    with pytest.raises(sake.AbortState):
        v.on_w0(b"\0" * 32)


def test_mac_forgery_without_checksum_fails():
    """an adversary not knowing c cannot produce MAC_c(w2) (random tags)."""
    v, d = sessions(group=sake.MODP2048)
    v2 = v.start()
    w2, tag = d.on_v2(v2)
    rnd = random.Random(3)
    for _ in range(2000):
        forged = bytes(rnd.getrandbits(8) for _ in range(16))
        assert not sake.mac_ok(sake.c_bytes(cpu_checksum(sake.challenge_nonce(v2))), w2, forged) or forged == tag


def test_device_chain_uses_checksum():
    """w0 = H(c || r) (Eq. (3)): a device with a wrong checksum is rejected by MAC_c(w2)."""
    v = sake.VerifierSession(group=sake.TEST_GROUP, expected_checksum=cpu_checksum, threshold_s=10.0,
                             rng=det_rng(4))
    d = sake.DeviceSession(group=sake.TEST_GROUP, checksum=lambda n: cpu_checksum(n) ^ 1, hash=sha, rng=det_rng(5))
    with pytest.raises(sake.AbortMac):
        sake.run_protocol(v, d)
