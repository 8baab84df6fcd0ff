"""Modified SAKE key establishment around the attestation (SAGE section 5.2.3,
Eqs. (1)-(8)).

    V: a <-R; v0 = g^a mod p; v1 = H(v0); v2 = H(v1)          (1)
    [t0] V -> D: v2                                             (2)
    D: c = checksum(challenge v2); r <-R;
       w0 = H(c || r); w1 = H(w0); w2 = H(w1)                   (3)
    [t1] D -> V: w2, MAC_c(w2)                                  (4)
    D: b <-R; k = g^b mod p                                     (5)
    V -> D: v1      D -> V: w1, k, MAC_w2(k)                    (6)
    V -> D: v0      D -> V: w0                                  (7)
    sk_VD = k^a = v0^b mod p                                    (8)

H = SHA-256, MAC = AES-CMAC.  Readings:
- the checksum challenge is the first 8 bytes of v2 (little-endian u64 nonce);
- c enters H and the MAC key as its 8 little-endian bytes; MAC keys are
  SHA-256(key material)[0:16];
- the verifier checks t1 - t0 against its timing model, w-chain
  consistency, then each MAC;
- default group: RFC 3526 2048-bit MODP group 14, g = 2.

Device role on the GPU: the checksum runs through sage_attest and the hash
chain w0..w2 through sage_kernel_hash (the SHA-256 kernel); the AES-CMAC and
the modular exponentiations run on the host (not data-parallel).
The verifier role is host code (the paper's SGX enclave).
"""
import hashlib
import os
import time
from dataclasses import dataclass, field

from cryptography.hazmat.primitives import cmac
from cryptography.hazmat.primitives.ciphers import algorithms

# RFC 3526 group 14: p = 2^2048 - 2^1984 - 1 + 2^64 * (floor(2^1918 pi) + 124476), g = 2
MODP2048_P = int(
    "FFFFFFFFFFFFFFFFC90FDAA22168C234C4C6628B80DC1CD129024E088A67CC74020BBEA63B139B22514A08798E3404DD"
    "EF9519B3CD3A431B302B0A6DF25F14374FE1356D6D51C245E485B576625E7EC6F44C42E9A637ED6B0BFF5CB6F406B7ED"
    "EE386BFB5A899FA5AE9F24117C4B1FE649286651ECE45B3DC2007CB8A163BF0598DA48361C55D39A69163FA8FD24CF5F"
    "83655D23DCA3AD961C62F356208552BB9ED529077096966D670C354E4ABC9804F1746C08CA18217C32905E462E36CE3B"
    "E39E772C180E86039B2783A2EC07A28FB5C55DF06F4C52C9DE2BCBF6955817183995497CEA956AE515D2261898FA0510"
    "15728E5A8AACAA68FFFFFFFFFFFFFFFF", 16)


@dataclass(frozen=True)
class DhGroup:
    p: int
    g: int
    nbits: int


MODP2048 = DhGroup(MODP2048_P, 2, 256)
TEST_GROUP = DhGroup(23, 5, 4)


class SakeAbort(Exception):
    pass


class AbortTiming(SakeAbort):
    pass


class AbortChainMismatch(SakeAbort):
    pass


class AbortMac(SakeAbort):
    pass


class AbortState(SakeAbort):
    pass


def H(x):
    return hashlib.sha256(x).digest()


def mac_key(key_material):
    """The 128-bit AES-CMAC key derived from key material: SHA-256(key_material)[0:16]."""
    return hashlib.sha256(key_material).digest()[:16]


def cmac_aes128(key16, msg):
    """AES-CMAC (RFC 4493) under a 16-byte key."""
    c = cmac.CMAC(algorithms.AES(bytes(key16)))
    c.update(msg)
    return c.finalize()


def mac(key_material, msg):
    """MAC of SAKE: AES-CMAC under mac_key(key_material)."""
    return cmac_aes128(mac_key(key_material), msg)


def mac_ok(key_material, msg, tag):
    """Constant-time check of a tag produced by mac()."""
    c = cmac.CMAC(algorithms.AES(mac_key(key_material)))
    c.update(msg)
    try:
        c.verify(tag)
        return True
    except Exception:
        return False


def int_bytes(x, group):
    return x.to_bytes((group.p.bit_length() + 7) // 8, "big")


def _random_exponent(rng, group):
    """Secret exponent in [1, p-2] from nbits/8 + 8 random bytes (bias < 2^-64)."""
    return int.from_bytes(rng(group.nbits // 8 + 8), "big") % (group.p - 2) + 1


def challenge_nonce(v2):
    """The checksum challenge derived from v2: its first 8 bytes, little-endian."""
    return int.from_bytes(v2[:8], "little")


def c_bytes(c):
    return int(c).to_bytes(8, "little")


@dataclass
class VerifierSession:
    """Verifier role (host enclave in the paper).  expected_checksum(nonce) ->
    the expected c for the device's attestation (precomputed by the verifier,
    P:313-314); threshold_s: accepted t1 - t0 (verifier.TimingModel.threshold
    plus protocol slack)."""
    group: DhGroup
    expected_checksum: object
    threshold_s: float
    rng: object = os.urandom
    fixed_secret: int = None          # tests only: use this a instead of a random one
    state: str = "init"
    a: int = 0
    v: list = field(default_factory=list)
    t0: float = 0.0
    w2: bytes = b""
    w1: bytes = b""
    k: int = 0
    key: int = None

    def start(self):
        if self.state != "init":
            raise AbortState("start twice")
        self.a = self.fixed_secret or _random_exponent(self.rng, self.group)
        v0 = int_bytes(pow(self.group.g, self.a, self.group.p), self.group)
        v1 = H(v0)
        v2 = H(v1)
        self.v = [v0, v1, v2]
        self.state = "sent_v2"
        self.t0 = time.monotonic()
        return v2

    def on_w2(self, w2, tag, t1=None):
        if self.state != "sent_v2":
            raise AbortState("w2 out of order")
        t1 = time.monotonic() if t1 is None else t1
        if t1 - self.t0 > self.threshold_s:
            raise AbortTiming("t1 - t0 = %.6f s > %.6f s" % (t1 - self.t0, self.threshold_s))
        c = self.expected_checksum(challenge_nonce(self.v[2]))
        if not mac_ok(c_bytes(c), w2, tag):
            raise AbortMac("MAC_c(w2)")
        self.w2 = w2
        self.state = "got_w2"
        return self.v[1]

    def on_w1k(self, w1, k, tag):
        if self.state != "got_w2":
            raise AbortState("w1 out of order")
        if H(w1) != self.w2:
            raise AbortChainMismatch("H(w1) != w2")
        if not mac_ok(self.w2, int_bytes(k, self.group), tag):
            raise AbortMac("MAC_w2(k)")
        if not 1 < k < self.group.p - 1:
            raise AbortChainMismatch("k out of range")
        self.w1, self.k = w1, k
        self.state = "got_w1"
        return self.v[0]

    def on_w0(self, w0):
        if self.state != "got_w1":
            raise AbortState("w0 out of order")
        if H(w0) != self.w1:
            raise AbortChainMismatch("H(w0) != w1")
        self.key = pow(self.k, self.a, self.group.p)
        self.state = "done"
        return self.key


@dataclass
class DeviceSession:
    """Device role.  checksum(nonce) -> c runs the attestation (the GPU kernel
    via sage_attest); hash(bytes) -> 32 bytes is SHA-256 (the GPU kernel via
    sage_kernel_hash).  Use `gpu_device_session` for the GPU-backed default."""
    group: DhGroup
    checksum: object
    hash: object
    rng: object = os.urandom
    fixed_secret: int = None          # tests only: use this b instead of a random one
    state: str = "init"
    w: list = field(default_factory=list)
    v2: bytes = b""
    v1: bytes = b""
    b: int = 0
    key: int = None

    def on_v2(self, v2):
        if self.state != "init":
            raise AbortState("v2 twice")
        c = self.checksum(challenge_nonce(v2))
        r = self.rng(32)
        w0 = self.hash(c_bytes(c) + r)
        w1 = self.hash(w0)
        w2 = self.hash(w1)
        self.w = [w0, w1, w2]
        self.v2 = v2
        self.state = "sent_w2"
        tag = mac(c_bytes(c), w2)
        self.b = self.fixed_secret or _random_exponent(self.rng, self.group)
        return w2, tag

    def on_v1(self, v1):
        if self.state != "sent_w2":
            raise AbortState("v1 out of order")
        if self.hash(v1) != self.v2:
            raise AbortChainMismatch("H(v1) != v2")
        self.v1 = v1
        k = pow(self.group.g, self.b, self.group.p)
        self.state = "sent_w1"
        return self.w[1], k, mac(self.w[2], int_bytes(k, self.group))

    def on_v0(self, v0):
        if self.state != "sent_w1":
            raise AbortState("v0 out of order")
        if self.hash(v0) != self.v1:
            raise AbortChainMismatch("H(v0) != v1")
        self.key = pow(int.from_bytes(v0, "big"), self.b, self.group.p)
        self.state = "done"
        return self.w[0]


def run_protocol(verifier, device, tamper=None):
    """Run Eqs. (2)-(8) over an in-process channel.  tamper(msg_name, value) ->
    value lets tests modify any message.  Returns (sk_V, sk_D)."""
    t = tamper or (lambda name, v: v)
    v2 = t("v2", verifier.start())
    w2, tag = device.on_v2(v2)
    w2, tag = t("w2", w2), t("mac_c_w2", tag)
    v1 = t("v1", verifier.on_w2(w2, tag))
    w1, k, tag2 = device.on_v1(v1)
    w1, k, tag2 = t("w1", w1), t("k", k), t("mac_w2_k", tag2)
    v0 = t("v0", verifier.on_w1k(w1, k, tag2))
    w0 = t("w0", device.on_v0(v0))
    sk_v = verifier.on_w0(w0)
    return sk_v, device.key


def gpu_device_session(ctx, region, rounds, group=MODP2048, rng=os.urandom):
    """Device role backed by the GPU: the checksum is sage_attest on `region`
    (device tensor) and the hash chain is sage_kernel_hash."""
    from . import sage

    def checksum(nonce):
        return ctx.attest(nonce, region, rounds).checksum

    def gpu_hash(msg):
        if len(msg) <= 128:                      # short messages travel as r (kernel parameters)
            h, _ = sage.kernel_hash(ctx.ctx, msg, None)
        else:                                    # e.g. v0 (256 bytes): stage it in device memory
            import torch
            buf = torch.frombuffer(bytearray(msg), dtype=torch.uint8).to(region.device)
            h, _ = sage.kernel_hash(ctx.ctx, b"", buf)
        return h

    return DeviceSession(group=group, checksum=checksum, hash=gpu_hash, rng=rng)
