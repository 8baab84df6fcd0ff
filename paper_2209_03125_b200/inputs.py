"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds none of the checksum method's arithmetic: regions are filled
from numpy's PCG64 generator and nonces are drawn from a separate PCG64 stream
("input recipe").  The paper's buffer layout is "the
checksum function itself" followed by "pseudo-randomly generated values"
(P:690); the prefix here is the checksum kernel's own cubin when available.
"""
import os

import numpy as np

REGION_FILL_SEED = 0x5EED0001
NONCE_MASTER_SEED = 0x220903125
C1_NONCE = 0x0123456789ABCDEF

_PKG = os.path.dirname(os.path.abspath(__file__))


def kernel_code_prefix():
    """Bytes of the checksum kernel's cubin (written by the build next to
    libsage.so), or b'' when it has not been built.  Used as the region prefix
    so the region carries the verification code."""
    path = os.path.join(_PKG, "sage_kernel.cubin")
    if os.path.exists(path):
        with open(path, "rb") as f:
            return f.read()
    return b""


def make_region(nbytes, fill_seed=REGION_FILL_SEED, prefix=b""):
    """Region of nbytes: prefix (truncated to fit) then PCG64 pseudo-random fill."""
    rng = np.random.Generator(np.random.PCG64(fill_seed))
    buf = rng.integers(0, 256, size=nbytes, dtype=np.uint8)
    if prefix:
        n = min(len(prefix), nbytes)
        buf[:n] = np.frombuffer(prefix[:n], dtype=np.uint8)
    return buf


def nonces(count, master_seed=NONCE_MASTER_SEED):
    """count u64 nonces from a PCG64 stream (python ints)."""
    rng = np.random.Generator(np.random.PCG64(master_seed))
    return [int(v) for v in rng.integers(0, 2**64, size=count, dtype=np.uint64, endpoint=False)]


def random_geometry(rng, max_blocks=4, max_threads=128):
    """A small random launch geometry (blocks, threads) with threads % 32 == 0."""
    blocks = int(rng.integers(1, max_blocks + 1))
    threads = 32 * int(rng.integers(1, max_threads // 32 + 1))
    return blocks, threads
