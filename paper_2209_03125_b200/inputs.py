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


def _elf_sections(blob):
    """{name: bytes} of an ELF64 little-endian file (plain header parsing)."""
    import struct
    if blob[:4] != b"\x7fELF" or blob[4] != 2:
        return {}
    shoff, = struct.unpack_from("<Q", blob, 0x28)
    shentsize, shnum, shstrndx = struct.unpack_from("<HHH", blob, 0x3A)
    hdrs = []
    for k in range(shnum):
        name, _typ, _flags, _addr, off, size = struct.unpack_from("<IIQQQQ", blob, shoff + k * shentsize)
        hdrs.append((name, off, size))
    _, stroff, strsize = hdrs[shstrndx]
    strtab = blob[stroff:stroff + strsize]
    out = {}
    for name, off, size in hdrs:
        end = strtab.find(b"\0", name)
        out[strtab[name:end].decode("latin-1")] = blob[off:off + size]
    return out


def kernel_code_prefix(pick_words=1, smem=True):
    """Machine code (SASS) of the checksum kernel variant itself, taken from the
    .text section of the cubin the build writes next to libsage.so; b'' when it
    has not been built.  Used as the region prefix so the checksummed region
    carries the checksum function's own instructions (self-verification,
    P:370-381; buffer layout P:365-367)."""
    path = os.path.join(_PKG, "sage_kernel.cubin")
    if not os.path.exists(path):
        return b""
    with open(path, "rb") as f:
        secs = _elf_sections(f.read())
    want = ".text._ZN4sage20sage_checksum_kernelILi%dELb%d" % (pick_words, 1 if smem else 0)
    for name, data in sorted(secs.items()):
        if name.startswith(want):
            return bytes(data)
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
