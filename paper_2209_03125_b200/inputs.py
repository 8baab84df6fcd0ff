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


def kernel_text(symbol):
    """Machine code (SASS) of one checksum kernel: the .text section of `symbol` in
    the cubin the build writes next to libsage.so (compiled from the same source
    with the same flags); b'' when it has not been built."""
    path = os.path.join(_PKG, "sage_kernel.cubin")
    if not os.path.exists(path):
        return b""
    tuned = os.path.join(_PKG, "sage_kernel_tuned.cubin")
    if os.path.exists(tuned) and not os.environ.get("SAGE_NO_TUNED"):
        # the c2a kernel runs from the control-bit-tuned cubin (same instructions,
        # tuned scheduling hints): its text is the running code
        with open(tuned, "rb") as f:
            secs = _elf_sections(f.read())
        if ".text." + symbol in secs:
            with open(path, "rb") as f:
                base = _elf_sections(f.read()).get(".text." + symbol, b"")
            if secs[".text." + symbol] != base:
                return bytes(secs[".text." + symbol])
    with open(path, "rb") as f:
        secs = _elf_sections(f.read())
    return bytes(secs.get(".text." + symbol, b""))


def kernel_code_prefix(ctx, nbytes, region_va=0):
    """Region prefix for a self-verifying attestation: the machine code of the very
    kernel an attestation of nbytes (at region_va) on context ctx launches
    (ctx.kernel_symbol asks the library which instantiation it picks), so the
    checksummed region carries the running checksum function's own instructions
    (self-verification; "the beginning of the buffer contains the
    checksum function itself")."""
    return kernel_text(ctx.kernel_symbol(nbytes, region_va))


def launched_kernel_prefix(nbytes, region_va=0, device=0, **cfg):
    """kernel_code_prefix for a context of configuration cfg (sage.Context keyword
    arguments: blocks, threads, pick_words, placement), created just to ask."""
    from .sage import Context
    with Context(device=device, **cfg) as ctx:
        return kernel_code_prefix(ctx, nbytes, region_va)


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
