"""CPU oracle for SCS-2 (the SAGE checksum loop, arXiv 2209.03125).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py
(its cpu_baseline leg and --impl reference arm) may import this package.  The
product package paper_2209_03125_b200 never imports it, and the two share no
code: the C oracle (sage_oracle.c) and the pure-Python oracle (ref.py) are
written from the SCS-2 text in DESIGN.md section 3.

Parity status: every SCS-2 step is pinned by tests/test_oracle_pins.py (see
DESIGN.md section 4 for the pin per step); none is "parity unpinned".
"""
import ctypes
import os
import subprocess
from concurrent.futures import ProcessPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sage_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "sha256_oracle.c")]
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force=False):
    """Compile sage_oracle.c with gcc -O2 (plain scalar, no -march)."""
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(s) for s in _SRCS):
        tmp = _LIB + ".%d.tmp" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-o", tmp] + _SRCS)
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u64, u32, p = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p
        L.sage_oracle_splitmix_mix.restype = u64
        L.sage_oracle_splitmix_mix.argtypes = [u64]
        L.sage_oracle_xs.restype = u64
        L.sage_oracle_xs.argtypes = [u64]
        L.sage_oracle_thread_init.restype = None
        L.sage_oracle_thread_init.argtypes = [u64, u64, p, p]
        L.sage_oracle_fold.restype = u64
        L.sage_oracle_fold.argtypes = [p, u64]
        L.sage_oracle_warp_rounds.restype = ctypes.c_int
        L.sage_oracle_warp_rounds.argtypes = [p, p, p, u64, u64, u64, u64, ctypes.c_uint]
        L.sage_oracle_warp.restype = ctypes.c_int
        L.sage_oracle_warp.argtypes = [u64, p, u64, u64, u64, u64, ctypes.c_uint, p]
        L.sage_oracle_sha256.restype = None
        L.sage_oracle_sha256.argtypes = [p, u64, p, u64, p]
        L.sage_oracle_attest.restype = ctypes.c_int
        L.sage_oracle_attest.argtypes = [u64, p, u64, u64, u64, u64, u64, ctypes.c_uint, p]
        L.sage_oracle_attest_counts.restype = ctypes.c_int
        L.sage_oracle_attest_counts.argtypes = [u64, p, u64, u64, u64, u64, u64, ctypes.c_uint, p, p]
        _lib = L
    return _lib


def _buf(region):
    arr = np.ascontiguousarray(np.frombuffer(bytes(region), dtype=np.uint8) if not isinstance(region, np.ndarray)
                               else region.view(np.uint8).reshape(-1))
    return arr, arr.ctypes.data_as(ctypes.c_void_p), arr.nbytes


def splitmix_mix(z):
    return lib().sage_oracle_splitmix_mix(z & (2**64 - 1))


def xs(x):
    return lib().sage_oracle_xs(x & (2**64 - 1))


def thread_init(nonce, g):
    a = np.zeros(16, dtype=np.uint32)
    x = ctypes.c_uint64(0)
    lib().sage_oracle_thread_init(nonce, g, a.ctypes.data_as(ctypes.c_void_p), ctypes.byref(x))
    return [int(v) for v in a], x.value


def fold(a, x):
    arr = np.asarray(a, dtype=np.uint32)
    return lib().sage_oracle_fold(arr.ctypes.data_as(ctypes.c_void_p), x)


def warp_rounds(A, X, region, base, r_begin, r_end, P=1):
    """Run rounds [r_begin, r_end) on an explicit warp state. A: (32,16) u32, X: (32,) u64.
    Returns new (A, X) arrays."""
    A = np.array(A, dtype=np.uint32).reshape(32, 16).copy()
    X = np.array(X, dtype=np.uint64).reshape(32).copy()
    arr, ptr, n = _buf(region)
    rc = lib().sage_oracle_warp_rounds(A.ctypes.data_as(ctypes.c_void_p), X.ctypes.data_as(ctypes.c_void_p),
                                       ptr, n, base, r_begin, r_end, P)
    if rc != 0:
        raise ValueError("oracle rejected arguments")
    return A, X


def warp_sum(nonce, region, base, rounds, w, P=1):
    arr, ptr, n = _buf(region)
    out = ctypes.c_uint64(0)
    rc = lib().sage_oracle_warp(nonce, ptr, n, base, rounds, w, P, ctypes.byref(out))
    if rc != 0:
        raise ValueError("oracle rejected arguments")
    return out.value


def attest(nonce, region, base, rounds, blocks, threads, P=1):
    arr, ptr, n = _buf(region)
    out = ctypes.c_uint64(0)
    rc = lib().sage_oracle_attest(nonce, ptr, n, base, rounds, blocks, threads, P, ctypes.byref(out))
    if rc != 0:
        raise ValueError("oracle rejected arguments")
    return out.value


def attest_counts(nonce, region, base, rounds, blocks, threads, P=1):
    """(checksum, per-chunk pick counts as a uint32 array) -- the inclusion
    experiment counted by the oracle."""
    arr, ptr, n = _buf(region)
    counts = np.zeros(n // (4 * P), dtype=np.uint32)
    out = ctypes.c_uint64(0)
    rc = lib().sage_oracle_attest_counts(nonce, ptr, n, base, rounds, blocks, threads, P, ctypes.byref(out),
                                         counts.ctypes.data_as(ctypes.c_void_p))
    if rc != 0:
        raise ValueError("oracle rejected arguments")
    return out.value, counts


def sha256(r, code):
    """SHA-256(r || code) (SAGE Eq. (9)) from the plain C oracle; r, code bytes-like
    or uint8 ndarrays."""
    def as_u8(b):
        return np.ascontiguousarray(b.view(np.uint8).reshape(-1) if isinstance(b, np.ndarray)
                                    else np.frombuffer(bytes(b), dtype=np.uint8))
    rb, cb = as_u8(r), as_u8(code)
    out = np.zeros(32, dtype=np.uint8)
    lib().sage_oracle_sha256(rb.ctypes.data_as(ctypes.c_void_p), rb.nbytes, cb.ctypes.data_as(ctypes.c_void_p),
                             cb.nbytes, out.ctypes.data_as(ctypes.c_void_p))
    return out.tobytes()


# ---- multi-process driver for large configs (one warp range per task) ----------
# Workers are spawned (not forked: the caller may hold CUDA / torch threads) and
# attach to the region through POSIX shared memory instead of pickling it.
_pool_region = None
_pool_shm = None


def _pool_init(shm_name, nbytes):
    global _pool_region, _pool_shm
    from multiprocessing import shared_memory
    _pool_shm = shared_memory.SharedMemory(name=shm_name)
    _pool_region = np.ndarray((nbytes,), dtype=np.uint8, buffer=_pool_shm.buf)


def _pool_task(args):
    nonce, base, rounds, w0, w1, P = args
    return [warp_sum(nonce, _pool_region, base, rounds, w, P) for w in range(w0, w1)]


class WarpPool:
    """A pool of spawned oracle workers sharing one region (POSIX shared memory);
    reuse it across calls so timings do not include process start-up.

        with WarpPool(region) as pool:
            sums = pool.warp_sums(nonce, base, rounds, warps, P)
    """

    def __init__(self, region, workers=None):
        import multiprocessing as mp
        from multiprocessing import shared_memory
        src = np.ascontiguousarray(region).view(np.uint8).reshape(-1) if isinstance(region, np.ndarray) else \
            np.frombuffer(bytes(region), dtype=np.uint8)
        build()
        self.workers = workers or len(os.sched_getaffinity(0))
        self.shm = shared_memory.SharedMemory(create=True, size=max(1, src.nbytes))
        np.ndarray((src.nbytes,), dtype=np.uint8, buffer=self.shm.buf)[:] = src
        self.ex = ProcessPoolExecutor(max_workers=self.workers, mp_context=mp.get_context("spawn"),
                                      initializer=_pool_init, initargs=(self.shm.name, src.nbytes))
        list(self.ex.map(_pool_noop, range(self.workers)))          # start every worker now

    def warp_sums(self, nonce, base, rounds, warps, P=1):
        warps = list(warps)
        tasks = [(nonce, base, rounds, w, w + 1, P) for w in warps]
        res = list(self.ex.map(_pool_task, tasks, chunksize=max(1, len(tasks) // (4 * self.workers))))
        return {w: r[0] for w, r in zip(warps, res)}

    def close(self):
        self.ex.shutdown()
        self.shm.close()
        self.shm.unlink()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def _pool_noop(_):
    return os.getpid()


def warp_sums_parallel(nonce, region, base, rounds, warps, P=1, workers=None):
    """Oracle warp partials for the listed warp indices, spread over host cores.
    The per-warp function is unchanged; this only fans warps out."""
    with WarpPool(region, workers) as pool:
        return pool.warp_sums(nonce, base, rounds, warps, P)
