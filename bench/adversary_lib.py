"""Build / load bench/libsage_adv.so, the TEST-ONLY timing-adversary library
(bench/adversary_lib.cu).  Not part of the product: only tests and bench
harnesses load it."""
import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "adversary_lib.cu")
DEPS = [SRC, os.path.join(HERE, "sage_lab.cuh")]
LIB = os.path.join(HERE, "libsage_adv.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
_lib = None


def build(force=False):
    if force or not os.path.exists(LIB) or any(os.path.getmtime(d) > os.path.getmtime(LIB) for d in DEPS):
        tmp = LIB + ".%d.tmp" % os.getpid()
        subprocess.check_call(["nvcc"] + ARCH + ["-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
                                                 "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


def load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        L.adv_count.restype = ctypes.c_int
        L.adv_name.restype = ctypes.c_char_p
        L.adv_name.argtypes = [ctypes.c_int]
        L.adv_memcopy.restype = ctypes.c_int
        L.adv_memcopy.argtypes = [ctypes.c_int]
        L.adv_probe.restype = ctypes.c_int
        L.adv_probe.argtypes = [ctypes.c_int]
        L.adv_attest.restype = ctypes.c_int
        L.adv_attest.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t,
                                 ctypes.c_uint32, ctypes.c_int64, ctypes.c_void_p,
                                 ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
        _lib = L
    return _lib


def adversaries(probes=False):
    """[(index, name, memory_copy)] of the adversary test's kernels (probes=True: the
    side experiments of scripts/memcopy_probe.py instead)."""
    L = load()
    return [(k, L.adv_name(k).decode(), bool(L.adv_memcopy(k))) for k in range(L.adv_count())
            if bool(L.adv_probe(k)) == probes]


def attest(k, nonce, region_ptr, nbytes, rounds, copy_delta=0, per_warp_ptr=None, device=0):
    """(checksum, elapsed_ns) of one attestation with adversary k."""
    cs, ns = ctypes.c_uint64(), ctypes.c_uint64()
    rc = load().adv_attest(k, device, nonce, region_ptr, nbytes, rounds, copy_delta, per_warp_ptr,
                           ctypes.byref(cs), ctypes.byref(ns))
    if rc != 0:
        raise RuntimeError("adv_attest(%d) failed: %d" % (k, rc))
    return cs.value, ns.value
