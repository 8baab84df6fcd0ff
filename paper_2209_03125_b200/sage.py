"""ctypes binding for libsage.so (include/sage.h).  Argument marshalling only:
every step of the checksum runs in the CUDA kernel behind the C ABI.

The functions keep the C names without the `sage_` prefix (sage_attest ->
attest).  There is no CPU fallback: if libsage.so is missing or cannot be
loaded, every call raises.
"""
import ctypes
import os

from .build import LIB

SAGE_OK = 0
SAGE_EINVAL = -1
SAGE_EUNSUPPORTED = -2
SAGE_ENOMEM = -3
SAGE_ECUDA = -4

SAGE_AUTO, SAGE_SMEM, SAGE_GLOBAL, SAGE_HYBRID = 0, 1, 2, 3
PLACEMENT_NAMES = {SAGE_SMEM: "smem", SAGE_GLOBAL: "global", SAGE_AUTO: "auto", SAGE_HYBRID: "hybrid"}

# every symbol include/sage.h declares
EXPORTS = ("sage_checksum_init", "sage_attest", "sage_attest_debug", "sage_attest_async", "sage_decode_raw",
           "sage_attest_host", "sage_attest_coverage", "sage_kernel_hash", "sage_host_region_va",
           "sage_placement_for", "sage_kernel_symbol", "sage_device_uuid", "sage_query", "sage_launch_count", "sage_stream",
           "sage_checksum_destroy", "sage_strerror", "sage_last_error")


class SageError(RuntimeError):
    def __init__(self, code, detail):
        self.code = code
        super().__init__("%s (%d): %s" % (_strerror(code), code, detail))


class sage_config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("blocks", ctypes.c_uint32), ("threads", ctypes.c_uint32),
                ("pick_words", ctypes.c_uint32), ("placement", ctypes.c_uint32), ("stream", ctypes.c_void_p)]


class sage_result(ctypes.Structure):
    _fields_ = [("checksum", ctypes.c_uint64), ("cycles", ctypes.c_uint64), ("elapsed_ns", ctypes.c_uint64),
                ("device_ns", ctypes.c_uint64), ("region_va", ctypes.c_uint64), ("placement", ctypes.c_uint32),
                ("blocks", ctypes.c_uint32), ("threads", ctypes.c_uint32), ("pick_words", ctypes.c_uint32),
                ("ilp", ctypes.c_uint32), ("tuned", ctypes.c_uint32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class sage_info(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("sm_count", ctypes.c_uint32), ("blocks", ctypes.c_uint32),
                ("threads", ctypes.c_uint32), ("pick_words", ctypes.c_uint32), ("placement", ctypes.c_uint32),
                ("ctas_per_sm_smem", ctypes.c_uint32), ("ctas_per_sm_global", ctypes.c_uint32),
                ("regs_per_thread", ctypes.c_uint32), ("smem_region_max", ctypes.c_uint64),
                ("ilp_smem", ctypes.c_uint32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def load(path=LIB):
    """Load libsage.so and declare the signatures. Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError("libsage.so not built (%s); run `python -m paper_2209_03125_b200.build`" % path)
    L = ctypes.CDLL(path)
    p, u64, sz, i = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_int
    L.sage_checksum_init.argtypes = [ctypes.POINTER(sage_config), ctypes.POINTER(p)]
    L.sage_attest.argtypes = [p, u64, p, sz, u64, ctypes.POINTER(sage_result)]
    L.sage_attest_debug.argtypes = [p, u64, p, sz, u64, p, ctypes.POINTER(sage_result)]
    L.sage_attest_async.argtypes = [p, u64, p, sz, u64, p, p]
    L.sage_decode_raw.argtypes = [p, ctypes.POINTER(sage_result)]
    L.sage_attest_coverage.argtypes = [p, u64, p, sz, u64, p, ctypes.POINTER(sage_result)]
    L.sage_kernel_hash.argtypes = [p, p, sz, p, sz, p, ctypes.POINTER(u64)]
    L.sage_attest_host.argtypes = [p, u64, p, sz, u64, ctypes.POINTER(sage_result)]
    L.sage_host_region_va.argtypes = [p, sz, ctypes.POINTER(u64)]
    L.sage_placement_for.argtypes = [p, sz, ctypes.POINTER(ctypes.c_uint32)]
    L.sage_kernel_symbol.argtypes = [p, u64, sz, ctypes.c_char_p, sz]
    L.sage_device_uuid.argtypes = [p, ctypes.POINTER(ctypes.c_uint8 * 16)]
    L.sage_query.argtypes = [p, ctypes.POINTER(sage_info)]
    L.sage_launch_count.argtypes = [p]
    L.sage_launch_count.restype = u64
    L.sage_stream.argtypes = [p]
    L.sage_stream.restype = p
    L.sage_checksum_destroy.argtypes = [p]
    L.sage_checksum_destroy.restype = None
    L.sage_strerror.argtypes = [i]
    L.sage_strerror.restype = ctypes.c_char_p
    L.sage_last_error.argtypes = []
    L.sage_last_error.restype = ctypes.c_char_p
    for name in ("sage_checksum_init", "sage_attest", "sage_attest_debug", "sage_attest_async", "sage_decode_raw",
                 "sage_attest_coverage", "sage_kernel_hash", "sage_attest_host", "sage_host_region_va",
                 "sage_placement_for", "sage_kernel_symbol", "sage_device_uuid", "sage_query"):
        getattr(L, name).restype = i
    _lib = L
    return L


def _strerror(code):
    return load().sage_strerror(code).decode()


def _check(rc):
    if rc != SAGE_OK:
        raise SageError(rc, load().sage_last_error().decode())


def _ptr(buf):
    """Device/host address of a torch tensor, numpy array or int."""
    if buf is None:
        return None
    if isinstance(buf, int):
        return buf
    if hasattr(buf, "data_ptr"):
        return buf.data_ptr()
    if hasattr(buf, "ctypes"):
        return buf.ctypes.data
    raise TypeError("expected a tensor, ndarray or address, got %r" % type(buf))


def _nbytes(buf, nbytes):
    if nbytes is not None:
        return int(nbytes)
    if hasattr(buf, "nbytes"):
        return int(buf.nbytes)
    if hasattr(buf, "element_size"):
        return int(buf.numel() * buf.element_size())
    raise TypeError("region size unknown; pass nbytes")


# ---- the C entry points, one Python function each -------------------------------------
def _stream_handle(stream):
    """cudaStream_t from a torch.cuda.Stream, an int handle or None (ctx-owned).
    Handle 0 (torch's legacy default stream) is refused: the library would read
    it as NULL and launch on its own stream, unordered with the caller's work."""
    if stream is None:
        return None
    h = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    if h == 0:
        raise ValueError("pass a non-default stream (e.g. torch.cuda.Stream()); handle 0 means ctx-owned")
    return h


def checksum_init(device=0, blocks=0, threads=0, pick_words=1, placement=SAGE_AUTO, stream=None):
    cfg = sage_config(device, blocks, threads, pick_words, placement, _stream_handle(stream))
    ctx = ctypes.c_void_p()
    _check(load().sage_checksum_init(ctypes.byref(cfg), ctypes.byref(ctx)))
    return ctx


def attest(ctx, nonce, region, rounds, nbytes=None):
    out = sage_result()
    _check(load().sage_attest(ctx, nonce, _ptr(region), _nbytes(region, nbytes), rounds, ctypes.byref(out)))
    return out


def attest_debug(ctx, nonce, region, rounds, per_warp_out, nbytes=None):
    out = sage_result()
    _check(load().sage_attest_debug(ctx, nonce, _ptr(region), _nbytes(region, nbytes), rounds, _ptr(per_warp_out),
                                    ctypes.byref(out)))
    return out


def attest_async(ctx, nonce, region, rounds, raw_out, per_warp_out=None, nbytes=None):
    _check(load().sage_attest_async(ctx, nonce, _ptr(region), _nbytes(region, nbytes), rounds, _ptr(raw_out),
                                    _ptr(per_warp_out)))


def attest_coverage(ctx, nonce, region, rounds, counts_out, nbytes=None):
    out = sage_result()
    _check(load().sage_attest_coverage(ctx, nonce, _ptr(region), _nbytes(region, nbytes), rounds, _ptr(counts_out),
                                       ctypes.byref(out)))
    return out


def kernel_hash(ctx, r, code, nbytes=None):
    """h = SHA-256(r || code) on the GPU (SAGE Eq. (9)); r: host bytes (<= 128),
    code: device tensor / address.  Returns (digest bytes, elapsed_ns)."""
    rb = bytes(r)
    rbuf = ctypes.create_string_buffer(rb, len(rb)) if rb else None
    out = ctypes.create_string_buffer(32)
    ns = ctypes.c_uint64()
    n = _nbytes(code, nbytes) if code is not None else 0
    _check(load().sage_kernel_hash(ctx, rbuf, len(rb), _ptr(code) if n else None, n, out, ctypes.byref(ns)))
    return out.raw, ns.value


def decode_raw(raw4):
    """raw4: host sequence of 4 u64 (e.g. raw_out.cpu())."""
    arr = (ctypes.c_uint64 * 4)(*[int(v) & (2**64 - 1) for v in raw4])
    out = sage_result()
    _check(load().sage_decode_raw(arr, ctypes.byref(out)))
    return out


def attest_host(ctx, nonce, host_region, rounds, nbytes=None):
    out = sage_result()
    _check(load().sage_attest_host(ctx, nonce, _ptr(host_region), _nbytes(host_region, nbytes), rounds,
                                   ctypes.byref(out)))
    return out


def host_region_va(ctx, nbytes):
    va = ctypes.c_uint64()
    _check(load().sage_host_region_va(ctx, nbytes, ctypes.byref(va)))
    return va.value


def placement_for(ctx, nbytes):
    pl = ctypes.c_uint32()
    _check(load().sage_placement_for(ctx, nbytes, ctypes.byref(pl)))
    return pl.value


def kernel_symbol(ctx, nbytes, region_va=0):
    """Mangled name of the checksum kernel an attestation of nbytes at region_va
    (0: a region not straddling a 4 GiB boundary) would launch."""
    buf = ctypes.create_string_buffer(512)
    _check(load().sage_kernel_symbol(ctx, int(region_va), int(nbytes), buf, len(buf)))
    return buf.value.decode()


def device_uuid(ctx):
    """The attested GPU's UUID, formatted as nvidia-smi prints it (GPU-8-4-4-4-12 hex)."""
    raw = (ctypes.c_uint8 * 16)()
    _check(load().sage_device_uuid(ctx, ctypes.byref(raw)))
    h = bytes(raw).hex()
    return "GPU-%s-%s-%s-%s-%s" % (h[:8], h[8:12], h[12:16], h[16:20], h[20:])


def query(ctx):
    info = sage_info()
    _check(load().sage_query(ctx, ctypes.byref(info)))
    return info


def launch_count(ctx):
    return load().sage_launch_count(ctx)


def stream(ctx):
    return load().sage_stream(ctx)


def checksum_destroy(ctx):
    load().sage_checksum_destroy(ctx)


def strerror(code):
    return _strerror(code)


def last_error():
    return load().sage_last_error().decode()


class Context:
    """Owns a sage_ctx; thin convenience wrapper over the functions above."""

    def __init__(self, device=0, blocks=0, threads=0, pick_words=1, placement=SAGE_AUTO, stream=None):
        self.ctx = checksum_init(device, blocks, threads, pick_words, placement, stream)
        self.pick_words = pick_words

    def attest(self, nonce, region, rounds, nbytes=None):
        return attest(self.ctx, nonce, region, rounds, nbytes)

    def attest_debug(self, nonce, region, rounds, per_warp_out, nbytes=None):
        return attest_debug(self.ctx, nonce, region, rounds, per_warp_out, nbytes)

    def attest_async(self, nonce, region, rounds, raw_out, per_warp_out=None, nbytes=None):
        return attest_async(self.ctx, nonce, region, rounds, raw_out, per_warp_out, nbytes)

    def attest_coverage(self, nonce, region, rounds, counts_out, nbytes=None):
        return attest_coverage(self.ctx, nonce, region, rounds, counts_out, nbytes)

    def kernel_hash(self, r, code, nbytes=None):
        return kernel_hash(self.ctx, r, code, nbytes)

    def attest_host(self, nonce, host_region, rounds, nbytes=None):
        return attest_host(self.ctx, nonce, host_region, rounds, nbytes)

    def host_region_va(self, nbytes):
        return host_region_va(self.ctx, nbytes)

    def placement_for(self, nbytes):
        return placement_for(self.ctx, nbytes)

    def kernel_symbol(self, nbytes, region_va=0):
        return kernel_symbol(self.ctx, nbytes, region_va)

    def device_uuid(self):
        return device_uuid(self.ctx)

    def query(self):
        return query(self.ctx)

    @property
    def launches(self):
        return launch_count(self.ctx)

    @property
    def stream(self):
        return stream(self.ctx)

    def close(self):
        if self.ctx is not None:
            checksum_destroy(self.ctx)
            self.ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
