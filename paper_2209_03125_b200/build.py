"""Build libsage.so (the C-ABI library) and the kernel cubin, in-tree, for sm_100a.

    python -m paper_2209_03125_b200.build
"""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libsage.so")
# Test-only bounds-checked build of the same sources (-DSAGE_BOUNDS_CHECK: every
# shared / global address a kernel reads is checked and a violation traps); not
# the product, kept beside the other test-only library under bench/.
CHECKED_LIB = os.path.join(ROOT, "bench", "libsage_checked.so")
CUBIN = os.path.join(PKG, "sage_kernel.cubin")
# The c2a kernel with control-bit-tuned scheduling hints: the
# cubin above with the yield hints of csrc/c2a_yield.json applied; the library
# launches the c2a kernel from it (and falls back to the embedded kernel if it is
# missing or does not match).
TUNED_CUBIN = os.path.join(PKG, "sage_kernel_tuned.cubin")
YIELD_SPEC = os.path.join(CSRC, "c2a_yield.json")
SOURCES = [os.path.join(CSRC, "sage_api.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "sage_kernel.cuh"), os.path.join(CSRC, "sage_hash.cuh"),
                  os.path.join(INCLUDE, "sage.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v", "-I" + INCLUDE, "-I" + CSRC]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale(target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in DEPS)


def _check_spills(log):
    bad = [ln for ln in log.splitlines() if "spill" in ln and not ln.strip().startswith("0 bytes")
           and " 0 bytes spill stores, 0 bytes spill loads" not in ln]
    if bad:
        raise RuntimeError("ptxas reported register spills in the checksum kernel:\n" + "\n".join(bad))


def build(force=False, verbose=False):
    """Compile libsage.so and sage_kernel.cubin if stale. Raises on failure or spills."""
    if force or _stale(LIB):
        tmp = LIB + ".%d.tmp" % os.getpid()
        cmd = [_nvcc()] + ARCH + FLAGS + ["-shared", "-Xcompiler", "-fPIC", "-o", tmp] + SOURCES
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + p.stdout + p.stderr)
        _check_spills(p.stdout + p.stderr)
        if verbose:
            sys.stderr.write(p.stderr)
        os.replace(tmp, LIB)
    if force or _stale(CUBIN):
        tmp = CUBIN + ".%d.tmp" % os.getpid()
        cmd = [_nvcc()] + ARCH + FLAGS + ["-cubin", "-o", tmp] + SOURCES
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError("nvcc -cubin failed:\n" + p.stdout + p.stderr)
        os.replace(tmp, CUBIN)
    build_tuned()
    return LIB


def _elf_section(blob, name):
    """(file offset, size) of ELF64 section `name`, or None."""
    import struct
    shoff, = struct.unpack_from("<Q", blob, 0x28)
    shentsize, shnum, shstrndx = struct.unpack_from("<HHH", blob, 0x3A)
    hdrs = [struct.unpack_from("<IIQQQQ", blob, shoff + k * shentsize) for k in range(shnum)]
    stroff = hdrs[shstrndx][4]
    for nm, _t, _f, _a, off, size in hdrs:
        end = blob.index(b"\0", stroff + nm)
        if blob[stroff + nm:end].decode("latin-1") == name:
            return off, size
    return None


def tuned_cubin(blob, spec):
    """The cubin `blob` with the spec's yield hints applied (bit `yield_bit` of the
    high 64-bit word of each listed instruction set to its target value), or None
    when the kernel's text is not the one the hints were searched on (checked by
    the SHA-256 of the untuned text): scheduling hints never change what an
    instruction computes, but they are only known to help that exact schedule."""
    import hashlib
    sec = _elf_section(blob, ".text." + spec["function"])
    if sec is None:
        return None
    off, size = sec
    bit = spec["yield_bit"]
    text = bytearray(blob[off:off + size])
    for a, v in spec["yield"].items():               # back to the untuned value for the hash
        p = int(a) + 8
        w = int.from_bytes(text[p:p + 8], "little")
        w = (w | (1 << bit)) if not v else (w & ~(1 << bit))
        text[p:p + 8] = w.to_bytes(8, "little")
    if hashlib.sha256(bytes(text)).hexdigest() != spec["untuned_text_sha256"]:
        return None
    out = bytearray(blob)
    for a, v in spec["yield"].items():
        p = off + int(a) + 8
        w = int.from_bytes(out[p:p + 8], "little")
        w = (w | (1 << bit)) if v else (w & ~(1 << bit))
        out[p:p + 8] = w.to_bytes(8, "little")
    return bytes(out)


def build_tuned():
    """Write TUNED_CUBIN from CUBIN and YIELD_SPEC (removes it when the spec does not
    match the build's kernel).  Returns the path or None."""
    import json
    if not os.path.exists(YIELD_SPEC) or not os.path.exists(CUBIN):
        return None
    spec = json.load(open(YIELD_SPEC))
    blob = open(CUBIN, "rb").read()
    out = tuned_cubin(blob, spec)
    if out is None:
        if os.path.exists(TUNED_CUBIN):
            os.remove(TUNED_CUBIN)
        sys.stderr.write("build: %s does not match the built c2a kernel; the library runs the untuned kernel\n"
                         % YIELD_SPEC)
        return None
    if not os.path.exists(TUNED_CUBIN) or open(TUNED_CUBIN, "rb").read() != out:
        tmp = TUNED_CUBIN + ".%d.tmp" % os.getpid()
        with open(tmp, "wb") as f:
            f.write(out)
        os.replace(tmp, TUNED_CUBIN)
    return TUNED_CUBIN


def build_checked(force=False):
    """Compile the bounds-checked library (CHECKED_LIB) if stale.  Register spills
    are allowed here: it is a correctness instrument, not timed."""
    if force or _stale(CHECKED_LIB):
        tmp = CHECKED_LIB + ".%d.tmp" % os.getpid()
        cmd = [_nvcc()] + ARCH + FLAGS + ["-DSAGE_BOUNDS_CHECK", "-shared", "-Xcompiler", "-fPIC", "-o", tmp] + SOURCES
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError("nvcc (bounds-checked build) failed:\n" + p.stdout + p.stderr)
        os.replace(tmp, CHECKED_LIB)
    return CHECKED_LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    if "--checked" in sys.argv:
        print(build_checked(force="--force" in sys.argv))
    print(LIB)
