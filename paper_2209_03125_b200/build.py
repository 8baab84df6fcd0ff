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
    return LIB


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
