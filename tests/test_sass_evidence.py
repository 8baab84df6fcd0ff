"""Build evidence from the compiled library (no GPU needed): the checksum
kernels are sm_100a SASS, stage the region with the TMA bulk-copy engine
(UBLKCP + mbarrier SYNCS), run R7 as IMAD + LEA.HI pairs, exchange through
SHFL.IDX, and fit 32 registers (2 x 1024 threads per SM) -- or,
for the two ILP-2 kernels, exactly the whole register file; the library holds
only the product's instantiations, and the lab template the timing adversaries
are built from matches the product's main loop."""
import re
import shutil
import subprocess

import pytest

from paper_2209_03125_b200 import build

pytestmark = pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump not available")


@pytest.fixture(scope="module")
def sass():
    lib = build.build()
    return subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout


@pytest.fixture(scope="module")
def res_usage():
    lib = build.build()
    return subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True, check=True).stdout


def _functions(sass):
    parts = re.split(r"\n\s+Function : ", sass)
    return {p.split("\n", 1)[0].strip(): p for p in parts[1:]}


def test_arch_is_sm100a(sass):
    assert "arch = sm_100a" in sass


def test_smem_kernels_use_tma_bulk_copy(sass):
    funcs = _functions(sass)
    prefix = "_ZN4sage20sage_checksum_kernelILi"
    smem = [n for n in funcs if n.startswith(prefix) and "ELb1E" in n[len(prefix):][:6]]   # <P, SMEM=true, ...>
    assert smem, "no SMEM checksum kernels found"
    for n in smem:
        body = funcs[n]
        assert "UBLKCP.S.G" in body, n
        assert "SYNCS.ARRIVE.TRANS64" in body and "SYNCS.PHASECHK.TRANS64" in body, n


def test_round_is_imad_leahi_and_shuffle(sass):
    funcs = _functions(sass)
    ks = [n for n in funcs if n.startswith("_ZN4sage20sage_checksum_kernel")]
    assert len(ks) >= 9
    for n in ks:
        body = funcs[n]
        assert "SHFL.IDX" in body, n
        assert len(re.findall(r"\bLEA\.HI\b", body)) >= 16, n
        assert len(re.findall(r"\bIMAD R\d+, R\d+, c\[0x0\]", body)) + \
            len(re.findall(r"\bIMAD R\d+, R\d+, UR\d+", body)) >= 16, n


# product template: sage_checksum_kernel<P, SMEM, STRADDLE, XS, UNROLL, ADDR, COUNT, ILP, PAD>
_PROD = re.compile(r"^_ZN4sage20sage_checksum_kernelILi(\d+)ELb(\d)ELb(\d)ELi(\d+)ELi(\d+)ELi(\d+)ELb(\d)ELi(\d)"
                   r"ELi(\d+)EEEvNS_10KernelArgsE$")

# The instantiations sage_api.cu launches: (P, SMEM, STRADDLE, XS, UNROLL, ADDR, COUNT, ILP, PAD)
PRODUCT_KERNELS = {
    (1, 1, 0, 16, 18, 4, 0, 2, 7): "c2a: P=1 SMEM, ILP 2 (1 CTA x 1024 threads x 2 lane states per SM)",
    (1, 1, 0, 16, 2, 8, 0, 2, 8): "SAGE_HYBRID (c2c)",
    (4, 1, 0, 16, 1, 8, 0, 2, 0): "SAGE_HYBRID, P=4 (c2cp4)",
    (1, 1, 0, 16, 32, 4, 0, 1, 0): "P=1 SMEM, ILP 1 (other geometries)",
    (1, 1, 1, 0, 16, 0, 0, 1, 0): "P=1 SMEM, region straddling 4 GiB",
    (1, 0, 1, 16, 16, 0, 0, 1, 0): "P=1 GLOBAL (c3)",
    (4, 1, 0, 0, 2, 2, 0, 1, 0): "P=4 SMEM",
    (4, 1, 1, 0, 2, 0, 0, 1, 0): "P=4 SMEM straddling",
    (4, 0, 1, 16, 16, 0, 0, 1, 0): "P=4 GLOBAL",
    (8, 1, 0, 0, 1, 1, 0, 1, 0): "P=8 SMEM",
    (8, 1, 1, 0, 1, 0, 0, 1, 0): "P=8 SMEM straddling",
    (8, 0, 1, 16, 1, 0, 0, 1, 0): "P=8 GLOBAL",
    (1, 0, 1, 0, 1, 0, 1, 1, 0): "coverage (COUNT), P=1",
    (4, 0, 1, 0, 1, 0, 1, 1, 0): "coverage (COUNT), P=4",
    (8, 0, 1, 0, 1, 0, 1, 1, 0): "coverage (COUNT), P=8",
}


def _product_key(name):
    m = _PROD.match(name)
    return tuple(int(v) for v in m.groups()) if m else None


def test_library_holds_only_the_product_kernels(sass):
    """libsage.so contains exactly the instantiations sage_api.cu launches (the
    checksum kernels above plus the SHA-256 kernel) -- no measurement variants
    (those are built from bench/sage_lab.cuh into bench binaries only)."""
    names = set(_functions(sass))
    assert names == {n for n in names if _product_key(n)} | {"_ZN4sage18sage_sha256_kernelENS_8HashArgsE"}, \
        sorted(n for n in names if not _product_key(n))
    assert {_product_key(n) for n in names if _product_key(n)} == set(PRODUCT_KERNELS)


def test_registers_allow_two_ctas_of_1024(res_usage):
    regs = {}
    name = None
    for ln in res_usage.splitlines():
        m = re.search(r"Function (\S+):", ln)
        if m:
            name = m.group(1)
        m = re.search(r"REG:(\d+)", ln)
        if m and name:
            regs[name] = int(m.group(1))
    ks = {_product_key(n): r for n, r in regs.items() if _product_key(n)}
    assert set(ks) == set(PRODUCT_KERNELS)
    for k, r in ks.items():
        if k[7] == 2:
            # the c2a (PAD 7) and SAGE_HYBRID (PAD 8) kernels: one CTA of 1024 threads per SM
            # must allocate the whole 64 K register file (allocated per warp in units of 256,
            # i.e. 8 registers per thread)
            assert 56 < r <= 64 and -(-r // 8) * 8 == 64, (k, r)
        else:
            assert r <= 32, (k, r)


def test_lab_template_matches_the_product_loop():
    """bench/sage_lab.cuh (the experiment harness the timing adversaries are built
    from) instantiated with the product's c2a and SAGE_HYBRID (P = 1, 4) parameters and every
    knob off has the same main-loop instruction stream as the product kernels (up to
    constant-bank offsets and branch addresses), so an adversary kernel is the
    product plus its injection."""
    import os
    import sys
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "scripts"))
    import sass_compare
    src = os.path.join(root, "bench", "sage_lab.cuh")
    with tempfile.TemporaryDirectory() as tmp:
        cu = os.path.join(tmp, "lab_eq.cu")
        with open(cu, "w") as f:
            f.write('#include "%s"\n' % src)
            f.write("template __global__ void sage_lab::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, 0, false, 0, 2, "
                    "0, 7>(const sage_lab::KernelArgs);\n")
            f.write("template __global__ void sage_lab::sage_checksum_kernel<1, true, false, 16, 2, 8, 0, 0, false, 0, 2, "
                    "0, 8>(const sage_lab::KernelArgs);\n")
            f.write("template __global__ void sage_lab::sage_checksum_kernel<4, true, false, 16, 1, 8, 0, 0, false, 0, 2, "
                    "0, 0>(const sage_lab::KernelArgs);\n")
        cubin = os.path.join(tmp, "lab_eq.cubin")
        subprocess.run(["nvcc"] + build.ARCH + ["-O3", "-std=c++17", "-cubin", "-o", cubin, cu], check=True,
                       capture_output=True)
        build.build()
        lab = sass_compare.functions(cubin)
        prod = sass_compare.functions(build.CUBIN)
        for key in ((1, 1, 0, 16, 18, 4, 0, 2, 7), (1, 1, 0, 16, 2, 8, 0, 2, 8), (4, 1, 0, 16, 1, 8, 0, 2, 0)):
            pn = [n for n in prod if _product_key(n) == key]
            ln = [n for n in lab if ("kernelILi%dE" % key[0]) in n and
                  "ELi%dELi%dELi0ELi0ELb0ELi0ELi2ELi0ELi%dE" % (key[4], key[5], key[8]) in n]
            assert len(pn) == 1 and len(ln) == 1, (pn, ln)
            a = sass_compare.main_loop(cubin, ln[0])
            b = sass_compare.main_loop(build.CUBIN, pn[0])
            assert a and a == b, key


@pytest.mark.parametrize("name,rounds", [("ILi1ELb1ELb0ELi16ELi18ELi4ELb0ELi2ELi7E", 36),
                                         ("ILi1ELb1ELb0ELi16ELi32ELi4ELb0ELi1ELi0E", 32)])
def test_c2a_kernel_op_mix(name, rounds):
    """The c2a product kernels (P=1, SMEM, non-straddling, XS=16, ADDR=4; ILP=2
    with 18 unrolled rounds of two lane states, and the ILP=1 fallback with 32):
    per logical round at most 30 ALU-pipe and 26 FMA-pipe instructions (one of them
    the IMAD.WIDE of x*M64), one LDS and one SHFL.IDX -- the minimum ALU count
    for SCS-2's shift/xor/rotate steps (DESIGN.md sections 7-8)."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    import sass_loop
    build.build()
    res = sass_loop.analyse(build.CUBIN, name)
    assert len(res) == 1, sorted(res)
    (d,) = res.values()
    assert d["rounds"] == rounds
    assert d["alu"] <= 30.1, d
    assert d["fma"] <= 26.1 and d["wide"] == 1.0, d
    assert d["hist"].get("LDS", 0) == rounds and d["hist"].get("SHFL.IDX", 0) == rounds, d


def test_bounds_checks_compile_out_of_the_product(sass):
    """The bounds checks (SAGE_CHECK) are in the test-only
    checked library -- a trap in every checksum kernel -- and nowhere in libsage.so,
    whose kernels are the same instantiations."""
    checked = build.build_checked()
    csass = subprocess.run(["cuobjdump", "-sass", checked], capture_output=True, text=True, check=True).stdout
    prod, chk = _functions(sass), _functions(csass)
    assert set(prod) == set(chk)
    for name, body in prod.items():
        assert "BPT.TRAP" not in body, name
        if "sage_checksum_kernel" in name:
            assert "BPT.TRAP" in chk[name], name
