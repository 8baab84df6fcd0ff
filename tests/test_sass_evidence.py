"""Build evidence from the compiled library (no GPU needed): the checksum
kernels are sm_100a SASS, stage the region with the TMA bulk-copy engine
(UBLKCP + mbarrier SYNCS), run R7 as IMAD + LEA.HI pairs, exchange through
SHFL.IDX, and fit 32 registers (2 x 1024 threads per SM)."""
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
    ks = {n: r for n, r in regs.items() if n.startswith("_ZN4sage20sage_checksum_kernel")}
    assert ks
    # <..., ILP=2, PROBE=0, PAD, SYNC=0, FEXTRA=0>: the c2a kernel (PAD 10) and the SAGE_HYBRID kernel (ADDR 8, PAD 8)
    ilp2 = [n for n in ks if re.search(r"ELi2ELi0ELi\d+ELi0ELi0EEEvNS_10KernelArgsE$", n)]
    assert len(ilp2) == 2 and any("ELi8ELi0ELi0ELb0ELi0ELi2ELi0ELi8E" in n for n in ilp2), ilp2
    for n, r in ks.items():
        if n in ilp2:
            # one CTA of 1024 threads per SM must allocate the whole 64 K register file:
            # registers are allocated per warp in units of 256, i.e. 8 per thread
            assert 56 < r <= 64 and -(-r // 8) * 8 == 64, (n, r)
        else:
            assert r <= 32, (n, r)


@pytest.mark.parametrize("name,rounds", [("ILi1ELb1ELb0ELi16ELi18ELi4ELi0ELi0ELb0ELi0ELi2ELi0ELi7E", 36),
                                         ("ILi1ELb1ELb0ELi16ELi32ELi4E", 32)])
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
