"""The control-bit-tuned c2a kernel: the library launches the
c2a kernel from sage_kernel_tuned.cubin -- the same instructions with tuned
scheduling hints -- and it returns the embedded kernel's result bit for bit
(a context created while SAGE_NO_TUNED is set launches the embedded kernel)."""
import os

import pytest

torch = pytest.importorskip("torch")

from paper_2209_03125_b200 import build, sage                             # noqa: E402
from paper_2209_03125_b200.inputs import kernel_code_prefix, make_region, nonces   # noqa: E402

pytestmark = pytest.mark.gpu


def test_c2a_runs_the_tuned_kernel():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if build.build_tuned() is None:
        pytest.skip("no yield spec for this build's kernel")
    region = torch.from_numpy(make_region(8192)).to("cuda")
    with sage.Context() as ctx:
        assert ctx.attest(nonces(1)[0], region, 1000).tuned == 1
        assert ctx.attest(nonces(1)[0], region[:4096], 1000).tuned == 1       # same kernel, 4 KiB
    with sage.Context(blocks=2, threads=64) as ctx:                          # not the c2a geometry
        assert ctx.attest(nonces(1)[0], region, 1000).tuned == 0
    with sage.Context(pick_words=4) as ctx:
        assert ctx.attest(nonces(1)[0], region, 1000).tuned == 0


def test_tuned_and_embedded_kernels_agree_bit_for_bit():
    """Every warp partial of a full-occupancy c2a attestation on the same region
    (same VA): the tuned kernel vs the embedded one (a context created while
    SAGE_NO_TUNED is set launches the embedded kernel)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if build.build_tuned() is None:
        pytest.skip("no yield spec for this build's kernel")
    nonce, R = nonces(7)[6], 20_011
    region = torch.from_numpy(make_region(8192)).to("cuda")
    out = {}
    for flag in ("", "1"):
        if flag:
            os.environ["SAGE_NO_TUNED"] = flag
        try:
            with sage.Context() as ctx:
                info = ctx.query()
                pw = torch.zeros(info.blocks * info.threads // 32, dtype=torch.int64, device="cuda")
                r = ctx.attest_debug(nonce, region, R, pw)
                out[flag] = (r.tuned, r.checksum, pw.cpu().tolist())
        finally:
            os.environ.pop("SAGE_NO_TUNED", None)
    assert out[""][0] == 1 and out["1"][0] == 0
    assert out[""][1:] == out["1"][1:]


def test_region_prefix_is_the_tuned_code():
    """Self-verification: the c2a region starts with the machine code that runs,
    i.e. the tuned text, not the embedded kernel's."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if build.build_tuned() is None:
        pytest.skip("no yield spec for this build's kernel")
    from paper_2209_03125_b200.inputs import _elf_sections
    with sage.Context() as ctx:
        sym = ctx.kernel_symbol(8192)
        pre = kernel_code_prefix(ctx, 8192)
    tuned = _elf_sections(open(build.TUNED_CUBIN, "rb").read())[".text." + sym]
    base = _elf_sections(open(build.CUBIN, "rb").read())[".text." + sym]
    assert pre == tuned and pre != base
