"""CPU checks of the scheduling-control-bit probe (scripts/sass_ctl_probe.py,
DESIGN.md section 8): the decoded reuse field agrees with cuobjdump's `.reuse`
annotations (which pins the bit layout), and a patch changes only the main loop's
control bits -- the disassembled instructions are identical."""
import os
import re
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))

pytestmark = pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump not available")


def _sass_text(path):
    """Disassembly without the encoding words and without `.reuse` annotations:
    cuobjdump prints `.reuse` only where bit 45 is also set (an instruction that
    yields drops the operand-reuse cache), so the annotation follows the patch
    while the reuse bits themselves are untouched."""
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    return [re.sub(r"\s+", " ", ln.split("/*")[1] if ln.strip().startswith("/*") else ln).replace(".reuse", "")
            for ln in out.splitlines() if not re.match(r"\s*/\* 0x", ln)]


@pytest.fixture(scope="module")
def probe():
    from paper_2209_03125_b200 import build
    build.build()
    import sass_ctl_probe
    return sass_ctl_probe


def test_reuse_field_matches_disassembly(probe):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", probe.FN, probe.CUBIN], capture_output=True, text=True,
                         check=True).stdout
    pairs = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(.*?);\s*/\* 0x[0-9a-f]+ \*/\s*\n\s*/\* (0x[0-9a-f]+) \*/", out)
    assert len(pairs) > 1000
    for text, hi in pairs:
        assert (".reuse" in text) == bool((int(hi, 16) >> 58) & 0xF), text
        if ".reuse" in text:
            assert (int(hi, 16) >> 45) & 1, text


@pytest.mark.parametrize("mode", ["yieldflip", "stall+1", "rand:3:0.05"])
def test_patch_touches_only_control_bits(probe, tmp_path, mode):
    blob = open(probe.CUBIN, "rb").read()
    new = probe.patched(blob, mode)
    assert new != blob and len(new) == len(blob)
    off, size = probe.text_section(blob, ".text." + probe.FN)
    lo, hi = probe.main_loop(probe.CUBIN)
    for i in range(len(blob)):
        if blob[i] != new[i]:
            assert off + lo <= i < off + hi and (i - off) % 16 >= 8, i     # high word of a loop instruction
    path = tmp_path / "patched.cubin"
    path.write_bytes(new)
    assert _sass_text(str(path)) == _sass_text(probe.CUBIN)


def test_tuned_cubin_differs_only_in_the_specs_yield_hints(probe):
    """The build's sage_kernel_tuned.cubin (the c2a kernel the library launches,
    DESIGN.md section 8) is sage_kernel.cubin with bit 45 changed at exactly the
    instructions csrc/c2a_yield.json lists, all inside the c2a round loop, and the
    same disassembly."""
    import json
    from paper_2209_03125_b200 import build
    if build.build_tuned() is None:
        pytest.skip("no yield spec for this build's kernel")
    spec = json.load(open(build.YIELD_SPEC))
    base, tuned = open(build.CUBIN, "rb").read(), open(build.TUNED_CUBIN, "rb").read()
    assert len(base) == len(tuned)
    off, _ = probe.text_section(base, ".text." + probe.FN)
    lo, hi = probe.main_loop(build.CUBIN)
    changed = [i for i in range(len(base)) if base[i] != tuned[i]]
    want = set()
    for a, v in spec["yield"].items():
        a = int(a)
        assert lo <= a < hi and a % 16 == 0
        p = off + a + 8
        wb, wt = (int.from_bytes(x[p:p + 8], "little") for x in (base, tuned))
        assert wb ^ wt == 1 << 45 and (wt >> 45) & 1 == v
        want.add(p + 5)                                    # bit 45 lives in byte 5 of the high word
    assert set(changed) == want
    assert _sass_text(build.TUNED_CUBIN) == _sass_text(build.CUBIN)
