"""The C-ABI library loads and exports every symbol include/sage.h declares
(no compute calls: this runs without a GPU)."""
import ctypes

import numpy as np
import os
import re
import subprocess

import pytest

from paper_2209_03125_b200 import build, sage

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "sage.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sage_[a-z_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return sage.load()


def test_library_exports_every_declared_symbol(lib):
    declared = _declared()
    assert "sage_attest" in declared and "sage_checksum_init" in declared
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(sage.EXPORTS) == declared


def test_bounds_checked_library_exports_the_same_symbols():
    """The test-only bounds-checked build (bench/libsage_checked.so, DESIGN.md
    section 8) is the same C ABI, so the parity suites can run through it."""
    checked = ctypes.CDLL(build.build_checked())
    for name in _declared():
        assert hasattr(checked, name), name


def test_strerror_and_codes(lib):
    assert sage.strerror(0) == "ok"
    assert sage.strerror(-1) == "invalid argument"
    assert sage.strerror(-2) == "unsupported configuration"
    assert sage.strerror(-4) == "CUDA error"


def test_header_matches_binding_structs(tmp_path):
    """The ctypes structs have the sizes and field offsets a C compiler gives the
    structs declared in include/sage.h."""
    structs = {"sage_config": sage.sage_config, "sage_result": sage.sage_result, "sage_info": sage.sage_info}
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "sage.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append('printf("%s %%zu\\n", sizeof(%s));' % (name, name))
        for f, _ in cls._fields_:
            lines.append('printf("%s.%s %%zu\\n", offsetof(%s, %s));' % (name, f, name, f))
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(ln.split() for ln in subprocess.run([str(exe)], capture_output=True, text=True,
                                                   check=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == ctypes.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(got["%s.%s" % (name, f)]) == getattr(cls, f).offset, (name, f)


def test_init_argument_validation_without_device(lib):
    # argument errors are reported before any device work
    with pytest.raises(sage.SageError) as e:
        sage.checksum_init(threads=48)
    assert e.value.code == sage.SAGE_EINVAL
    with pytest.raises(sage.SageError) as e:
        sage.checksum_init(pick_words=2)
    assert e.value.code == sage.SAGE_EINVAL


def test_no_oracle_in_product_path():
    """The product package never imports or loads the oracle."""
    pkg = os.path.join(ROOT, "paper_2209_03125_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in src and "from oracle" not in src and "liboracle" not in src, fn


def test_null_context_is_rejected_without_device(lib):
    """Every entry point checks its context before touching CUDA."""
    calls = [lambda: sage.attest(None, 0, 0x1000, 1, nbytes=16),
             lambda: sage.attest_host(None, 0, np.zeros(16, np.uint8), 1),
             lambda: sage.host_region_va(None, 16),
             lambda: sage.placement_for(None, 16),
             lambda: sage.kernel_symbol(None, 16),
             lambda: sage.query(None),
             lambda: sage.kernel_hash(None, b"", None)]
    for call in calls:
        with pytest.raises(sage.SageError) as e:
            call()
        assert e.value.code == sage.SAGE_EINVAL
    assert sage.launch_count(None) == 0
