"""The C-ABI library loads and exports every symbol include/sage.h declares
(no compute calls: this runs without a GPU)."""
import ctypes

import numpy as np
import os
import re

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


def test_strerror_and_codes(lib):
    assert sage.strerror(0) == "ok"
    assert sage.strerror(-1) == "invalid argument"
    assert sage.strerror(-2) == "unsupported configuration"
    assert sage.strerror(-4) == "CUDA error"


def test_header_matches_binding_structs():
    # sage_result / sage_config layouts as declared in sage.h
    assert ctypes.sizeof(sage.sage_config) == 4 + 4 * 4 + 8 + 4  # int + 4 u32 + pad + void*
    assert ctypes.sizeof(sage.sage_result) == 5 * 8 + 4 * 4


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
             lambda: sage.query(None),
             lambda: sage.kernel_hash(None, b"", None)]
    for call in calls:
        with pytest.raises(sage.SageError) as e:
            call()
        assert e.value.code == sage.SAGE_EINVAL
    assert sage.launch_count(None) == 0
