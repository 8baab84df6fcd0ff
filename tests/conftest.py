import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_addoption(parser):
    parser.addoption("--sage-lib", default=None,
                     help="load this build of the C-ABI library instead of libsage.so (e.g. the bounds-checked "
                          "bench/libsage_checked.so)")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libsage.so")
    config.addinivalue_line("markers", "statistical: decided by timing statistics on the GPU (run after the "
                                       "deterministic tests)")
    lib = config.getoption("--sage-lib")
    if lib:
        from paper_2209_03125_b200 import sage
        loaded = sage.load(os.path.abspath(lib))
        assert os.path.realpath(loaded._name) == os.path.realpath(lib), (loaded._name, lib)


def pytest_report_header(config):
    lib = config.getoption("--sage-lib")
    return ["C-ABI library under test: %s" % os.path.abspath(lib)] if lib else []


def pytest_collection_modifyitems(config, items):
    """Run the statistical timing tests last (stable order otherwise): under `-x` a
    timing outlier must not keep the bit-exact parity tests from running."""
    items.sort(key=lambda item: item.get_closest_marker("statistical") is not None)
