import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libsage.so")
    config.addinivalue_line("markers", "statistical: decided by timing statistics on the GPU (run after the "
                                       "deterministic tests)")


def pytest_collection_modifyitems(config, items):
    """Run the statistical timing tests last (stable order otherwise): under `-x` a
    timing outlier must not keep the bit-exact parity tests from running."""
    items.sort(key=lambda item: item.get_closest_marker("statistical") is not None)
