"""B200-native SAGE checksum hot path (arXiv 2209.03125, section 5.2.2).

The checksum runs only in the sm_100a CUDA kernel behind the C ABI in
include/sage.h (libsage.so, built in-tree by paper_2209_03125_b200.build);
`sage` is the ctypes binding.  There is no CPU fallback: calls raise if the
library is missing.
"""
from . import inputs, verifier                      # noqa: F401
from .sage import (SAGE_AUTO, SAGE_GLOBAL, SAGE_HYBRID, SAGE_SMEM, Context, SageError,  # noqa: F401
                   attest, attest_async, attest_coverage, attest_debug, attest_host, checksum_destroy,
                   checksum_init, decode_raw, host_region_va, kernel_hash, launch_count, load, placement_for,
                   query)
