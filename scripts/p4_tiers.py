"""P = 4 placement tiers (session 2): device time of the product's SMEM, HYBRID
and GLOBAL kernels for 16-B picks at 64 KiB ... 1 MiB (R = 1e5; 2e4 at 1 MiB),
to set SAGE_AUTO's P = 4 rule (development aid, like quick_time.py)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from quick_time import time_cfg  # noqa: E402

from paper_2209_03125_b200 import sage  # noqa: E402

if __name__ == "__main__":
    for nbytes in (64 << 10, 128 << 10, 256 << 10, 512 << 10, 1 << 20):
        R = 20_000 if nbytes >= (1 << 20) else 100_000
        for pl in (sage.SAGE_SMEM, sage.SAGE_HYBRID, sage.SAGE_GLOBAL):
            if pl == sage.SAGE_SMEM and nbytes > (64 << 10):
                continue
            for rep in range(2):
                d = time_cfg(nbytes, 4, R, placement=pl)
                d["placement_name"] = sage.PLACEMENT_NAMES[pl]
                print(json.dumps(d), flush=True)
