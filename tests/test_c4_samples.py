"""CPU check of the stored config-4 samples: the per-warp partials recorded by
scripts/timing_distribution.py on the B200 (from the GPU kernel) are recomputed
by the oracle on the same region bytes and device VA.  Skips when no capture
is committed.  Up to four samples per R <= 10^5, two at 10^6 and one at 10^7
are recomputed (one warp at 10^7 rounds is ~5 s of oracle time); merged
captures carry each sample's own region VA."""
import json
import os

import numpy as np
import pytest

import oracle

PROFILES = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
PATHS = [os.path.join(PROFILES, "r01", f) for f in ("scs2/c4_timing.json", "scs2/c4_timing_full.json",
                                                    "ilp2/c4_timing_full.json", "final/c4_timing_full.json",
                                                    "final/c4_timing_full_v2.json")] + \
    [os.path.join(PROFILES, "r02", "final", "c4_timing.json"), os.path.join(PROFILES, "r02", "c4", "c4_timing_1000.json")]


@pytest.mark.parametrize("path", PATHS)
def test_c4_sampled_warps_match_oracle(path):
    if not os.path.exists(path):
        pytest.skip("no config-4 capture committed")
    with open(path) as f:
        d = json.load(f)
    region = np.frombuffer(bytes.fromhex(d["region_hex"]), dtype=np.uint8)
    checked = 0
    for ent in d["per_R"]:
        assert ent["sum_of_partials_ok"] == ent["n_attest"]
        R = ent["rounds"]
        k = 4 if R < 1_000_000 else 2 if R < 10_000_000 else 1 if R == 10_000_000 and "chunks" in ent else 0
        for s in ent["samples"][:k]:
            want = oracle.warp_sum(s["nonce"], region, s.get("region_va", d["region_va"]), R, s["warp"], d["P"])
            assert want == s["warp_partial"], (ent["rounds"], s)
            checked += 1
    assert checked > 0
