"""Host logic of scripts/schedule_search.py (no GPU, no compile)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))

import schedule_search as S  # noqa: E402


def test_parse_range_and_grid():
    assert S.parse_range("16-19") == [16, 17, 18, 19]
    assert S.parse_range("1,4,8") == [1, 4, 8]
    assert S.parse_range("0-2,7") == [0, 1, 2, 7]
    pts = S.grid([17, 18], [6, 7], [16], [4])
    assert pts == [(16, 17, 4, 6), (16, 17, 4, 7), (16, 18, 4, 6), (16, 18, 4, 7)]
