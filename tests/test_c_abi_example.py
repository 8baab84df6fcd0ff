"""The C ABI from plain C: examples/attest_cli.c compiles as C99 against
include/sage.h and links libsage.so alone (static CUDA runtime inside); on a
GPU it attests and matches the oracle."""
import json
import os
import shutil
import subprocess

import numpy as np
import pytest

from paper_2209_03125_b200 import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2209_03125_b200")


def compile_cli(tmp_path):
    build.build()
    exe = str(tmp_path / "attest_cli")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "attest_cli.c"), "-o", exe, "-L", PKG, "-lsage",
                    "-Wl,-rpath," + PKG], check=True, capture_output=True, text=True)
    return exe


@pytest.mark.skipif(shutil.which("gcc") is None, reason="no gcc")
def test_example_compiles_and_links_as_c99(tmp_path):
    exe = compile_cli(tmp_path)
    out = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "libsage.so" in out and "libcudart" not in out


@pytest.mark.gpu
def test_example_runs_and_matches_oracle(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    exe = compile_cli(tmp_path)
    res = json.loads(subprocess.run([exe, "100", "4096", "0x77"], check=True, capture_output=True,
                                    text=True).stdout)
    host = np.array([(i * 2654435761 >> 13) & 0xFF for i in range(4096)], dtype=np.uint8)
    want = oracle.attest(0x77, host, int(res["region_va"], 16), 100, res["blocks"], res["threads"], 1)
    assert int(res["checksum"], 16) == want
