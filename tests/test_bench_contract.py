"""bench.py's output contract (the JSON line the driver parses): the oracle
(reference) arm on CPU, and on a GPU our arm at N=1 and the N=2 torchrun path
(two replicas sharing one GPU over gloo plumbing, 8(e))."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout                 # rank 0 prints exactly one JSON line
    return json.loads(lines[0])


def _check_base(line, n_gpus, steps, warmup):
    assert BASE_KEYS <= set(line), BASE_KEYS - set(line)
    assert line["metric"].startswith("checksum rounds/s")
    assert line["unit"] == "thread-rounds/s" and line["higher_is_better"] is True
    assert line["n_gpus"] == n_gpus and line["steps"] == steps and line["warmup"] == warmup
    assert line["value"] > 0 and line["ms_per_step"] > 0
    assert line["scaling"] == "weak" and line["vs_baseline"] is None
    assert line["dtype"] == "u32" and line["data"] == "synthetic"
    assert "workload" in line["config"]
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["unit"] == line["unit"]
    assert "h2d_bytes_per_step" in e2e and "d2h_bytes_per_step" in e2e


def test_reference_arm_on_cpu():
    line = _run(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "3"], 600)
    _check_base(line, 1, 2, 3)
    assert line["impl"] == "reference"
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


@pytest.mark.gpu
def test_our_arm_one_gpu():
    line = _run(["--config", "c2a", "--rounds", "2000", "--steps", "4", "--warmup", "3"], 900)
    _check_base(line, 1, 4, 3)
    assert line["gpu_launches"] == 4                 # one checksum kernel per timed step
    # value from the device time of the timed region (CUDA events, max over ranks), which
    # contains the four kernels and lies inside the host's wall-clock bracket
    tm = line["timing"]
    assert abs(line["ms_per_step"] * 4 / 1e3 - tm["device_s"]) < 1e-9
    assert 4 * line["kernel_ms"]["min"] / 1e3 <= tm["device_s"] <= tm["host_wall_s"]
    rf = line["roofline"]
    assert rf["bound"] == "alu" and 0 < rf["frac"] <= 1 and rf["peak"] > 0
    assert abs(rf["achieved"] / rf["peak"] - rf["frac"]) < 1e-9
    assert line["e2e"]["h2d_bytes_per_step"] == 8192 and line["e2e"]["d2h_bytes_per_step"] == 32
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["parity_on_sample"] is True and cb["cores"] >= 1
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"])
    assert line["attest_ms"]["p99"] >= line["attest_ms"]["p50"] > 0
    assert line["config"]["kernel"].startswith("_ZN4sage20sage_checksum_kernel")
    # the secondary configs timed in the same process
    ex = line["extra"]
    assert set(ex) == {"c2c", "c2cp4", "c2cp8", "c3p1", "c3p8", "attest_ms_r1e4"}
    for name in ("c2c", "c2cp4", "c2cp8", "c3p1", "c3p8"):
        e = ex[name]
        assert e["steps"] == 5 and e["gpu_launches"] == 5 and e["kernel_ms"]["mean"] > 0
        assert 0 < e["roofline"]["frac"] <= 1 and {"sm_mhz", "reasons"} <= set(e["clocks"])
    assert ex["c2c"]["placement"] == "hybrid" and "binding_limit" in ex["c2c"]["roofline"]
    assert ex["c3p1"]["roofline"]["bound"] == "hbm" and ex["c3p8"]["roofline"]["bound"] == "hbm"
    assert ex["attest_ms_r1e4"]["p50"] > 0


@pytest.mark.gpu
def test_our_arm_two_replicas_torchrun():
    line = _run(["--gpus", "2", "--config", "c2a", "--rounds", "2000", "--steps", "3", "--warmup", "3"], 900)
    _check_base(line, 2, 3, 3)
    reps = line["replicas"]
    assert len(reps) == 2 and {r["rank"] for r in reps} == {0, 1}
    assert reps[0]["nonce"] != reps[1]["nonce"]       # an independent nonce stream per replica
    assert all(r["sampled_parity_sum_ok"] for r in reps)
    assert all({"sm_mhz", "sm_max_mhz", "reasons", "power_w_median"} <= set(r["clocks"]) for r in reps)
    assert all(r["kernel_ms_mean"] > 0 for r in reps)
    assert "cpu_baseline" not in line                 # rank 0 at N=1 only


def _bench_module():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_main", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_roofline_records_on_cpu():
    """The roofline record's arithmetic (no GPU): the integer-issue fraction of an
    SMEM run, the HBM sector fraction, and the L1->L2 request-ceiling fraction of a
    SAGE_HYBRID run counts only the picks above the staged prefix."""
    b = _bench_module()
    peaks = {"hbm_gbs": 6400.0, "sm_max_mhz": 2000.0}
    n, R, t = 303104, 100_000, 0.05
    rf = b.roofline("smem", 8192, 1, n, R, t, peaks, "test", 148, "none")
    assert rf["bound"] == "alu" and rf["ops_per_thread_round"] == 59
    assert rf["frac"] == pytest.approx(n * R * 59 / t / (148 * 4 * 32 * 2e9))
    assert "l2_request_ceiling_picks_per_s" not in rf
    rf = b.roofline("global", 256 << 20, 1, n, 10_000, t, peaks, "test", 148, "none", gather_ceiling=1e11)
    assert rf["bound"] == "hbm" and rf["frac"] == pytest.approx(n * 1e4 * 32 / t / 1e9 / 6400.0)
    assert rf["frac_of_random_gather_ceiling"] == pytest.approx(n * 1e4 / t / 1e11)
    share = (524288 - b.HYBRID_STAGE) / 524288
    assert share == 0.625
    rf = b.roofline("hybrid", 524288, 1, n, R, t, peaks, "test", 148, "none", l2_ceiling=(2.7e11, share))
    assert rf["frac_of_l2_request_ceiling"] == pytest.approx(n * R * share / t / 2.7e11)
    assert b.l2_request_ceiling("smem", 8192) is None and b.l2_request_ceiling("global", 256 << 20) is None
