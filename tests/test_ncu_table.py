"""scripts/ncu_table.py (the counter tables under profiles/r02/) on a synthetic
ncu --csv launch list: per-pick division, duplicate launches averaged, missing
metrics shown as '-'."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_table_from_synthetic_csv(tmp_path):
    rows = ['"ID","Kernel Name","Metric Name","Metric Unit","Metric Value"']
    for launch, ms in ((0, "2,000,000"), (1, "4,000,000")):        # ns; averaged -> 3 ms
        rows += ['"%d","void k<1, 0>(Args)","gpu__time_duration.sum","ns","%s"' % (launch, ms),
                 '"%d","void k<1, 0>(Args)","dram__bytes_read.sum","byte","%d"' % (launch, 6400 * (launch + 1)),
                 '"%d","void k<1, 0>(Args)","lts__t_sector_hit_rate.pct","%%","12.5"' % launch]
    path = tmp_path / "l.csv"
    path.write_text("==PROF== Connected\n" + "\n".join(rows) + "\n")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_table.py"), "100", "x=%s" % path],
                         capture_output=True, text=True, check=True).stdout.splitlines()
    assert out[0].startswith("| launch | picks/s | ms | L2 hit %")
    cells = [c.strip() for c in out[2].split("|")[1:-1]]
    assert cells[0] == "x <1, 0>"
    assert abs(float(cells[1]) - 100 / 3e-3) < 50             # picks/s from the mean time (3 sig. digits)
    assert cells[2] == "3.00" and cells[3] == "12.5"
    assert cells[4] == "96.0"                                 # (6400 + 12800) / 2 / 100 bytes per pick
    assert cells[5] == "-"
