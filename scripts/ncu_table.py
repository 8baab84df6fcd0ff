"""Markdown table of per-pick counters from `ncu --metrics ... --csv` launch lists
(the c3 / c2c counter tables under profiles/r02/).

    python scripts/ncu_table.py N_THREAD_ROUNDS label=file.csv [label=file.csv ...]

Every launch (ID) of the file becomes a row (duplicates of the same kernel name in
one file are averaged); per-pick quantities divide by N_THREAD_ROUNDS (n * R of
the profiled launch)."""
import collections
import csv
import sys

COLS = [
    ("ms", "gpu__time_duration.sum", 1e-6, "{:.2f}"),
    ("L2 hit %", "lts__t_sector_hit_rate.pct", 1, "{:.1f}"),
    ("DRAM B/pick", "dram__bytes_read.sum", "pick", "{:.1f}"),
    ("DRAM busy %", "dram__throughput.avg.pct_of_peak_sustained_elapsed", 1, "{:.1f}"),
    ("L1->L2 sectors/pick", "l1tex__m_xbar2l1tex_read_sectors.sum", "pick", "{:.2f}"),
    ("L2 sectors/pick", "lts__t_sectors_srcunit_tex_op_read.sum", "pick", "{:.2f}"),
    ("L2 miss sectors/pick", "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum", "pick", "{:.2f}"),
    ("L1->xbar req busy %", "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed", 1, "{:.1f}"),
    ("L2 sector BW %", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", 1, "{:.1f}"),
]


def load(path):
    rows = list(csv.reader(ln for ln in open(path) if not ln.startswith("==")))
    hdr = rows[0]
    ik, im, iv, iid = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) > iv:
            per.setdefault(r[iid], {"_k": r[ik]})[r[im]] = float(r[iv].replace(",", ""))
    by_kernel = collections.OrderedDict()
    for d in per.values():
        by_kernel.setdefault(d["_k"], []).append(d)
    return by_kernel


def main(argv):
    n = float(argv[1])
    print("| launch | picks/s | " + " | ".join(c[0] for c in COLS) + " |")
    print("|---" * (len(COLS) + 2) + "|")
    for spec in argv[2:]:
        label, path = spec.split("=", 1)
        for k, ds in load(path).items():
            avg = {m: sum(d.get(m, 0.0) for d in ds) / len(ds) for m in ds[0] if m != "_k"}
            cells = []
            for _, m, scale, fmt in COLS:
                if m not in avg:
                    cells.append("-")
                    continue
                v = avg[m] / n if scale == "pick" else avg[m] * scale
                cells.append(fmt.format(v))
            rate = n / (avg["gpu__time_duration.sum"] * 1e-9)
            tag = k[k.find("<"):k.find(">") + 1] if "<" in k else k[:40]
            print("| %s %s | %.3g | %s |" % (label, tag, rate, " | ".join(cells)))


if __name__ == "__main__":
    main(sys.argv)
