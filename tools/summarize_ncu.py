"""Summaries of ncu output for profiles/ (markdown on stdout).

  python tools/summarize_ncu.py launches gpurun_out/r1/launches.csv [--solve 2]
      per-kernel launch count, mean duration and share of one solve from a
      `ncu --metrics gpu__time_duration.sum --csv` launch list (tools/profile_solve.py
      runs --solves N; --solve picks which one, by splitting at the norm2[b] launches)
  python tools/summarize_ncu.py full gpurun_out/r1/full.ncu-rep
      duration, DRAM bytes, throughput, occupancy and registers per captured launch
      of a `--set full` report
"""
import collections
import csv
import io
import re
import subprocess
import sys


def short(name):
    name = re.sub(r"\(f3rg::.*$|\(CsrDev.*$|\(const void.*$|\(void \*.*$", "", name)
    name = name.replace("void ", "").replace("f3rg::", "").replace("(int)", "")
    return name.strip()


def launches(path, solve=None):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    H = rows[h]
    ki, vi, ii = H.index("Kernel Name"), H.index("Metric Value"), H.index("ID")
    seq = [(short(r[ki]), float(r[vi].replace(",", ""))) for r in rows[h + 1:] if len(r) > vi]
    # solves start with the bnorm reduction (k_dot over b, first launch of run())
    starts = [i for i, (k, _) in enumerate(seq) if k.startswith("k_dot<2, 2")]
    if solve is not None and starts:
        s = starts[min(solve, len(starts)) - 1]
        e = starts[solve] if solve < len(starts) else len(seq)
        seq = seq[s:e]
    agg = collections.OrderedDict()
    for k, v in seq:
        agg.setdefault(k, []).append(v)
    tot = sum(v for _, v in seq)
    print(f"launches: {len(seq)}, summed kernel time {tot / 1e6:.3f} ms "
          "(ncu-serialised, cache state per launch as left by the previous kernel)\n")
    print("| kernel | launches | mean us | total ms | share |")
    print("|---|---:|---:|---:|---:|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / 1e6:.3f} | {sum(v) / tot:.3f} |")


UNIT = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "byte": 1.0, "Kbyte": 1e3,
        "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte/s": 1e12, "Gbyte/s": 1e9, "Mbyte/s": 1e6}

# (metric, label, scale from SI base units)
METRICS = [
    ("gpu__time_duration.sum", "us", 1e6),
    ("dram__bytes_read.sum", "MB rd", 1e-6),
    ("dram__bytes_write.sum", "MB wr", 1e-6),
    ("dram__bytes.sum.per_second", "DRAM GB/s", 1e-9),
    ("dram__cycles_active.min.pct_of_peak_sustained_elapsed", "DRAM busy min %", 1),
    ("dram__cycles_active.max.pct_of_peak_sustained_elapsed", "DRAM busy max %", 1),
    ("lts__t_sector_hit_rate.pct", "L2 hit %", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("launch__grid_size", "grid", 1),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    H, U = rows[0], rows[1]
    idx = {m: H.index(m) for m, _, _ in METRICS if m in H}
    ki = H.index("Kernel Name")
    print("| kernel | " + " | ".join(lbl for m, lbl, _ in METRICS if m in idx) + " | DRAM bytes/launch |")
    print("|---|" + "---:|" * (len(idx) + 1))
    for r in rows[2:]:
        if len(r) <= ki:
            continue
        def val(m):
            return float(r[idx[m]].replace(",", "")) * UNIT.get(U[idx[m]], 1.0)

        cells = []
        for m, _, sc in METRICS:
            if m in idx:
                v = val(m) * sc
                cells.append(f"{v:.1f}" if v < 1e4 else f"{v:.0f}")
        rd = val("dram__bytes_read.sum") if "dram__bytes_read.sum" in idx else 0
        wr = val("dram__bytes_write.sum") if "dram__bytes_write.sum" in idx else 0
        print(f"| `{short(r[ki])}` | " + " | ".join(cells) + f" | {rd + wr:.0f} |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        sv = int(sys.argv[sys.argv.index("--solve") + 1]) if "--solve" in sys.argv else None
        launches(sys.argv[2], sv)
    else:
        full(sys.argv[2])
