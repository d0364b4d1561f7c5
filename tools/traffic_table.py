"""Writes the measured DRAM traffic per launch of the captured kernels into
profiles/traffic.json (read by bench.py for roofline.traffic):

    python tools/traffic_table.py CONFIG capture_raw.csv [more_raw.csv ...]

Each csv is `ncu -i X.ncu-rep --page raw --csv` of a `--set full` capture; the
value is dram__bytes_read.sum + dram__bytes_write.sum of each captured launch,
keyed by the engine's kernel name (richardson[f16,f16,f32], ...)."""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "traffic.json")
PN = {"0": "f16", "1": "f32", "2": "f64"}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def engine_name(kernel):
    """void f3rg::k_richardson<(int)0, (int)0, (int)1, (int)8>(...) -> richardson[f16,f16,f32]"""
    m = re.search(r"k_(\w+?)<([^>]*)>", kernel)
    if not m:
        return None
    args = re.findall(r"\d+", m.group(2))
    return f"{m.group(1)}[{','.join(PN[a] for a in args[:3])}]"


def main(config, paths):
    table = json.load(open(OUT)) if os.path.exists(OUT) else {}
    row = table.setdefault(f"config{config}", {})
    for path in paths:
        rows = list(csv.reader(open(path)))
        head, units = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(head, r))
            name = engine_name(d.get("Kernel Name", ""))
            if not name:
                continue
            tot = 0.0
            for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                tot += float(d[key].replace(",", "")) * UNIT[units[head.index(key)]]
            row[name] = tot
            print(config, name, f"{tot / 1e9:.3f} GB")
    row["source"] = [os.path.relpath(p, ROOT) for p in paths]
    json.dump(table, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(int(sys.argv[1]), sys.argv[2:])
