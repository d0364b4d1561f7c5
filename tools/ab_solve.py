"""A/B timing of the config-2 solve across environment variants (library builds,
F3RG_* switches): runs each variant in its own process, interleaved R times, and
prints the median graph-mode time per variant.

    python tools/ab_solve.py R "" "F3RG_PDL=0" "F3RG_LIB=paper_2505_20719_b200/lib/variants/x.so"
"""
import os
import re
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
reps = int(sys.argv[1])
variants = sys.argv[2:] or [""]
times = {v: [] for v in variants}
for _ in range(reps):
    for v in variants:
        env = dict(os.environ)
        for kv in v.split():
            k, val = kv.split("=", 1)
            env[k] = val
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "profile_solve.py"), "--solves", "4"],
                             env=env, capture_output=True, text=True).stdout
        ts = [float(x) for x in re.findall(r"t=([0-9.]+) ms", out)][2:]
        times[v].extend(ts)
for v in variants:
    t = times[v]
    print(f"{v or '(default)':70s} median {statistics.median(t):7.3f} ms  min {min(t):7.3f}  n={len(t)}")
