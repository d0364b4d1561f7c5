"""Standalone SpMV rate per precision triple on one BASELINE config (the bench's
spmv_per_precision), for tile-config sweeps (F3RG_LIB=<variant .so>) and single-
kernel ncu captures (--once pa,px,py: warm-up + one launch of that triple).

    python tools/spmv_probe.py --config 5
    ncu ... python tools/spmv_probe.py --config 5 --once 2,2,2
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--once", default=None)
args = ap.parse_args()

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2505_20719_b200 as f  # noqa: E402
from paper_2505_20719_b200 import problems  # noqa: E402

p = problems.problem(args.config)
reps = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values))
if args.once:
    pa, px, py = (int(v) for v in args.once.split(","))
    x = f.DenseVector(torch.rand(p.n, device="cuda", dtype=torch.float64).to(f.torch_dtype(px)))
    y = f.DenseVector(p.n, f.Precision(py))
    for _ in range(2):
        f.spmv(reps.at(f.Precision(pa)), x, y)
    torch.cuda.synchronize()
    print("done")
else:
    for row in bench.spmv_per_precision(f, torch, reps, p):
        print(json.dumps({"lib": os.path.basename(os.environ.get("F3RG_LIB", "default")), **row}))
