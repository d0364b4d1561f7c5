"""Runs the config-N fp16-F3R solve `--solves` times (first one = warm-up) for
ncu / compute-sanitizer captures. Prints the outer count and time per solve."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2505_20719_b200 as f  # noqa: E402
from paper_2505_20719_b200 import csr_cache, problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--grid", type=int, default=None)
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--spec", default="F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > identity")
ap.add_argument("--eager", action="store_true", help="launch kernels eagerly (profile mode) instead of the graph")
a = ap.parse_args()
p = csr_cache.load(a.config) if a.grid is None else problems.problem(a.config, grid=a.grid)
reps = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values))
s = f.build(f.parse_solver_spec(a.spec), reps, f.IdentityPrecond(p.n))
b = torch.from_numpy(__import__("numpy").ascontiguousarray(p.b)).cuda()
for i in range(a.solves):
    s.set_profile(a.eager)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.reset()
    r = s.run(b, f.RunOptions(tol=1e-10))
    torch.cuda.synchronize()
    print(f"solve {i}: outer={r.report.outer_iterations} res={r.report.final_true_residual:.3e} "
          f"t={1e3 * (time.perf_counter() - t0):.2f} ms hist={['%.2e' % h for h in r.report.residual_history]}")
if a.eager:
    for k in sorted(s.profile(), key=lambda k: -k[1]):
        print(f"{k[0]:40s} {k[1]:9.3f} ms {k[2]:6d} launches {k[3] / k[2] / (k[1] / k[2] * 1e-3) / 1e9:8.1f} GB/s")
