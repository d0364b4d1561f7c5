"""Does the dot summation order alone explain outer-count differences at large n?

Runs the CPU oracle (our restatement of the reference, sequential dots exactly as
src/vector_ops.cpp:20-28) twice on the same problem: once with the reference's
sequential order and once with pairwise summation at the same precision (the
order class of the device's tree reductions). Test infrastructure / experiment
only; writes one JSON line per run.

    python tools/dot_order_experiment.py 5 [n]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

from oracle_bind import Oracle  # noqa: E402

from paper_2505_20719_b200 import problems  # noqa: E402

SPEC = "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > identity"

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
grid = int(sys.argv[2]) if len(sys.argv) > 2 else None
p = problems.problem(cfg, grid=grid)
o = Oracle()
for pairwise in (0, 1):
    o.lib.or_set_pairwise_dots(pairwise)
    t0 = time.time()
    r = o.solve((p.n, p.row_ptr, p.col_idx), p.values, SPEC, p.b, tol=1e-10)
    print(json.dumps({"config": cfg, "n": p.n, "nnz": p.nnz, "dots": "pairwise" if pairwise else "sequential",
                      "outer": r.outer_iterations, "res": r.final_true_residual, "hist": r.residual_history,
                      "seconds": round(time.time() - t0, 1)}), flush=True)
