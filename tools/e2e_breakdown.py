"""Where the end-to-end (host buffers) time goes beyond the device solve, config 2."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_20719_b200 as f  # noqa: E402
from paper_2505_20719_b200 import problems  # noqa: E402

p = problems.problem(2)
reps = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values))
s = f.build(f.parse_solver_spec("F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > identity"), reps,
            f.IdentityPrecond(p.n))
o = f.RunOptions(tol=1e-10)
bd = torch.from_numpy(p.b).cuda()
bh = torch.from_numpy(p.b).pin_memory().numpy()
xh = torch.empty(p.n, dtype=torch.float64).pin_memory().numpy()
for _ in range(3):
    s.reset(); s.run(bd, o); s.reset(); s.run(bh, o, out=xh)
torch.cuda.synchronize()


def wall(fn, k=5):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    return np.median(ts)


print("device solve (wall)       %.3f ms" % wall(lambda: (s.reset(), s.run(bd, o))))
print("device solve, no x        %.3f ms" % wall(lambda: (s.reset(), s.run(bd, o, want_x=False))))
print("host solve (pinned b, x)  %.3f ms" % wall(lambda: (s.reset(), s.run(bh, o, out=xh))))
t = torch.empty(p.n, dtype=torch.float64, device="cuda")
print("H2D 16.8 MB pinned        %.3f ms" % wall(lambda: t.copy_(torch.from_numpy(bh), non_blocking=True)))
print("D2H 16.8 MB pinned        %.3f ms" % wall(lambda: torch.from_numpy(xh).copy_(t, non_blocking=True)))
r = s.run(bd, o)
print("report build              %.3f ms" % wall(lambda: s.innermost_omegas()))
