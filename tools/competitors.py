"""fp16-F3R against the reference's fp64 competitor solvers on the device, BASELINE
configs: outer/iteration counts and time-to-solution (the paper's comparison, on
B200). CG, BiCGStab, FGMRES(64) (fgmres_restarted) and fp16-F3R, each with
M = identity and with the reference bench's block-Jacobi default
(IC(0) on symmetric problems, ILU(0) otherwise; 4 blocks; fp16 factors for F3R,
fp64 for the fp64 solvers, as src/bench.cpp:171-177 resolves them).

    python tools/competitors.py [configs...]      (default: 1 2 3 4)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_20719_b200 as f  # noqa: E402
from paper_2505_20719_b200 import problems  # noqa: E402

SPEC = "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > identity"
TOL = 1e-10
for cfg in [int(c) for c in sys.argv[1:]] or [1, 2, 3, 4]:
    p = problems.problem(cfg)
    reps = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values))
    out = {"config": cfg, "n": p.n, "nnz": p.nnz}
    s = f.build(f.parse_solver_spec(SPEC), reps, f.IdentityPrecond(p.n))
    b = torch.from_numpy(p.b).cuda()
    for _ in range(2):
        s.reset(); s.run(b, f.RunOptions(tol=TOL))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.reset(); r = s.run(b, f.RunOptions(tol=TOL), want_x=False).report
    torch.cuda.synchronize()
    out["f3r16"] = {"outer": r.outer_iterations, "res": r.final_true_residual, "s": time.perf_counter() - t0}
    for name, solve in (("cg", f.cg_solve), ("bicgstab", f.bicgstab_solve)):
        if name == "cg" and cfg in (3, 5):
            continue  # non-symmetric
        solve(reps, f.IdentityPrecond(p.n), p.b, f.ReferenceSolveOptions(tol=TOL))  # warm-up
        t0 = time.perf_counter()
        k = solve(reps, f.IdentityPrecond(p.n), p.b, f.ReferenceSolveOptions(tol=TOL))
        out[name] = {"iterations": k.outer_iterations, "converged": k.converged, "flag": k.flag,
                     "res": k.final_true_residual, "s": time.perf_counter() - t0}
    # FGMRES(64), and both solvers with the bench-default block-Jacobi M
    sym = cfg in (1, 2, 4)
    kind = "ic0" if sym else "ilu0"
    a = f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values)
    M64 = f.BlockJacobiIlu0.factorize(a, f.IluConfig(4, 1.0, sym, f.Precision.P64))
    for name, solve in (("cg", f.cg_solve), ("bicgstab", f.bicgstab_solve)):
        if name == "cg" and not sym:
            continue
        solve(reps, M64, p.b, f.ReferenceSolveOptions(tol=TOL))  # warm-up
        t0 = time.perf_counter()
        k = solve(reps, M64, p.b, f.ReferenceSolveOptions(tol=TOL))
        out[f"{name}/{kind}"] = {"iterations": k.outer_iterations, "converged": k.converged, "flag": k.flag,
                                 "res": k.final_true_residual, "s": time.perf_counter() - t0}
    for label, M in (("identity", f.IdentityPrecond(p.n)), (kind, M64)):
        f.fgmres_restarted(reps, M, p.b, 64, f.FgmresOptions(tol=TOL))  # warm-up
        t0 = time.perf_counter()
        k = f.fgmres_restarted(reps, M, p.b, 64, f.FgmresOptions(tol=TOL))
        out[f"fgmres64/{label}"] = {"iterations": k.outer_iterations, "converged": k.converged, "flag": k.flag,
                                    "res": k.final_true_residual, "s": time.perf_counter() - t0}
    M16 = f.BlockJacobiIlu0.factorize(a, f.IluConfig(4, 1.0, sym, f.Precision.P16))
    spec_m = SPEC.rsplit(">", 1)[0] + f"> {kind}(blocks=4,alpha=1,prec=f16)"
    sm = f.build(f.parse_solver_spec(spec_m), reps, M16)
    sm.reset(); sm.run(b, f.RunOptions(tol=TOL))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sm.reset(); r = sm.run(b, f.RunOptions(tol=TOL), want_x=False).report
    torch.cuda.synchronize()
    out[f"f3r16/{kind}"] = {"outer": r.outer_iterations, "res": r.final_true_residual, "s": time.perf_counter() - t0}
    print(json.dumps(out), flush=True)
