"""Times the fp16-F3R solve with the reference bench's default primary
preconditioner (block-Jacobi IC(0)/ILU(0), 4 blocks, fp16 factors) beside the
M = identity solve, on one BASELINE config; per-kernel breakdown of one eager solve.

    python tools/precond_timing.py [--config 2] [--solves 3] [--kind ic0|ilu0]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--grid", type=int, default=0)
    ap.add_argument("--solves", type=int, default=3)
    ap.add_argument("--kind", default="ic0")
    ap.add_argument("--blocks", type=int, default=4)
    ap.add_argument("--apply-only", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import problems
    p = problems.problem(a.config, grid=a.grid) if a.grid else problems.problem(a.config)
    A = f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values)
    reps = f.make_replicas(A)
    sym = a.kind == "ic0"
    t0 = time.time()
    M = f.BlockJacobiIlu0.factorize(A, f.IluConfig(a.blocks, 1.0, sym, f.Precision.P16))
    t_fact = time.time() - t0
    spec = f"F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > {a.kind}(blocks={a.blocks},alpha=1,prec=f16)"
    out = {"config": a.config, "n": p.n, "nnz": p.nnz, "kind": a.kind, "blocks": a.blocks,
           "factorize_s_host": t_fact, "sweep_levels": M.sweep_levels()}
    # the apply alone: fp16 r -> fp16 z, as inside the Richardson level
    r = f.DenseVector(torch.from_numpy(p.b).cuda().half().contiguous())
    z = f.DenseVector(p.n, f.Precision.P16)
    for _ in range(3):
        M.apply(r, z)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        M.apply(r, z)
    e1.record()
    torch.cuda.synchronize()
    out["apply_ms"] = e0.elapsed_time(e1) / 20
    out["us_per_level"] = 1000 * out["apply_ms"] / (out["sweep_levels"][0] + out["sweep_levels"][1])
    if a.apply_only:
        print(json.dumps(out, indent=1))
        return
    b = torch.from_numpy(p.b).cuda()
    for label, m in (("identity", f.IdentityPrecond(p.n)), (a.kind, M)):
        s = f.build(f.parse_solver_spec(spec if m is M else spec.rsplit(">", 1)[0] + "> identity"), reps, m)
        times, rep = [], None
        for _ in range(a.solves + 1):
            s.reset()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            rep = s.run(b, f.RunOptions(tol=1e-10)).report
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        s.reset()
        s.set_profile(True)
        s.run(b, f.RunOptions(tol=1e-10))
        prof = sorted(s.profile(), key=lambda r: -r[1])
        out[label] = {"ms": sorted(times[1:])[len(times[1:]) // 2], "outer": rep.outer_iterations,
                      "residual": rep.final_true_residual, "precond_invocations": rep.precond_invocations,
                      "profile": [(n, round(ms, 3), ln) for n, ms, ln, _ in prof[:12]]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
