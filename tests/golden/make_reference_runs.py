"""Runs the UNMODIFIED reference (oracle/_ref/libf3r_ref.so, built from
/root/reference/proj/src) on the BASELINE.json configurations with the identity
primary preconditioner (SURVEY.md §8 scope decision) at tol 1e-10, and records
outer-iteration counts, residual histories and timings in reference_runs.json.

These are the outer-count oracle for the full-size configs and the denominator
of bench.py's reference-arm extrapolation. Test infrastructure only.

    python tests/golden/make_reference_runs.py 1 2 [3 4 5] [--mode=fp16-f3r-ic0,...]
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

from oracle_bind import Reference  # noqa: E402

from paper_2505_20719_b200 import problems  # noqa: E402

SPECS = {
    "fp16-f3r": "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > identity",
    "fp32-f3r": "F100:f64/f64 > F8:f32/f32 > F4:f32/f32 > R2:f32,c=64 > identity",
    "fp64-f3r": "F100:f64/f64 > F8:f64/f64 > F4:f64/f64 > R2:f64,c=64 > identity",
    # the reference bench's default primary preconditioner (include/f3r/bench.hpp:31-34,
    # src/bench.cpp:160-177): block-Jacobi IC(0) on symmetric problems, ILU(0)
    # otherwise, 4 blocks, alpha 1, factors at the Richardson precision
    "fp16-f3r-ic0": "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > ic0(blocks=4,alpha=1,prec=f16)",
    "fp16-f3r-ilu0": "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > ilu0(blocks=4,alpha=1,prec=f16)",
}
PRECOND = {"fp16-f3r-ic0": (4, 1.0, True, 0), "fp16-f3r-ilu0": (4, 1.0, False, 0)}
OUT = os.path.join(HERE, "reference_runs.json")


def main(configs, modes=("fp16-f3r",)):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    r = Reference()
    r.set_threads(os.cpu_count())
    for c in configs:
        p = problems.problem(int(c))
        m = r.matrix(p.row_ptr, p.col_idx, p.values)
        for mode in modes:
            t0 = time.time()
            M = r.ilu(m, *PRECOND[mode]) if mode in PRECOND else None
            rep = r.solve(m, SPECS[mode], p.b, tol=1e-10, want_x=False, precond=M)
            data[f"config{c}/{mode}"] = {
                "n": p.n, "nnz": p.nnz, "outer_iterations": rep.outer_iterations,
                "precond_invocations": rep.precond_invocations, "converged": rep.converged,
                "final_true_residual": rep.final_true_residual, "residual_history": rep.residual_history,
                "level_iterations": rep.level_iterations, "omegas_final": rep.omegas_final,
                "wall_seconds": rep.wall_seconds, "threads": r.max_threads(), "host": os.uname().nodename,
                "elapsed_incl_setup": time.time() - t0,
            }
            print(c, mode, rep.outer_iterations, rep.final_true_residual, rep.wall_seconds, flush=True)
            json.dump(data, open(OUT, "w"), indent=1)
        del m


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    modes = ("fp16-f3r", "fp32-f3r", "fp64-f3r") if "--all-modes" in sys.argv else ("fp16-f3r",)
    for a in sys.argv[1:]:
        if a.startswith("--mode="):
            modes = tuple(a[7:].split(","))
    main(args or ["1", "2"], modes)
