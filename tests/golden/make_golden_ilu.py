"""Golden vectors for the block-Jacobi ILU(0)/IC(0) primary preconditioner
(reference src/ilu.cpp:38-263), generated from the UNMODIFIED reference library
(oracle/_ref/libf3r_ref.so, built from /root/reference/proj/src by oracle/Makefile).
They pin the C restatement (oracle/f3r_oracle.c or_ilu_*) on machines where the
reference is absent.

    python tests/golden/make_golden_ilu.py   ->  tests/golden/reference_ilu.npz
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_bind import FactorizationFailed, Reference  # noqa: E402

# (grid, beta, symmetric, nblocks, prec, alpha): IC only on the symmetric stencil
FACTORS = [
    (3, 0.0, 1, 4, 0, 1.0), (3, 0.0, 0, 4, 0, 1.0), (3, 0.5, 0, 3, 0, 1.0), (3, 0.5, 0, 1, 1, 1.3),
    (3, 0.0, 1, 7, 2, 1.0), (3, 0.5, 0, 5, 2, 1.1), (4, 0.0, 1, 2, 1, 1.0),
]
SOLVE_SPECS = [
    "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > ic0(blocks=4,prec=f16)",
    "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > ilu0(blocks=4,prec=f16)",
    "F100:f64/f64 > F8:f32/f32 > F4:f32/f32 > R2:f32,c=64 > ic0(blocks=4,prec=f32)",
    "F30:f64/f64 > ilu0(blocks=3,prec=f64)",
    "F100:f64/f64 > F8:f32/f32 > ic0(blocks=2,prec=f16)",
]
ERRORS = [  # (n, row_ptr, col_idx, vals, symmetric, prec) -> message
    (2, [0, 1, 2], [1, 0], [1.0, 1.0], 0, 2),
    (2, [0, 2, 4], [0, 1, 0, 1], [1.0, 2.0, 2.0, 1.0], 1, 2),
    (1, [0, 1], [0], [1e-9], 0, 0),
    (1, [0, 1], [0], [1e6], 1, 0),
]


def scaled_stencil(r, l, beta):
    rp, ci, va = r.generate_stencil(l, l, l, beta)
    vs, _, _ = r.diagonal_scale(rp, ci, va)
    return rp, ci, vs


def main():
    r = Reference()
    out = {}
    rng = np.random.default_rng(20261020)
    for (l, beta) in ((3, 0.0), (3, 0.5), (4, 0.0)):  # the matrices, so the oracle tests need no reference
        rp, ci, vs = scaled_stencil(r, l, beta)
        key = f"mat{l}_{int(beta * 10)}"
        out[key + "_rp"], out[key + "_ci"], out[key + "_vals"] = rp, ci, vs
    for i, (l, beta, sym, nb, prec, alpha) in enumerate(FACTORS):
        rp, ci, vs = scaled_stencil(r, l, beta)
        n = len(rp) - 1
        m = r.matrix(rp, ci, vs)
        M = r.ilu(m, nb, alpha, sym, prec)
        out[f"f{i}_cfg"] = np.array([l, beta, sym, nb, prec, alpha])
        for pr in (0, 1, 2):
            x = r.copy(rng.uniform(-1, 1, n), 2, pr)
            out[f"f{i}_r{pr}"] = x
            for pz in (0, 1, 2):
                out[f"f{i}_z{pr}{pz}"] = M.apply(x, pr, pz)
    # a Richardson call sequence with M (updates at calls 64 and 128), fp16 and fp32
    rp, ci, vs = scaled_stencil(r, 3, 0.0)
    n = len(rp) - 1
    m = r.matrix(rp, ci, vs)
    for p in (0, 1):
        M = r.ilu(m, 4, 1.0, 1, p)
        st = r.richardson(2, 64)
        zs = []
        for call in range(130):
            v = r.copy(np.random.default_rng(3000 + call).uniform(-1, 1, n), 2, p)
            zs.append(st.apply(m, p, v, precond=M))
        om, cnt = st.state()
        out[f"rich{p}_z_last"], out[f"rich{p}_z_64"] = zs[-1], zs[63]
        out[f"rich{p}_omegas"], out[f"rich{p}_counters"] = om, np.array(cnt, dtype=np.uint64)
    # full composed solves on the scaled 16^3 HPCG stencil, M from the spec terminal
    rp, ci, vs = scaled_stencil(r, 4, 0.0)
    m = r.matrix(rp, ci, vs)
    b = np.random.default_rng(7).uniform(-1, 1, len(rp) - 1)
    out["solve_b"] = b
    for i, spec in enumerate(SOLVE_SPECS):
        term = spec.split(">")[-1].strip()
        sym = term.startswith("ic0")
        nb = int(term.split("blocks=")[1].split(",")[0])
        prec = {"f16": 0, "f32": 1, "f64": 2}[term.split("prec=")[1].rstrip(")")]
        M = r.ilu(m, nb, 1.0, sym, prec)
        rep = r.solve(m, spec, b, tol=1e-10, precond=M)
        out[f"solve{i}_hist"] = np.array(rep.residual_history)
        out[f"solve{i}_x"] = rep.x
        out[f"solve{i}_meta"] = np.array([rep.converged, rep.outer_iterations, rep.precond_invocations,
                                          rep.final_true_residual])
        out[f"solve{i}_levels"] = np.array(rep.level_iterations, dtype=np.uint64)
        out[f"solve{i}_omegas"] = np.array(rep.omegas_final)
        out[f"solve{i}_m"] = np.array([nb, sym, prec])
    out["solve_specs"] = np.array(SOLVE_SPECS)
    msgs = []
    for (n, rp, ci, va, sym, prec) in ERRORS:
        mm = r.matrix(np.array(rp, np.uint32), np.array(ci, np.uint32), np.array(va))
        try:
            r.ilu(mm, 1, 1.0, sym, prec)
            msgs.append("")
        except FactorizationFailed as e:
            msgs.append(str(e))
    out["error_msgs"] = np.array(msgs)
    path = os.path.join(HERE, "reference_ilu.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
