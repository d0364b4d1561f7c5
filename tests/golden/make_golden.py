"""Generates the golden vectors in tests/golden/*.npz from the UNMODIFIED reference
(oracle/_ref/libf3r_ref.so, compiled from /root/reference/proj/src by oracle/Makefile).
The reference ships no golden files (its tests regenerate fixtures from SplitMix64
seeds); these pin our C restatement (oracle/f3r_oracle.c) to it bit-for-bit, so
the oracle can be trusted on machines where the reference is absent (GPU box).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

from oracle_bind import Reference  # noqa: E402

SPECS = [
    "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > identity",
    "F100:f64/f64 > F8:f32/f32 > F4:f32/f32 > R2:f32,c=64",
    "F100:f64/f64 > F8:f64/f64 > F4:f64/f64 > R2:f64,c=64",
    "F100:f64/f64 > F64:f16/f16",
    "F16:f64/f64",
    "R2:f64,c=3",
    "F10:f64/f64 > R3:f16,c=2,omega=0.7",
    "F2:f64/f64 > F2:f64/f64",
]

SPEC_STRINGS = [
    "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > ilu0(blocks=8,alpha=1.0,prec=f16)",
    "F100:f64/f64>F8:f32/f32 >F4:f16/f32>R2:f16 , c = 64>identity",
    "R2:f16,c=0,omega=0.75",
    "F8:f32/f32 > ic0",
    "F8:f32/f32 > ilu0()",
    "F8:f32/f32 > ilu0(prec=f32, blocks=3)",
    "F8:f32/f32 > ic0(alpha=1.5)",
    "R1:f64,omega=1e-3",
    "F16:f64/f64",
]
BAD_SPECS = ["", "F8", "F8:f32", "F0:f64/f64", "F8:f31/f32", "X8:f64/f64", "F8:f64/f64 > identity > F2:f32/f32",
             "R2:f16,q=3", "F8:f64/f64 >> F2:f32/f32", "F-1:f64/f64", "R2:f16,c=-1", "ilu0(blocks=2)",
             "F8:f64/f64 > ilu0(foo=1)", "F8:f64/f64 > ilu0 blocks", "R2:f16,omega=abc"]


def scaled_stencil(r, l, beta):
    rp, ci, va = r.generate_stencil(l, l, l, beta)
    vs, _, _ = r.diagonal_scale(rp, ci, va)
    return rp, ci, vs


def main():
    r = Reference()
    rng = np.random.default_rng(20260519)
    out = {}
    # ---- binary16: exhaustive decode + targeted demotions
    out["half_decode"] = np.array([r.lib.ref_float_from_half(b) for b in range(65536)], dtype=np.float32)
    probes = np.concatenate([
        rng.uniform(-70000, 70000, 2000), rng.uniform(-1e-4, 1e-4, 2000), rng.standard_normal(2000),
        np.array([65504, 65519.99, 65520, 65536, 6e-8, 5.960464477539063e-08, 2.9802322387695312e-08, 1e-9,
                  0.0, -0.0, 1.0, 1 + 2 ** -11, 1 + 3 * 2 ** -11, 2049.0, 2051.0, np.inf, -np.inf]),
    ])
    out["half_probe_in"] = probes
    out["half_from_double"] = np.array([r.lib.ref_half_from_double(float(x)) for x in probes], dtype=np.uint16)
    out["half_from_float"] = np.array([r.lib.ref_half_from_float(np.float32(x)) for x in probes], dtype=np.uint16)

    # ---- kernels on the scaled HPGMP 8^3 stencil (non-symmetric, 512 rows)
    rp, ci, vs = scaled_stencil(r, 3, 0.5)
    n = len(rp) - 1
    m = r.matrix(rp, ci, vs)
    out["k_rp"], out["k_ci"], out["k_vals"] = rp, ci, vs
    for p in (0, 1, 2):
        out[f"k_replica{p}"] = r.replica_values(m, p, len(ci))
    xs = {}
    for p in (0, 1, 2):
        xs[p] = r.copy(rng.uniform(-2, 2, n), 2, p)  # exactly representable at p
        out[f"k_x{p}"] = xs[p]
        out[f"k_y{p}"] = r.copy(rng.uniform(-2, 2, n), 2, p)
    for pa in (0, 1, 2):
        for px in (0, 1, 2):
            for py in (0, 1, 2):
                out[f"spmv_{pa}{px}{py}"] = r.spmv(m, pa, xs[px], px, py)
    alpha = -0.6180339887498949
    for px in (0, 1, 2):
        for py in (0, 1, 2):
            x, y = out[f"k_x{px}"], out[f"k_y{py}"]
            out[f"dot_{px}{py}"] = np.array([r.dot(x, px, y, py, fl) for fl in (0, 1, 2)])
            out[f"axpy_{px}{py}"] = r.axpy(alpha, x, px, y, py)
            out[f"copy_{px}{py}"] = r.copy(x, px, py)
            for po in (0, 1, 2):
                out[f"add_scaled_{px}{py}{po}"] = r.add_scaled(x, px, alpha, y, py, po)
        out[f"norm2_{px}"] = np.array([r.norm2(out[f"k_x{px}"], px)])
        out[f"scale_{px}"] = r.scale(alpha, out[f"k_x{px}"], px)

    # ---- Richardson state over 130 calls (updates at 64 and 128), fp16 and fp64
    for p in (0, 2):
        st = r.richardson(2, 64)
        zs = []
        for call in range(130):
            v = r.copy(np.random.default_rng(1000 + call).uniform(-1, 1, n), 2, p)
            zs.append(st.apply(m, p, v))
        om, cnt = st.state()
        out[f"rich{p}_z_last"] = zs[-1]
        out[f"rich{p}_z_64"] = zs[63]
        out[f"rich{p}_omegas"] = om
        out[f"rich{p}_counters"] = np.array(cnt, dtype=np.uint64)
        out[f"rich{p}_log"] = st.log()

    # ---- fgmres_cycle per working precision
    b = rng.uniform(0, 1, n)
    for pw in (0, 1, 2):
        bp = r.copy(b, 2, pw)
        x, it, est, flags = r.fgmres_cycle(m, pw, pw, bp, np.zeros(n), 12, None, True)
        out[f"cycle{pw}_x"], out[f"cycle{pw}_est"] = x, est
        out[f"cycle{pw}_meta"] = np.array([it, *flags])

    # ---- full composed solves on the scaled 16^3 HPCG stencil (seeded rhs)
    rp2, ci2, vs2 = scaled_stencil(r, 4, 0.0)
    m2 = r.matrix(rp2, ci2, vs2)
    b2 = np.random.default_rng(7).uniform(-1, 1, len(rp2) - 1)
    out["solve_b"] = b2
    for i, spec in enumerate(SPECS):
        opts = dict(tol=1e-10)
        if spec.startswith("F2:"):
            opts = dict(tol=1e-300, max_outer_restarts=3, max_outer_total=300)
        rep = r.solve(m2, spec, b2, **opts)
        out[f"solve{i}_hist"] = np.array(rep.residual_history)
        out[f"solve{i}_x"] = rep.x
        out[f"solve{i}_meta"] = np.array([rep.converged, rep.outer_iterations, rep.precond_invocations,
                                          rep.final_true_residual])
        out[f"solve{i}_levels"] = np.array(rep.level_iterations, dtype=np.uint64)
        out[f"solve{i}_omegas"] = np.array(rep.omegas_final)
        out[f"solve{i}_flag"] = np.array(rep.flag)
    out["solve_specs"] = np.array(SPECS)

    # ---- spec grammar: canonical forms and rejections
    out["spec_in"] = np.array(SPEC_STRINGS)
    out["spec_canonical"] = np.array([r.spec_canonical(s) for s in SPEC_STRINGS])
    bad_ok = []
    for s in BAD_SPECS:
        try:
            r.spec_canonical(s)
            bad_ok.append(1)
        except RuntimeError:
            bad_ok.append(0)
    out["spec_bad"] = np.array(BAD_SPECS)
    out["spec_bad_accepted"] = np.array(bad_ok)

    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
