"""GPU parity of the block-Jacobi ILU(0)/IC(0) primary preconditioner
(reference src/ilu.cpp:38-263) and of the solves that use it, through the C ABI.

* apply: bit-exact against the oracle (pinned to the reference by
  tests/test_oracle_ilu.py) for every factor / input / output precision, ILU and
  IC, several block counts, on the five generator families -- the device sweeps
  change only the order rows are computed in, never a row's own arithmetic;
* repeated applies (the sweeps' epoch words cycle) and precision switches;
* Richardson with M: bit-exact on plain calls, the weight schedule as the oracle's;
* full nested solves with M: the reference's outer counts (±10 %), tol met;
* the reference bench's default configuration (IC(0), 4 blocks, fp16 factors) at
  BASELINE configs 1 and 2 against the UNMODIFIED reference's recorded runs."""
import json
import os

import numpy as np
import pytest

from _util import TOL as PTOL, normwise, rand_vec, small_problems

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
TOL = 1e-10


@pytest.fixture(scope="module")
def probs(cuda):
    return small_problems()


def _csr(p):
    import paper_2505_20719_b200 as f
    return f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values)


def _sym(name):
    return name in ("hpcg16", "poisson24", "aniso16")


def test_apply_bit_exact_all_precisions(probs, oracle):
    import paper_2505_20719_b200 as f
    for name, p in probs:
        a = (p.n, p.row_ptr, p.col_idx)
        for sym in ((True, False) if _sym(name) else (False,)):
            for nb in (1, 4, 9):
                for pf in (0, 1, 2):
                    M = f.BlockJacobiIlu0.factorize(_csr(p), f.IluConfig(nb, 1.0, sym, f.Precision(pf)))
                    O = oracle.ilu(a, p.values, nb, 1.0, sym, pf)
                    for pr in (0, 1, 2):
                        r = rand_vec(oracle, pr, p.n, 7 + pr + 3 * nb)
                        for pz in (0, 1, 2):
                            z = f.DenseVector(p.n, f.Precision(pz))
                            M.apply(f.DenseVector(r, f.Precision(pr)), z)
                            want = O.apply(r, pr, pz)
                            got = z.numpy()
                            assert np.array_equal(got, want), (name, sym, nb, pf, pr, pz,
                                                               np.abs(got - want).max())


def test_apply_repeated_and_switching(probs, oracle):
    """200 applies cycle the epoch words; switching the compute precision clears
    the cells; every result stays bit-exact."""
    import paper_2505_20719_b200 as f
    name, p = probs[0]
    a = (p.n, p.row_ptr, p.col_idx)
    M = f.BlockJacobiIlu0.factorize(_csr(p), f.IluConfig(4, 1.0, True, f.Precision.P16))
    O = oracle.ilu(a, p.values, 4, 1.0, True, 0)
    for it in range(200):
        pr = 0 if it % 50 < 45 else 2  # mostly fp16 (C = f16), some fp64 inputs (C = f64)
        r = rand_vec(oracle, pr, p.n, 1000 + it)
        z = f.DenseVector(p.n, f.Precision(pr))
        M.apply(f.DenseVector(r, f.Precision(pr)), z)
        assert np.array_equal(z.numpy(), O.apply(r, pr, pr)), it


def test_apply_across_epoch_skip(probs, oracle, monkeypatch):
    """the epoch tags skip multiples of 2^16 (so zeroed cells never look current);
    the frontier hint counts launches separately, so applies that cross the skip --
    reached after ~65k applies by a long-lived solver -- stay correct (and do not
    hang). F3RG_SWEEP_EPOCH0 starts the tags just below the skip."""
    import paper_2505_20719_b200 as f
    monkeypatch.setenv("F3RG_SWEEP_EPOCH0", str(65536 - 3))
    name, p = probs[0]
    a = (p.n, p.row_ptr, p.col_idx)
    M = f.BlockJacobiIlu0.factorize(_csr(p), f.IluConfig(4, 1.0, True, f.Precision.P16))
    O = oracle.ilu(a, p.values, 4, 1.0, True, 0)
    for it in range(8):
        r = rand_vec(oracle, 0, p.n, 500 + it)
        z = f.DenseVector(p.n, f.Precision.P16)
        M.apply(f.DenseVector(r, f.Precision.P16), z)
        assert np.array_equal(z.numpy(), O.apply(r, 0, 0)), it


def test_sweep_depth_matches_stencil_levels(cuda):
    """27-point lexicographic 16^3, 4 blocks of 4 planes: forward depth x + 2y + 4z + 1."""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import problems
    p = problems.problem(2, grid=16)
    M = f.BlockJacobiIlu0.factorize(_csr(p), f.IluConfig(4, 1.0, True, f.Precision.P16))
    fwd, bwd = M.sweep_levels()
    assert fwd == 15 + 2 * 15 + 4 * 3 + 1 and bwd == fwd
    assert M.block_ranges() == [0, 1024, 2048, 3072, 4096]


def test_factorization_errors_surface(cuda):
    import paper_2505_20719_b200 as f
    with pytest.raises(f.FactorizationError, match="non-positive pivot in block 0, row 1"):
        f.BlockJacobiIlu0.factorize(f.SparseCsr(2, [0, 2, 4], [0, 1, 0, 1], [1.0, 2.0, 2.0, 1.0]),
                                    f.IluConfig(1, 1.0, True))
    with pytest.raises(f.FactorizationError, match="lost the diagonal of row 0"):
        f.BlockJacobiIlu0.factorize(f.SparseCsr(1, [0, 1], [0], [1e-9]), f.IluConfig(1, 1.0, False, f.Precision.P16))


@pytest.mark.parametrize("prec", [0, 1])
def test_richardson_with_m_sequence(cuda, oracle, prec):
    """130 calls of richardson_apply on (A, M = IC(0)): plain calls bit-exact, update
    calls (64, 128) within the tolerance of their tree-ordered fp32 dots."""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import problems
    p = problems.problem(2, grid=16)
    reps = f.make_replicas(_csr(p))
    a = (p.n, p.row_ptr, p.col_idx)
    vp = oracle.round_vec(prec, p.values)
    M = f.BlockJacobiIlu0.factorize(_csr(p), f.IluConfig(4, 1.0, True, f.Precision(prec)))
    O = oracle.ilu(a, p.values, 4, 1.0, True, prec)
    st = f.RichardsonState(reps.at(f.Precision(prec)), 2, 64)
    om, cnt = np.ones(2), [1, 0, 0]
    for call in range(1, 131):
        v = rand_vec(oracle, prec, p.n, 500 + call)
        z_ref, om_ref, cnt_ref = oracle.richardson_apply(a, vp, prec, 2, 64, om, cnt, v, precond=O)
        zd = f.DenseVector(p.n, f.Precision(prec))
        f.richardson_apply(st, f.DenseVector(v, f.Precision(prec)), zd, M)
        z = zd.numpy()
        w, counters = st._state()
        assert counters == cnt_ref, call
        if call % 64 == 0:
            assert np.allclose(w, om_ref, rtol=1e-5, atol=0), (call, w, om_ref)
            assert normwise(z, z_ref) <= PTOL[prec], call
            om, cnt = np.array(w), counters
        else:
            assert w == list(om_ref)
            assert np.array_equal(z, z_ref), (call, np.abs(z - z_ref).max())
            om, cnt = om_ref, cnt_ref


SPECS_M = [
    ("F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > ic0(blocks=4,prec=f16)", 4, 0),
    ("F100:f64/f64 > F8:f32/f32 > F4:f32/f32 > R2:f32,c=64 > ilu0(blocks=3,prec=f32)", 3, 1),
    ("F30:f64/f64 > ilu0(blocks=3,prec=f64)", 3, 2),
    ("F100:f64/f64 > F8:f32/f32 > ic0(blocks=2,prec=f16)", 2, 0),
]


@pytest.mark.parametrize("spec,nb,prec", SPECS_M, ids=["f3r16-ic0", "f3r32-ilu0", "fgmres-ilu0", "f2-ic0"])
def test_solves_with_m_match_oracle(probs, oracle, spec, nb, prec):
    import paper_2505_20719_b200 as f
    for name, p in probs:
        sym = "ic0" in spec and _sym(name)
        a = (p.n, p.row_ptr, p.col_idx)
        M = f.BlockJacobiIlu0.factorize(_csr(p), f.IluConfig(nb, 1.0, sym, f.Precision(prec)))
        O = oracle.ilu(a, p.values, nb, 1.0, sym, prec)
        s = f.build(f.parse_solver_spec(spec), f.make_replicas(_csr(p)), M)
        rep = s.run(p.b, f.RunOptions(tol=TOL)).report
        ref = oracle.solve(a, p.values, spec, p.b, tol=TOL, precond=O)
        assert rep.converged == ref.converged, name
        if ref.converged:
            assert rep.final_true_residual <= TOL, (name, rep.final_true_residual)
        assert abs(rep.outer_iterations - ref.outer_iterations) <= max(1, round(0.1 * ref.outer_iterations)), \
            (name, spec, rep.outer_iterations, ref.outer_iterations)
        assert rep.precond_invocations == rep.level_iterations[-1] or "R2" not in spec
        for a_, b_ in zip(rep.residual_history[1:], ref.residual_history[1:]):
            if max(a_, b_) < 1e-11:
                continue
            assert abs(np.log10(a_) - np.log10(b_)) <= 1.0, (name, rep.residual_history, ref.residual_history)


def test_solves_match_reference_golden(cuda):
    """the committed runs of the UNMODIFIED reference (tests/golden/reference_ilu.npz)"""
    import paper_2505_20719_b200 as f
    g = np.load(os.path.join(HERE, "golden", "reference_ilu.npz"))
    rp, ci, vs = g["mat4_0_rp"], g["mat4_0_ci"], g["mat4_0_vals"]
    a = f.SparseCsr(len(rp) - 1, rp, ci, vs)
    for i, spec in enumerate(g["solve_specs"]):
        nb, sym, prec = (int(v) for v in g[f"solve{i}_m"])
        M = f.BlockJacobiIlu0.factorize(a, f.IluConfig(nb, 1.0, bool(sym), f.Precision(prec)))
        rep = f.build(f.parse_solver_spec(str(spec)), f.make_replicas(a), M).run(g["solve_b"],
                                                                               f.RunOptions(tol=TOL)).report
        conv, outer, pinv, final = g[f"solve{i}_meta"]
        assert rep.converged == bool(conv)
        assert abs(rep.outer_iterations - int(outer)) <= max(1, round(0.1 * outer)), (spec, rep.outer_iterations,
                                                                                       outer)
        assert rep.final_true_residual <= TOL


def test_create_from_spec_terminal(cuda, oracle):
    """f3rg_solver_create with precond_kind IC0: factorised from the spec terminal"""
    import ctypes as C
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import problems
    p = problems.problem(2, grid=16)
    reps = f.make_replicas(_csr(p))
    spec = "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > ic0(blocks=4,prec=f16)"
    h = C.c_void_p()
    L = f.lib()
    assert L.f3rg_solver_create(C.byref(h), reps.dev.h, spec.encode(), 1) == 0, L.f3rg_last_error()
    r = f._Report()
    b = np.ascontiguousarray(p.b)
    x = np.zeros(p.n)
    assert L.f3rg_solve(h, b.ctypes.data, x.ctypes.data, C.byref(f.RunOptions(tol=TOL)._c()), C.byref(r)) == 0
    L.f3rg_solver_destroy(h)
    O = oracle.ilu((p.n, p.row_ptr, p.col_idx), p.values, 4, 1.0, True, 0)
    ref = oracle.solve((p.n, p.row_ptr, p.col_idx), p.values, spec, p.b, tol=TOL, precond=O)
    assert r.converged and r.outer_iterations == ref.outer_iterations


def _recorded(key):
    d = json.load(open(os.path.join(HERE, "golden", "reference_runs.json")))
    if key not in d:
        pytest.skip(f"{key} not recorded")
    return d[key]


@pytest.mark.parametrize("cfg,kind", [(1, "ic0"), (2, "ic0"), (3, "ilu0"), (5, "ilu0")])
def test_bench_default_m_vs_reference_run(cuda, cfg, kind):
    """BASELINE configs with the reference bench's default M (IC(0) on the symmetric
    ones, ILU(0) otherwise; 4 blocks, fp16) against the UNMODIFIED reference's
    recorded full runs (tests/golden/reference_runs.json)"""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import problems
    ref = _recorded(f"config{cfg}/fp16-f3r-{kind}")
    p = problems.problem(cfg)
    spec = f"F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > {kind}(blocks=4,alpha=1,prec=f16)"
    M = f.BlockJacobiIlu0.factorize(_csr(p), f.IluConfig(4, 1.0, kind == "ic0", f.Precision.P16))
    rep = f.build(f.parse_solver_spec(spec), f.make_replicas(_csr(p)), M).run(p.b, f.RunOptions(tol=TOL)).report
    assert rep.converged and rep.final_true_residual <= TOL
    assert abs(rep.outer_iterations - ref["outer_iterations"]) <= max(1, round(0.1 * ref["outer_iterations"]))
