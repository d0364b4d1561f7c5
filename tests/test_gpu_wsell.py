"""The windowed SELL engine (csrc/wsell.cuh, engine 3) against the CPU oracle.

The engine keeps the reference's per-row arithmetic (one thread per row, entries in
stored order, src/csr.cpp:23-37) but moves the rows into a sliced, chunk-major
layout and serves the gathers from a shared-memory band of x, so every SpMV must
stay BIT-EXACT. The cases cover: every precision triple on the small problems;
a matrix whose columns sit exactly on the band's edges (first/last ring slot and
one past, for each ring width); config-5 rows at a size where every CTA slides its
band over several windows; empty and very long rows; Richardson call sequences
(plain calls bit-exact, update calls within tolerance); nested solves, with
sequential reductions bit-identical to the oracle's history.
"""
import numpy as np
import pytest

from _util import TOL, rand_vec, small_problems

pytestmark = pytest.mark.gpu

TRIPLES = [(pa, px, py) for pa in (0, 1, 2) for px in (0, 1, 2) for py in (0, 1, 2)]
SOME = [(0, 0, 0), (0, 1, 1), (0, 0, 1), (1, 1, 1), (2, 1, 2), (2, 2, 2), (0, 2, 0)]
# band half-widths W of the three ring widths (wsell.cuh: RN = 128 KB / element size,
# TW rows per window, W = (RN - 2 TW) / 2) for 2-, 4- and 8-byte ring elements
BANDS = (24576, 12288, 6144, 16384)  # + the packed fp16 stream's band (wsell_pk.cuh: 49,152-slot ring, 8192-row windows)


def _reps(f, n, rp, ci, va, monkeypatch, on="1"):
    monkeypatch.setenv("F3RG_WSELL", on)
    reps = f.make_replicas(f.SparseCsr(n, rp, ci, va))
    monkeypatch.delenv("F3RG_WSELL")
    return reps


def _check(f, oracle, reps, n, rp, ci, va, triples, seed=7, tag=""):
    a = (n, rp, ci)
    for pa, px, py in triples:
        x = rand_vec(oracle, px, n, seed + 3 * pa + px)
        y = f.DenseVector(n, py)
        f.spmv(reps.at(pa), f.DenseVector(x, px), y)
        want = oracle.spmv(a, oracle.round_vec(pa, va), pa, x, px, py)
        got = y.numpy()
        assert np.array_equal(got, want), (tag, pa, px, py, np.abs(got - want).max())


def test_engine_selection(cuda, monkeypatch):
    """irregular square matrices get the windowed engine by default; stencils keep
    the row tiles; F3RG_WSELL forces either way"""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import problems
    p5 = problems.problem(5, grid=6000)
    r5 = f.make_replicas(f.SparseCsr(p5.n, p5.row_ptr, p5.col_idx, p5.values))
    assert r5.engine() == 3
    p2 = problems.problem(2, grid=12)
    r2 = f.make_replicas(f.SparseCsr(p2.n, p2.row_ptr, p2.col_idx, p2.values))
    assert r2.engine() in (0, 1)
    assert _reps(f, p2.n, p2.row_ptr, p2.col_idx, p2.values, monkeypatch, "1").engine() == 3
    assert _reps(f, p5.n, p5.row_ptr, p5.col_idx, p5.values, monkeypatch, "0").engine() == 2


def test_all_triples_small_problems(cuda, oracle, monkeypatch):
    import paper_2505_20719_b200 as f
    for name, p in small_problems():
        reps = _reps(f, p.n, p.row_ptr, p.col_idx, p.values, monkeypatch)
        assert reps.engine() == 3
        _check(f, oracle, reps, p.n, p.row_ptr, p.col_idx, p.values, TRIPLES, tag=name)
        assert np.array_equal(reps.at(0).values(), oracle.round_vec(0, p.values)), name


def _band_edge_matrix(n):
    """rows i with columns i + d for d in 0, +-W, +-(W+1) of every ring width (clipped
    to [0, n)): the band's first and last slot and one past each, on every row of
    every window"""
    offs = sorted({0} | {s * d for w in BANDS for d in (w, w + 1, 2 * w + 8192, 2 * w + 8193) for s in (1, -1)})
    offs = np.array(offs, dtype=np.int64)
    rows = np.arange(n, dtype=np.int64)
    cols = rows[:, None] + offs[None, :]
    ok = (cols >= 0) & (cols < n)
    lens = ok.sum(1)
    rp = np.zeros(n + 1, np.uint32)
    rp[1:] = np.cumsum(lens)
    ci = cols[ok].astype(np.uint32)  # row-major, ascending within a row
    va = np.random.default_rng(1).uniform(-1, 1, ci.size)
    return rp, ci, va


def test_band_edges(cuda, oracle, monkeypatch):
    import paper_2505_20719_b200 as f
    n = 3_000_000  # ~20 windows of 8192 rows per CTA on 148 SMs
    rp, ci, va = _band_edge_matrix(n)
    reps = _reps(f, n, rp, ci, va, monkeypatch)
    _check(f, oracle, reps, n, rp, ci, va, SOME, tag="band-edges")


def test_config5_rows_sliding_band(cuda, oracle):
    """config-5 rows (log-normal lengths, +-N(0, 5000^2) band, 5 % long range) at
    n = 4e6: every CTA slides its band over several windows, and the fp64 ring
    (W = 6144) leaves a quarter of the entries to the far path"""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import problems
    p = problems.problem(5, grid=4_000_000)
    reps = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values))
    assert reps.engine() == 3
    _check(f, oracle, reps, p.n, p.row_ptr, p.col_idx, p.values, SOME, tag="config5@4e6")


def test_empty_and_long_rows(cuda, oracle, monkeypatch):
    import paper_2505_20719_b200 as f
    rng = np.random.default_rng(3)
    n = 9000
    lens = rng.integers(0, 40, n)
    lens[5] = 0
    lens[17] = 8999
    lens[18] = 5000
    lens[19] = 0
    lens[4096:6144] = 0  # a whole sort window of empty rows
    cols = [np.sort(rng.choice(n, size=min(L, n), replace=False)) for L in lens]
    rp = np.zeros(n + 1, np.uint32)
    rp[1:] = np.cumsum([len(c) for c in cols])
    ci = np.concatenate(cols).astype(np.uint32)
    va = rng.uniform(-1, 1, ci.size)
    reps = _reps(f, n, rp, ci, va, monkeypatch)
    _check(f, oracle, reps, n, rp, ci, va, TRIPLES, tag="ragged")


def test_richardson_sequence(cuda, oracle, monkeypatch):
    """130 richardson_apply calls on the windowed engine: plain calls (z1 held in
    the ring, fused sweep) bit-exact, update calls 64 and 128 within fp16 tolerance"""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import problems
    p = problems.problem(5, grid=30000)
    reps = _reps(f, p.n, p.row_ptr, p.col_idx, p.values, monkeypatch)
    assert reps.engine() == 3
    a = (p.n, p.row_ptr, p.col_idx)
    v16 = oracle.round_vec(0, p.values)
    st = f.RichardsonState(reps.a16, 2, 64)
    om = np.ones(2)
    cnt = [1, 0, 0]
    for call in range(1, 131):
        v = rand_vec(oracle, 0, p.n, 100 + call)
        z_ref, om_ref, cnt_ref = oracle.richardson_apply(a, v16, 0, 2, 64, om, cnt, v)
        zd = f.DenseVector(p.n, 0)
        f.richardson_apply(st, f.DenseVector(v, 0), zd)
        z = zd.numpy()
        w, counters = st._state()
        assert counters == cnt_ref, call
        if call % 64 == 0:
            assert np.allclose(w, om_ref, rtol=1e-5, atol=0), (call, w, om_ref)
            assert np.linalg.norm(z - z_ref) <= TOL[0] * np.linalg.norm(z_ref), call
            om, cnt = np.array(w), counters
        else:
            assert w == list(om_ref)
            assert np.array_equal(z, z_ref), (call, np.abs(z - z_ref).max())
            om, cnt = om_ref, cnt_ref


def test_seq_solve_matches_oracle(cuda, oracle, monkeypatch):
    """fp16-F3R on config-5 rows through the windowed engine with sequential
    reductions: the oracle's outer count, residual history and solution, bit for bit"""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import problems
    p = problems.problem(5, grid=20000)
    reps = _reps(f, p.n, p.row_ptr, p.col_idx, p.values, monkeypatch)
    spec = "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > identity"
    a = (p.n, p.row_ptr, p.col_idx)
    ref = oracle.solve(a, p.values, spec, p.b, tol=1e-10)
    with f.seq_reductions():
        solver = f.build(f.parse_solver_spec(spec), reps, f.IdentityPrecond(p.n))
        run = solver.run(p.b, f.RunOptions(tol=1e-10))
    rep = run.report
    assert rep.outer_iterations == ref.outer_iterations
    assert rep.residual_history == list(ref.residual_history)
    assert np.array_equal(run.x, ref.x)


def test_tree_solve_criteria(cuda, oracle, monkeypatch):
    """default (tree) reductions: converged to tol, outer count within +-10 % of the
    oracle's, for fp16-F3R and fp32-F3R"""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import problems
    p = problems.problem(5, grid=60000)
    reps = _reps(f, p.n, p.row_ptr, p.col_idx, p.values, monkeypatch)
    a = (p.n, p.row_ptr, p.col_idx)
    for spec in ("F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > identity",
                 "F100:f64/f64 > F8:f32/f32 > F4:f32/f32 > R2:f32,c=64 > identity"):
        ref = oracle.solve(a, p.values, spec, p.b, tol=1e-10)
        solver = f.build(f.parse_solver_spec(spec), reps, f.IdentityPrecond(p.n))
        rep = solver.run(p.b, f.RunOptions(tol=1e-10)).report
        assert rep.converged and rep.final_true_residual <= 1e-10, (spec, rep)
        assert abs(rep.outer_iterations - ref.outer_iterations) <= max(1, round(0.1 * ref.outer_iterations)), spec
