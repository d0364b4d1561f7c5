"""GPU parity of the kernel-level entry points against the CPU oracle (the plain-C
restatement, itself pinned bit-for-bit to the reference in test_oracle_golden.py).

Bars (BASELINE.json north_star): SpMV and every element-wise kernel are
BIT-EXACT (same per-row order, no FMA, same rounding); reductions (dot, norm2)
differ only by summation order and must agree within the normwise tolerance of
their accumulation precision (1e-12 fp64, 1e-5 fp32, 2e-3 fp16).
"""
import numpy as np
import pytest

from _util import TOL, rand_vec, small_problems

pytestmark = pytest.mark.gpu

PRECS = (0, 1, 2)


@pytest.fixture(scope="module")
def probs(cuda):
    import paper_2505_20719_b200 as f
    out = []
    for name, p in small_problems():
        reps = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values))
        out.append((name, p, reps))
    return out


def test_replicas_are_rne_demotions(probs, oracle):
    for name, p, reps in probs:
        for prec in PRECS:
            dev = reps.at(prec).values()
            assert np.array_equal(dev, oracle.round_vec(prec, p.values)), (name, prec)


@pytest.mark.parametrize("pa", PRECS)
def test_spmv_bit_exact_all_precisions(probs, oracle, pa):
    import paper_2505_20719_b200 as f
    for name, p, reps in probs:
        a = (p.n, p.row_ptr, p.col_idx)
        vals = oracle.round_vec(pa, p.values)
        for px in PRECS:
            x = rand_vec(oracle, px, p.n, 7 + px)
            for py in PRECS:
                want = oracle.spmv(a, vals, pa, x, px, py)
                y = f.DenseVector(p.n, py)
                f.spmv(reps.at(pa), f.DenseVector(x, px), y)
                got = y.numpy()
                assert np.array_equal(got, want), (name, pa, px, py, np.abs(got - want).max())


@pytest.mark.parametrize("shape", ["0", "1", "2"])
@pytest.mark.parametrize("columns", ["u32", "d16"])
def test_spmv_both_column_streams(cuda, oracle, columns, shape, monkeypatch):
    """the u32 index stream and the 16-bit delta stream (D16) give identical bits,
    with the regular, the short-row and the gather-bound tile shape (spmv.cuh TileCfg)"""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import problems
    if columns == "u32":
        monkeypatch.setenv("F3RG_COLUMNS", "u32")
    monkeypatch.setenv("F3RG_SHAPE", shape)
    p = problems.problem(4, grid=20)
    reps = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values))
    a = (p.n, p.row_ptr, p.col_idx)
    for pa, px, py in [(0, 0, 0), (0, 1, 1), (1, 1, 1), (2, 2, 2), (2, 1, 2), (0, 2, 0)]:
        x = rand_vec(oracle, px, p.n, 3 + pa)
        y = f.DenseVector(p.n, py)
        f.spmv(reps.at(pa), f.DenseVector(x, px), y)
        assert np.array_equal(y.numpy(), oracle.spmv(a, oracle.round_vec(pa, p.values), pa, x, px, py)), (pa, px, py)


def test_spmv_long_rows_and_empty_rows(cuda, oracle):
    """rows longer than a shared-memory tile and empty rows (CSR edge cases), on
    every column stream (u32, D16 and, for fp16, P16)"""
    import paper_2505_20719_b200 as f
    rng = np.random.default_rng(3)
    n = 9000
    lens = rng.integers(0, 40, n)
    lens[5] = 0
    lens[17] = 8999  # longer than every tile capacity (TNNZ <= 7168)
    lens[18] = 5000  # longer than an fp64 tile only
    lens[19] = 0
    rows, cols = [], []
    for i, L in enumerate(lens):
        c = np.sort(rng.choice(n, size=min(L, n), replace=False))
        cols.append(c)
    rp = np.zeros(n + 1, np.uint32)
    rp[1:] = np.cumsum([len(c) for c in cols])
    ci = np.concatenate(cols).astype(np.uint32)
    va = rng.uniform(-1, 1, ci.size)
    a = (n, rp, ci)
    import os
    for fmt, shape, srt in (("", "0", "0"), ("d16", "0", "0"), ("u32", "0", "0"), ("", "1", "0"),
                            ("u32", "1", "0"), ("", "0", "1"), ("u32", "1", "1"), ("", "2", "1"),
                            ("u32", "2", "0")):
        os.environ["F3RG_COLUMNS"] = fmt
        os.environ["F3RG_SHAPE"] = shape  # regular / short-row tiles
        os.environ["F3RG_SORT_ROWS"] = srt  # matrix row order / row-sorted stream
        try:
            reps = f.make_replicas(f.SparseCsr(n, rp, ci, va))
        finally:
            os.environ.pop("F3RG_COLUMNS")
            os.environ.pop("F3RG_SHAPE")
            os.environ.pop("F3RG_SORT_ROWS")
        for pa in PRECS:
            vals = oracle.round_vec(pa, va)
            for px, py in ((pa, pa), (0, 1), (2, 2)):
                x = rand_vec(oracle, px, n, 11)
                y = f.DenseVector(n, py)
                f.spmv(reps.at(pa), f.DenseVector(x, px), y)
                assert np.array_equal(y.numpy(), oracle.spmv(a, vals, pa, x, px, py)), (fmt, shape, srt, pa, px, py)


@pytest.mark.parametrize("sigma", ["64", "1000000"])
def test_spmv_sorted_rows_bit_exact(probs, oracle, sigma, monkeypatch):
    """the row-sorted tile stream (rows ordered by length inside windows of sigma
    rows, the epilogue writing through the permutation) is bit-exact with the
    oracle on every small problem, precision triple and column stream"""
    import paper_2505_20719_b200 as f
    monkeypatch.setenv("F3RG_SORT_ROWS", "1")
    monkeypatch.setenv("F3RG_SORT_SIGMA", sigma)
    for name, p, _ in probs:
        a = (p.n, p.row_ptr, p.col_idx)
        for fmt in ("", "u32"):
            monkeypatch.setenv("F3RG_COLUMNS", fmt)
            reps = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values))
            for pa, px, py in [(0, 0, 0), (0, 1, 1), (1, 1, 1), (2, 2, 2), (2, 1, 2), (0, 2, 0)]:
                x = rand_vec(oracle, px, p.n, 5 + pa)
                y = f.DenseVector(p.n, py)
                f.spmv(reps.at(pa), f.DenseVector(x, px), y)
                want = oracle.spmv(a, oracle.round_vec(pa, p.values), pa, x, px, py)
                assert np.array_equal(y.numpy(), want), (name, sigma, fmt, pa, px, py)
            # the replica values read back in the matrix's own row order
            assert np.array_equal(reps.at(0).values(), oracle.round_vec(0, p.values)), name


def test_elementwise_bit_exact(cuda, oracle):
    import paper_2505_20719_b200 as f
    n = 100_003
    for px in PRECS:
        for py in PRECS:
            x = rand_vec(oracle, px, n, 1, -3, 3)
            y = rand_vec(oracle, py, n, 2, -3, 3)
            alpha = -0.7310585786300049
            yd = f.DenseVector(y, py)
            f.axpy(alpha, f.DenseVector(x, px), yd)
            assert np.array_equal(yd.numpy(), oracle.axpy(alpha, x, px, y, py)), ("axpy", px, py)
            for po in PRECS:
                od = f.DenseVector(n, po)
                f.add_scaled(f.DenseVector(x, px), alpha, f.DenseVector(y, py), od)
                assert np.array_equal(od.numpy(), oracle.add_scaled(x, px, alpha, y, py, po)), ("add_scaled", px, py, po)
            cd = f.DenseVector(n, py)
            f.copy_into(f.DenseVector(x, px), cd)
            assert np.array_equal(cd.numpy(), oracle.copy(x, px, py)), ("copy", px, py)
        x = rand_vec(oracle, px, n, 3, -3, 3)
        xd = f.DenseVector(x, px)
        f.scale_in_place(1.0 / 3.0, xd)
        assert np.array_equal(xd.numpy(), oracle.scale(1.0 / 3.0, x, px)), ("scale", px)
        fd = f.DenseVector(n, px)
        f.fill(fd, 0.1)
        assert np.all(fd.numpy() == oracle.round_vec(px, np.array([0.1]))[0])


@pytest.mark.parametrize("n", [1, 31, 4097, 1_000_003])
def test_reductions_within_tolerance(cuda, oracle, n):
    import paper_2505_20719_b200 as f
    for px in PRECS:
        for py in PRECS:
            x = rand_vec(oracle, px, n, 5)
            y = rand_vec(oracle, py, n, 6)
            exact = float(np.sum(x.astype(np.longdouble) * y.astype(np.longdouble)))
            scale = float(np.sum(np.abs(x * y))) or 1.0
            for floor in (1, 2):
                c = max(floor, px, py)
                u = {1: 2.0 ** -24, 2: 2.0 ** -53}[c]
                got = f.dot_at_least(f.DenseVector(x, px), f.DenseVector(y, py), floor)
                want = oracle.dot(x, px, y, py, floor)
                # device (fixed tree) within the tree bound of the exact dot; the
                # reference's sequential sum within its own (n u) bound; and the two
                # within the normwise tolerance wherever the sequential bound allows it
                assert abs(got - exact) <= (np.log2(max(n, 2)) + 2) * u * scale, (px, py, floor, got, exact)
                assert abs(want - exact) <= (n + 2) * u * scale
                assert abs(got - want) <= max(TOL[c], (n + 2) * u) * scale, (px, py, floor, got, want)
        x = rand_vec(oracle, px, n, 8)
        got = f.norm2(f.DenseVector(x, px))
        want = oracle.norm2(x, px)
        if px == 0 and n > 4097:
            continue  # a sum of squares beyond 65504 overflows any fp16 accumulation
        if px == 0:
            # fp16 accumulation: the reference's sequential fp16 sum stagnates once the
            # partial sum dwarfs the addends; the device's fixed tree does not. Both are
            # checked against the exact norm with the classical bounds (n u and log2(n) u).
            exact = float(np.sqrt(np.sum(x * x)))
            u = 2.0 ** -11
            assert abs(got - exact) <= (np.ceil(np.log2(max(n, 2))) + 2) * u * exact + 1e-7
            assert abs(want - exact) <= (n + 2) * u * exact + 1e-7
        else:
            u = {1: 2.0 ** -24, 2: 2.0 ** -53}[px]
            exact = float(np.sqrt(np.sum(x.astype(np.longdouble) ** 2)))
            assert abs(got - exact) <= (np.log2(max(n, 2)) + 3) * u * exact
            assert abs(got - want) <= max(TOL[px], (n + 3) * u) * max(want, 1e-300)


def test_dimension_errors(cuda):
    import paper_2505_20719_b200 as f
    with pytest.raises(f.DimensionError):
        f.axpy(1.0, f.DenseVector(3, 2), f.DenseVector(4, 2))
    with pytest.raises(f.DimensionError):
        f.dot(f.DenseVector(3, 2), f.DenseVector(4, 2))
    with pytest.raises(f.DimensionError):
        f.make_replicas(f.SparseCsr(2, [0, 1, 2], [1, 0], [1.0, 1.0]))  # fine
        f.make_replicas(f.SparseCsr(2, [0, 2, 2], [1, 0], [1.0, 1.0]))  # decreasing columns


@pytest.mark.parametrize("shape", ["", "2"])
def test_richardson_state_sequence(cuda, oracle, shape, monkeypatch):
    """richardson_apply over 130 calls (updates at calls 64 and 128): weights and
    counters follow the reference's schedule; outputs bit-exact on every
    non-update call and within fp16 tolerance overall. shape "2": the gather-bound
    tile shape with the row-sorted stream, whose plain calls materialise z1 first"""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import problems
    if shape:
        monkeypatch.setenv("F3RG_SHAPE", shape)
        monkeypatch.setenv("F3RG_SORT_ROWS", "1")
        monkeypatch.setenv("F3RG_SORT_SIGMA", "256")
    p = problems.problem(2, grid=16)
    reps = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values))
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
            # w' from tree-ordered fp32 dots: equal to ~fp32 rounding
            assert np.allclose(w, om_ref, rtol=1e-5, atol=0), (call, w, om_ref)
            assert np.linalg.norm(z - z_ref) <= TOL[0] * np.linalg.norm(z_ref), call
            om, cnt = np.array(w), counters  # continue from the device's state
        else:
            assert w == list(om_ref)
            assert np.array_equal(z, z_ref), (call, np.abs(z - z_ref).max())
            om, cnt = om_ref, cnt_ref


@pytest.mark.parametrize("gap", [65535, 65536, 65537])
def test_d16_gap_boundary(cuda, oracle, gap):
    """D16 stores in-row gaps minus one (columns strictly increase, so gaps are >= 1):
    a gap of 65,536 -- config 4's plane stride -- still streams 2-byte deltas, one
    of 65,537 falls back to u32 indices; the products are the same either way"""
    import paper_2505_20719_b200 as f
    n = 70000
    rng = np.random.default_rng(9)
    cols = []
    for i in range(n):
        c = {i}
        if i + gap < n and i % 7 == 0:
            c.add(i + gap)  # the widest gap of the matrix
        for j in rng.integers(max(0, i - 50), min(n, i + 50), 3):
            c.add(int(j))
        cols.append(np.array(sorted(c), np.uint32))
    rp = np.zeros(n + 1, np.uint32)
    rp[1:] = np.cumsum([len(c) for c in cols])
    ci = np.concatenate(cols)
    va = rng.uniform(-1, 1, ci.size)
    reps = f.make_replicas(f.SparseCsr(n, rp, ci, va))
    nnz = ci.size
    u32 = nnz * (2 + 4) + 4 * (n + 1)
    d16 = nnz * (2 + 2) + 4 * n + 4 * (n + 1)
    assert reps.stream_bytes(0) == (d16 if gap <= 65536 else u32)
    for pa, px, py in ((0, 0, 0), (0, 1, 1), (1, 1, 1), (2, 2, 2)):
        x = rand_vec(oracle, px, n, 4 + pa)
        y = f.DenseVector(n, py)
        f.spmv(reps.at(pa), f.DenseVector(x, px), y)
        assert np.array_equal(y.numpy(), oracle.spmv((n, rp, ci), oracle.round_vec(pa, va), pa, x, px, py)), (gap, pa)
