"""Problem setup: the Matrix Market reader/writer of libf3rg.so
(csrc/mmio.cpp, restating reference src/matrix_market.cpp:33-127) against the
UNMODIFIED reference's outputs (tests/golden/reference_mm.npz, and live where
oracle/_ref is built) -- bit-identical CSR and the same ParseError messages; and the
device diagonal scaling (f3rg_matrix_create_scaled) against the reference's
diagonal_scale, bit-exact (GPU)."""
import os

import numpy as np
import pytest

import paper_2505_20719_b200 as f
from mm_cases import CASES

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "reference_mm.npz"))


@pytest.mark.parametrize("name,text", CASES, ids=[c[0] for c in CASES])
def test_read_matrix_market_matches_reference(tmp_path, name, text):
    path = tmp_path / (name + ".mtx")
    path.write_text(text)
    want = str(G[name + "_err"])
    if want:
        with pytest.raises(f.ParseError) as e:
            f.read_matrix_market(str(path))
        assert str(e.value) == want
        return
    a = f.read_matrix_market(str(path))
    assert np.array_equal(a.row_ptr, G[name + "_rp"])
    assert np.array_equal(a.col_idx, G[name + "_ci"])
    assert np.array_equal(a.values.view(np.uint64), G[name + "_v"].view(np.uint64))


def test_write_read_round_trip(tmp_path):
    from paper_2505_20719_b200 import problems
    p = problems.problem(5, grid=3000)  # unstructured, values with full fp64 mantissas
    a = f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values)
    path = str(tmp_path / "u.mtx")
    f.write_matrix_market(path, a)
    b = f.read_matrix_market(path)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
    assert np.array_equal(a.values, b.values)  # %.17g round-trips binary64


def test_missing_file_is_parse_error():
    with pytest.raises(f.ParseError, match="cannot open"):
        f.read_matrix_market("/nonexistent/x.mtx")


def test_live_reader_vs_reference(tmp_path, reference):
    rng = np.random.default_rng(3)
    lines = []
    for _ in range(400):
        i, j = rng.integers(1, 60, 2)
        lines.append(f"{i} {j} {rng.standard_normal():.17g}")
    path = tmp_path / "r.mtx"
    path.write_text("%%MatrixMarket matrix coordinate real general\n59 59 400\n" + "\n".join(lines) + "\n")
    rp, ci, va = reference.read_matrix_market(str(path))
    a = f.read_matrix_market(str(path))
    assert np.array_equal(a.row_ptr, rp) and np.array_equal(a.col_idx, ci) and np.array_equal(a.values, va)


@pytest.mark.gpu
def test_device_diagonal_scale_bit_exact(cuda, reference):
    from paper_2505_20719_b200 import problems
    for cfg, grid in ((3, 12), (5, 4000)):
        p = problems.problem(cfg, grid=grid)
        # undo nothing: scale an unscaled variant (row-dependent values, random rhs)
        rng = np.random.default_rng(cfg)
        vals = p.values * rng.uniform(0.5, 2.0, p.values.size)
        b = rng.uniform(-1, 1, p.n)
        a = f.SparseCsr(p.n, p.row_ptr, p.col_idx, vals)
        s = f.diagonal_scale(a, b)
        vo, bo, d = reference.diagonal_scale(p.row_ptr, p.col_idx, vals, b)
        assert np.array_equal(s.replicas.host.values, vo)
        assert np.array_equal(s.rhs, bo) and np.array_equal(s.d, d)
        # the replicas are the scaled matrix's: an fp16 SpMV equals the unscaled-path one
        r2 = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, vo))
        x = f.DenseVector(rng.uniform(-1, 1, p.n), f.Precision.P16)
        y1, y2 = f.DenseVector(p.n, f.Precision.P32), f.DenseVector(p.n, f.Precision.P32)
        f.spmv(s.replicas.a16, x, y1)
        f.spmv(r2.a16, x, y2)
        assert np.array_equal(y1.numpy(), y2.numpy())


@pytest.mark.gpu
def test_device_diagonal_scale_errors(cuda):
    with pytest.raises(f.FactorizationError, match="missing diagonal entry in row 1"):
        f.diagonal_scale(f.SparseCsr(2, [0, 1, 2], [0, 0], [1.0, 1.0]), np.ones(2))
    with pytest.raises(f.FactorizationError, match="zero diagonal entry in row 0"):
        f.diagonal_scale(f.SparseCsr(2, [0, 1, 2], [0, 1], [0.0, 1.0]), np.ones(2))
