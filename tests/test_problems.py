"""CPU: the synthetic problem generators (host C++ in libf3rg.so) follow the
reference's conventions and, for config 2, reproduce the reference's own
generate_stencil + diagonal_scale + rhs bit-for-bit."""
import hashlib

import numpy as np
import pytest

from paper_2505_20719_b200 import problems


def splitmix_unit(seed, n):
    M = (1 << 64) - 1
    s, out = seed, np.empty(n)
    for i in range(n):
        s = (s + 0x9E3779B97F4A7C15) & M
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        z ^= z >> 31
        out[i] = (z >> 11) * 2.0 ** -53
    return out


@pytest.mark.parametrize("l", [1, 3, 4])
def test_config2_recipe_matches_reference(reference, l):
    g = 2 ** l
    p = problems.problem(2, grid=g)
    rp, ci, va = reference.generate_stencil(l, l, l, 0.0)
    assert np.array_equal(p.row_ptr, rp) and np.array_equal(p.col_idx, ci)
    xt = 2.0 * splitmix_unit(1, p.n) - 1.0
    b = reference.spmv(reference.matrix(rp, ci, va), 2, xt, 2, 2)
    vs, bs, d = reference.diagonal_scale(rp, ci, va, b)
    assert np.array_equal(p.values, vs) and np.array_equal(p.b, bs) and np.array_equal(p.d, d)


def test_hpgmp_beta(reference):
    from paper_2505_20719_b200.problems import STENCIL27, generate
    p = generate(STENCIL27, (8, 8, 8), 0.5, 0, 0, 3)
    rp, ci, va = reference.generate_stencil(3, 3, 3, 0.5)
    vs, _, _ = reference.diagonal_scale(rp, ci, va)
    assert np.array_equal(p.col_idx, ci) and np.array_equal(p.values, vs)


@pytest.mark.parametrize("config,grid", [(1, 12), (3, 10), (4, 10), (5, 3000)])
def test_structure_and_scaling(config, grid):
    p = problems.problem(config, grid=grid)
    rp, ci = p.row_ptr.astype(np.int64), p.col_idx.astype(np.int64)
    assert rp[0] == 0 and rp[-1] == p.nnz and np.all(np.diff(rp) >= 1)
    for i in range(p.n):  # strictly increasing columns, diagonal present and == 1 after scaling
        c = ci[rp[i]:rp[i + 1]]
        assert np.all(np.diff(c) > 0)
        k = np.searchsorted(c, i)
        assert c[k] == i and p.values[rp[i] + k] == pytest.approx(1.0, abs=1e-15)
    assert np.all(np.isfinite(p.b))


def test_config1_poisson_values():
    p = problems.problem(1, grid=4)
    # interior row of the unscaled 7-point Laplacian: 6 on the diagonal, -1 off -> scaled -1/6
    i = 1 + 4 * (1 + 4 * 1)
    row = p.values[p.row_ptr[i]:p.row_ptr[i + 1]]
    assert len(row) == 7 and np.allclose(sorted(row), [-1 / 6] * 6 + [1.0])


def test_config3_upwind_nonsymmetric():
    p = problems.problem(3, grid=4)
    i = 1 + 4 * (1 + 4 * 1)
    row = p.values[p.row_ptr[i]:p.row_ptr[i + 1]]
    assert np.allclose(row, [-2 / 9, -2 / 9, -2 / 9, 1.0, -1 / 9, -1 / 9, -1 / 9])


def test_config4_symmetric_and_b_is_row_sum():
    p = problems.problem(4, grid=6)
    import scipy.sparse as sp
    A = sp.csr_matrix((p.values, p.col_idx, p.row_ptr), shape=(p.n, p.n))
    # symmetric up to the scaling's rounding: (a d_i) d_j vs (a d_j) d_i, as in the reference
    assert abs(A - A.T).max() <= 4e-16 * abs(A).max()
    assert np.array_equal(p.b, np.array([sum(A.data[A.indptr[i]:A.indptr[i + 1]]) for i in range(p.n)]))


def test_config5_row_lengths_and_dominance():
    p = problems.problem(5, grid=20000)
    lens = np.diff(p.row_ptr)
    assert lens.min() >= 5 and lens.max() <= 200
    assert 25 <= lens.mean() <= 35
    import scipy.sparse as sp
    # undo the symmetric scaling: a_ij = a~_ij / (d_i d_j); the generator sets
    # a_ii = 1.1 * sum_j |a_ij| (strict row diagonal dominance of the unscaled A)
    rows = np.repeat(np.arange(p.n), np.diff(p.row_ptr))
    raw = p.values / (p.d[rows] * p.d[p.col_idx])
    A = sp.csr_matrix((raw, p.col_idx, p.row_ptr), shape=(p.n, p.n))
    diag = A.diagonal()
    off = np.asarray(abs(A).sum(axis=1)).ravel() - diag
    assert np.allclose(diag, 1.1 * off, rtol=1e-12)


def test_generators_are_pinned():
    """checksums of the test-size instances (regenerating them must not drift)"""
    def h(p):
        m = hashlib.sha256()
        for a in (p.row_ptr, p.col_idx, p.values, p.b):
            m.update(np.ascontiguousarray(a).tobytes())
        return m.hexdigest()[:16]
    got = {c: h(problems.problem(c, grid=g)) for c, g in [(1, 8), (2, 8), (3, 8), (4, 8), (5, 2000)]}
    assert got == PINNED, got


PINNED = {1: '58d4dc78c920da29', 2: '008e09aaa0c600d5', 3: 'e0fcbc8c666672ad', 4: '845e6b7d1e3a2c11',
          5: '434b411e5ba661c7'}


@pytest.mark.parametrize("config,grid", [(1, 8), (2, 8), (3, 8), (4, 8), (5, 3000)])
def test_binary_cache_matches_generator(tmp_path, monkeypatch, config, grid):
    """lib/f3rg_gen's binary CSR cache (csr_cache) holds exactly the
    bytes problems.problem() builds in-process, and the config tables agree"""
    from paper_2505_20719_b200 import csr_cache
    monkeypatch.setenv("F3RG_CACHE_DIR", str(tmp_path))
    assert csr_cache.CONFIGS[config] == problems.CONFIGS[config][:6]
    c = csr_cache.load(config, grid)
    p = problems.problem(config, grid=grid)
    assert (c.n, c.nnz, c.name) == (p.n, p.nnz, p.name)
    for a, b in ((c.row_ptr, p.row_ptr), (c.col_idx, p.col_idx), (c.values, p.values), (c.b, p.b)):
        assert a.dtype == b.dtype and np.array_equal(np.asarray(a), b)
    assert csr_cache.load(config, grid).path == c.path  # second call reads the existing file
