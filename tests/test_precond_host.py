"""CPU: the product's host factorisation of the block-Jacobi ILU(0)/IC(0) primary
preconditioner (libf3rg.so factorize_host, restating reference src/ilu.cpp:38-185)
against the oracle's (pinned to the reference by tests/test_oracle_ilu.py): the
stored factors must be bit-identical, and every factorisation error must carry
the reference's class and message. No GPU needed (the factorisation is host code)."""
import numpy as np
import pytest

import paper_2505_20719_b200 as f
from oracle_bind import FactorizationFailed
from paper_2505_20719_b200 import problems

CASES = [("hpcg8", problems.problem(2, grid=8), (True, False)),
         ("convdiff10", problems.problem(3, grid=10), (False,)),
         ("aniso8", problems.problem(4, grid=8), (True, False)),
         ("unstructured3000", problems.problem(5, grid=3000), (False,))]


@pytest.mark.parametrize("name,p,syms", CASES, ids=[c[0] for c in CASES])
def test_factors_bit_identical_to_oracle(oracle, name, p, syms):
    a = f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values)
    for sym in syms:
        for nb in (1, 4, 7):
            for prec in (0, 1, 2):
                for alpha in (1.0, 1.25):
                    (lp, li, lv), (up, ui, uv) = f.ilu_factorize_host(a, f.IluConfig(nb, alpha, sym, f.Precision(prec)))
                    M = oracle.ilu((p.n, p.row_ptr, p.col_idx), p.values, nb, alpha, sym, prec)
                    L, U = M.factors(0), M.factors(1)
                    for got, want in zip((lp, li, lv, up, ui, uv), (*L, *U)):
                        assert np.array_equal(got, want), (name, sym, nb, prec, alpha)


def test_factorization_errors_match_reference():
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_ilu.npz"))
    cases = [(2, [0, 1, 2], [1, 0], [1.0, 1.0], 0, 2), (2, [0, 2, 4], [0, 1, 0, 1], [1.0, 2.0, 2.0, 1.0], 1, 2),
             (1, [0, 1], [0], [1e-9], 0, 0), (1, [0, 1], [0], [1e6], 1, 0)]
    for (n, rp, ci, va, sym, prec), want in zip(cases, g["error_msgs"]):
        a = f.SparseCsr(n, rp, ci, va)
        if str(want):
            with pytest.raises(f.FactorizationError) as e:
                f.ilu_factorize_host(a, f.IluConfig(1, 1.0, bool(sym), f.Precision(prec)))
            assert str(e.value) == str(want)
        else:
            f.ilu_factorize_host(a, f.IluConfig(1, 1.0, bool(sym), f.Precision(prec)))
    a = f.SparseCsr(2, [0, 1, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(f.FactorizationError, match=r"nblocks must be in \[1, n\]"):
        f.ilu_factorize_host(a, f.IluConfig(3))
    with pytest.raises(f.FactorizationError, match="alpha must be positive"):
        f.ilu_factorize_host(a, f.IluConfig(1, alpha=-1.0))


def test_block_ranges_follow_reference_split():
    a = problems.problem(2, grid=8)
    A = f.SparseCsr(a.n, a.row_ptr, a.col_idx, a.values)
    (lp, li, _), _ = f.ilu_factorize_host(A, f.IluConfig(5, 1.0, True, f.Precision.P16))
    # base = n / 5, remainder to the leading blocks (src/ilu.cpp:47-54): no entry of a
    # row may reach below its block's first row
    n, base, rem = a.n, a.n // 5, a.n % 5
    starts = [0]
    for b in range(5):
        starts.append(starts[-1] + base + (1 if b < rem else 0))
    for b in range(5):
        lo, hi = starts[b], starts[b + 1]
        cols = li[lp[lo]:lp[hi]]
        assert cols.min() >= lo and cols.max() < hi
