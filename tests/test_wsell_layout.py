"""Host logic of the packed windowed SELL layout (csrc/wsell_pk_layout.hpp), checked on the
CPU through the C ABI (f3rg_wsell_pk_selfcheck): every row's slot sequence -- ring-slot
codes, escape pairs of far columns, padding -- must decode back to the CSR row in stored
order (the order the reference sums in, src/csr.cpp:23-37), far pairs must not straddle a
quad, and band / far classification must follow the window geometry of state.hpp. The check
runs for both geometries: the packed fp16 stream's (2-byte rings) and the 4-byte rings'.
"""
import numpy as np
import pytest

import paper_2505_20719_b200 as f
from paper_2505_20719_b200 import problems

RING, TW, W = 49152, 8192, 16384


def _csr_from_rows(n, rows):
    rp = np.zeros(n + 1, np.uint32)
    rp[1:] = np.cumsum([len(r) for r in rows])
    ci = np.concatenate([np.asarray(r, dtype=np.uint32) for r in rows]) if rp[-1] else np.zeros(0, np.uint32)
    return rp, ci


def test_config5_rows():
    p = problems.problem(5, grid=120_000)
    st = f.wsell_pk_selfcheck(p.n, p.row_ptr, p.col_idx)
    nnz = int(p.col_idx.size)
    # every entry has a slot, every far entry a second one
    assert st["slots"] >= nnz + st["far"] and st["slots"] % 128 == 0
    assert st["slices"] == -(-p.n // 2048) * 64
    # 5 % uniform long-range entries + the band's tails beyond 3.3 sigma + reserved-slot columns
    assert 0.03 * nnz < st["far"] < 0.09 * nnz


@pytest.mark.parametrize("ctas", [1, 3, 148])
def test_stencil_and_cta_counts(ctas):
    p = problems.problem(2, grid=24)  # 27-point 24^3: every column inside the band
    st = f.wsell_pk_selfcheck(p.n, p.row_ptr, p.col_idx, ctas)
    assert st["far"] == 0


def test_band_edges_and_reserved_slot():
    """columns exactly on the band's first / last row and one past, and columns whose ring slot is
    the reserved zero slot (RING - 1): the latter are far whatever their distance"""
    n = 6 * TW + 1234
    rows = []
    for i in range(n):
        B = i // TW * TW
        B1 = i // 4096 * 4096  # the 4-byte rings' geometry (class 1): 32,768 slots, 4096-row windows, W = 12,288
        cand = {i, B - W, B - W - 1, B + TW + W - 1, B + TW + W, RING - 1, 2 * RING - 1, (i + 7) % n,
                B1 - 12288, B1 - 12289, B1 + 4096 + 12288 - 1, B1 + 4096 + 12288, 32767, 65535}
        rows.append(sorted(c for c in cand if 0 <= c < n))
    rp, ci = _csr_from_rows(n, rows)
    st = f.wsell_pk_selfcheck(n, rp, ci, 5)
    assert st["far"] > 0


def test_ragged_rows_and_all_far():
    rng = np.random.default_rng(11)
    n = 70_000
    lens = rng.integers(0, 30, n)
    lens[3] = 0
    lens[100] = 900  # one long row: its slice is padded to its width
    lens[2048:4096] = 0  # a whole sort window of empty rows
    rows = [np.sort(rng.choice(n, size=L, replace=False)) for L in lens]  # uniform columns: mostly far
    rp, ci = _csr_from_rows(n, rows)
    st = f.wsell_pk_selfcheck(n, rp, ci, 7)
    assert st["far"] > 0.2 * ci.size


def test_empty_matrix_rows():
    n = 5000
    rp = np.zeros(n + 1, np.uint32)
    st = f.wsell_pk_selfcheck(n, rp, np.zeros(0, np.uint32), 4)
    assert st["far"] == 0 and st["slots"] == 0
