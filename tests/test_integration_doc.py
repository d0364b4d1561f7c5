"""The ctypes stub printed in INTEGRATION.md §3 is executed verbatim, so the
binding a maintainer would copy is known to work against the C ABI."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    assert blocks, "INTEGRATION.md lost its python stub"
    return blocks[0]


def test_stub_compiles():
    compile(_stub(), "INTEGRATION.md", "exec")


@pytest.mark.gpu
def test_stub_solves(cuda):
    from paper_2505_20719_b200 import LIB_PATH, problems
    ns = {"LIB": LIB_PATH}
    exec(_stub(), ns)
    p = problems.problem(1, grid=16)
    x, rep = ns["solve"](p.row_ptr, p.col_idx, p.values, p.b,
                         "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > identity")
    assert rep.converged == 1 and rep.final_true_residual <= 1e-10
    import scipy.sparse as sp
    a = sp.csr_matrix((p.values, p.col_idx, p.row_ptr), shape=(p.n, p.n))
    assert np.linalg.norm(p.b - a @ x) / np.linalg.norm(p.b) <= 1e-10
