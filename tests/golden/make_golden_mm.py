"""Golden outputs of the UNMODIFIED reference's Matrix Market reader
(read_matrix_market, src/matrix_market.cpp:33-113) on tests/mm_cases.py.

    python tests/golden/make_golden_mm.py   ->  tests/golden/reference_mm.npz
"""
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from mm_cases import CASES  # noqa: E402
from oracle_bind import Reference  # noqa: E402


def main():
    r = Reference()
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name, text in CASES:
            path = os.path.join(d, name + ".mtx")
            open(path, "w").write(text)
            try:
                rp, ci, va = r.read_matrix_market(path)
                out[name + "_rp"], out[name + "_ci"], out[name + "_v"] = rp, ci, va
                out[name + "_err"] = np.array("")
            except RuntimeError as e:
                out[name + "_err"] = np.array(str(e).split(": ", 1)[1])
    path = os.path.join(HERE, "reference_mm.npz")
    np.savez_compressed(path, **out)
    print("wrote", path)


if __name__ == "__main__":
    main()
