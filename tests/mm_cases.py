"""Matrix Market test inputs (test infrastructure): each case is (name, text); the
expected CSR / error message of the reference reader is pinned in
tests/golden/reference_mm.npz (tests/golden/make_golden_mm.py)."""

CASES = [
    ("general", "%%MatrixMarket matrix coordinate real general\n% a comment\n3 3 4\n1 1 4.5\n2 2 -1e-3\n3 1 2\n2 3 0.1\n"),
    ("symmetric_dups", "%%MatrixMarket matrix coordinate real symmetric\n4 4 6\n1 1 2\n2 1 -1\n2 1 -0.25\n3 3 1e300\n"
                       "4 2 0.3333333333333333\n4 4 7\n"),
    ("pattern", "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 3\n1 1\n3 1\n3 3\n"),
    ("integer_upper", "%%MATRIXMARKET MATRIX COORDINATE INTEGER GENERAL\n\n2 2 3\n\n1 2 -7\n2 1 3\n2 2 1\n"),
    ("dup_sum_order", "%%MatrixMarket matrix coordinate real general\n2 2 5\n1 1 1e16\n1 1 1\n1 1 -1e16\n1 1 1\n2 2 1\n"),
    ("empty_rows", "%%MatrixMarket matrix coordinate real general\n5 5 2\n2 2 1\n5 1 3\n"),
    ("bad_banner", "MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n"),
    ("array", "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n"),
    ("complex", "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n"),
    ("hermitian", "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n"),
    ("nonsquare", "%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1\n"),
    ("out_of_bounds", "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n"),
    ("truncated", "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n"),
    ("missing_value", "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n"),
    ("bad_size", "%%MatrixMarket matrix coordinate real general\n2 x 1\n1 1 1\n"),
    ("empty", ""),
]
