"""CPU: the block-Jacobi ILU(0)/IC(0) primary preconditioner of the oracle
(oracle/f3r_oracle.c or_ilu_*, restating reference src/ilu.cpp:38-263) pinned
bit-exactly to the UNMODIFIED reference through tests/golden/reference_ilu.npz
(tests/golden/make_golden_ilu.py), plus the reference's own ILU unit cases
(tests/test_ilu.cpp:29-163) restated against the oracle, and -- where
oracle/_ref is built -- live comparisons on fresh inputs."""
import os

import numpy as np
import pytest

from oracle_bind import FactorizationFailed

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "reference_ilu.npz"))


def mat(l, beta):
    k = f"mat{l}_{int(beta * 10)}"
    rp, ci, vs = G[k + "_rp"], G[k + "_ci"], G[k + "_vals"]
    return (len(rp) - 1, rp, ci), vs


def test_apply_matches_reference_golden(oracle):
    i = 0
    while f"f{i}_cfg" in G:
        l, beta, sym, nb, prec, alpha = G[f"f{i}_cfg"]
        a, vs = mat(int(l), float(beta))
        M = oracle.ilu(a, vs, int(nb), float(alpha), bool(sym), int(prec))
        for pr in (0, 1, 2):
            for pz in (0, 1, 2):
                got = M.apply(G[f"f{i}_r{pr}"], pr, pz)
                assert np.array_equal(got, G[f"f{i}_z{pr}{pz}"]), (i, pr, pz)
        i += 1
    assert i >= 7


def test_richardson_with_m_matches_reference_golden(oracle):
    a, vs = mat(3, 0.0)
    n = a[0]
    for p in (0, 1):
        M = oracle.ilu(a, vs, 4, 1.0, True, p)
        vp = oracle.round_vec(p, vs)
        om, cnt = np.ones(2), [1, 0, 0]
        zs = []
        for call in range(130):
            v = oracle.round_vec(p, np.random.default_rng(3000 + call).uniform(-1, 1, n))
            z, om, cnt = oracle.richardson_apply(a, vp, p, 2, 64, om, cnt, v, precond=M)
            zs.append(z)
        assert np.array_equal(zs[63], G[f"rich{p}_z_64"])
        assert np.array_equal(zs[-1], G[f"rich{p}_z_last"])
        assert np.array_equal(om, G[f"rich{p}_omegas"])
        assert cnt == list(G[f"rich{p}_counters"])


def test_solves_with_m_match_reference_golden(oracle):
    a, vs = mat(4, 0.0)
    b = G["solve_b"]
    for i, spec in enumerate(G["solve_specs"]):
        nb, sym, prec = G[f"solve{i}_m"]
        M = oracle.ilu(a, vs, int(nb), 1.0, bool(sym), int(prec))
        rep = oracle.solve(a, vs, str(spec), b, tol=1e-10, precond=M)
        conv, outer, pinv, final = G[f"solve{i}_meta"]
        assert rep.converged == bool(conv) and rep.outer_iterations == int(outer), spec
        assert rep.precond_invocations == int(pinv)
        assert rep.final_true_residual == final
        assert np.array_equal(np.array(rep.residual_history), G[f"solve{i}_hist"])
        assert np.array_equal(rep.x, G[f"solve{i}_x"])
        assert rep.level_iterations == list(G[f"solve{i}_levels"])
        assert np.array_equal(np.array(rep.omegas_final), G[f"solve{i}_omegas"])


def test_factorization_errors_match_reference_messages(oracle):
    cases = [(2, [0, 1, 2], [1, 0], [1.0, 1.0], 0, 2), (2, [0, 2, 4], [0, 1, 0, 1], [1.0, 2.0, 2.0, 1.0], 1, 2),
             (1, [0, 1], [0], [1e-9], 0, 0), (1, [0, 1], [0], [1e6], 1, 0)]
    for (n, rp, ci, va, sym, prec), want in zip(cases, G["error_msgs"]):
        a = (n, np.array(rp, np.uint32), np.array(ci, np.uint32))
        try:
            oracle.ilu(a, np.array(va), 1, 1.0, bool(sym), prec)
            got = ""
        except FactorizationFailed as e:
            got = str(e)
        assert got == str(want)
    a = (2, np.array([0, 1, 2], np.uint32), np.array([0, 1], np.uint32))
    with pytest.raises(FactorizationFailed, match=r"nblocks must be in \[1, n\]"):
        oracle.ilu(a, np.ones(2), 3)
    with pytest.raises(FactorizationFailed, match="alpha must be positive"):
        oracle.ilu(a, np.ones(2), 1, alpha=0.0)


# ---- the reference's own unit cases (tests/test_ilu.cpp), restated ----------------
def csr(d):
    d = np.asarray(d, float)
    rp, ci, va = [0], [], []
    for row in d:
        nz = np.nonzero(row)[0]
        ci += list(nz)
        va += list(row[nz])
        rp.append(len(ci))
    return (d.shape[0], np.array(rp, np.uint32), np.array(ci, np.uint32)), np.array(va)


def test_identity_factorizes_to_identity(oracle):  # test_ilu.cpp:29-36
    a, v = csr(np.eye(4))
    for nb in (1, 2, 4):
        z = oracle.ilu(a, v, nb).apply(np.array([1.0, 2, 3, 4]), 2, 2)
        assert list(z) == [1.0, 2, 3, 4]


def test_dense_2x2_hand_elimination(oracle):  # test_ilu.cpp:38-60
    a, v = csr([[4.0, 1.0], [1.0, 4.0]])
    z = oracle.ilu(a, v, 1).apply(np.ones(2), 2, 2)
    assert abs(4 * z[0] + z[1] - 1) < 1e-15 and abs(z[0] + 4 * z[1] - 1) < 1e-15
    z = oracle.ilu(a, v, 1, alpha=1.2).apply(np.array([1.0, 0.0]), 2, 2)
    u22 = 4.8 - 1.0 / 4.8
    z2 = (-1.0 / 4.8) / u22
    assert z[1] == pytest.approx(z2, rel=1e-15) and z[0] == pytest.approx((1.0 - z2) / 4.8, rel=1e-15)


def test_one_row_blocks_are_boosted_jacobi(oracle):  # test_ilu.cpp:62-72
    a, v = csr([[4.0, -1, 0], [-1, 5, -1], [0, -1, 6]])
    z = oracle.ilu(a, v, 3, alpha=1.5).apply(np.ones(3), 2, 2)
    assert np.allclose(z, [1 / 6.0, 1 / 7.5, 1 / 9.0], rtol=1e-15)


def test_no_dropped_fill_is_exact_inverse(oracle):  # test_ilu.cpp:74-89
    rng = np.random.default_rng(3)
    d = np.zeros((6, 6))
    for s in (0, 3):
        q = rng.uniform(-1, 1, (3, 3))
        d[s:s + 3, s:s + 3] = q @ q.T + 3 * np.eye(3)
    a, v = csr(d)
    r = rng.uniform(-1, 1, 6)
    z = oracle.ilu(a, v, 2).apply(r, 2, 2)
    assert np.allclose(z, np.linalg.solve(d, r), rtol=1e-12, atol=1e-14)


def test_ic_symmetric_and_close_to_ilu(oracle):  # test_ilu.cpp:91-118
    a, vs = mat(3, 0.0)
    n = a[0]
    mic, milu = oracle.ilu(a, vs, 2, symmetric=True), oracle.ilu(a, vs, 2)
    for i in (0, 5, 31):
        for j in (1, 17, 40):
            ei, ej = np.zeros(n), np.zeros(n)
            ei[i], ej[j] = 1, 1
            assert abs(mic.apply(ei, 2, 2)[j] - mic.apply(ej, 2, 2)[i]) <= 1e-12
    r = np.random.default_rng(5).uniform(-1, 1, n)
    assert np.allclose(mic.apply(r, 2, 2), milu.apply(r, 2, 2), rtol=1e-12, atol=1e-15)


def test_apply_linear_at_fp64(oracle):  # test_ilu.cpp:120-134
    a, vs = mat(3, 0.5)
    M = oracle.ilu(a, vs, 4)
    rng = np.random.default_rng(23)
    r1, r2 = rng.uniform(-1, 1, a[0]), rng.uniform(-1, 1, a[0])
    assert np.allclose(M.apply(2.5 * r1 + r2, 2, 2), 2.5 * M.apply(r1, 2, 2) + M.apply(r2, 2, 2), rtol=1e-12,
                       atol=1e-14)


def test_fp16_factors_with_fp64_input_compute_at_fp64(oracle):  # test_ilu.cpp:153-163
    a, v = csr([[4.0, 1.0], [1.0, 4.0]])
    r = np.array([1.0, 2.0])
    assert np.array_equal(oracle.ilu(a, v, 1, prec=0).apply(r, 2, 2), oracle.ilu(a, v, 1, prec=2).apply(r, 2, 2))


def test_live_against_reference(oracle, reference):
    rng = np.random.default_rng(11)
    for (l, beta) in ((3, 0.0), (3, 0.5)):
        rp, ci, va = reference.generate_stencil(l, l, l, beta)
        vs, _, _ = reference.diagonal_scale(rp, ci, va)
        a = (len(rp) - 1, rp, ci)
        m = reference.matrix(rp, ci, vs)
        for sym in ((0, 1) if beta == 0 else (0,)):
            for nb in (1, 2, 6):
                for prec in (0, 1, 2):
                    M, R = oracle.ilu(a, vs, nb, 1.0, sym, prec), reference.ilu(m, nb, 1.0, sym, prec)
                    for pr in (0, 2):
                        x = oracle.round_vec(pr, rng.uniform(-3, 3, a[0]))
                        assert np.array_equal(M.apply(x, pr, pr), R.apply(x, pr, pr)), (l, beta, sym, nb, prec, pr)
