"""Sequential-reduction validation mode (f3rg_set_seq_reductions / F3RG_SEQ_REDUCTIONS):
every dot and norm of the device path summed in index order, as the reference's
dot_core (src/vector_ops.cpp:20-28). With it the device reproduces the reference's
reductions bit for bit, so the parity gates hold on long vectors too:

* dot / dot_at_least / norm2 bit-exact against the oracle (itself pinned to the
  reference) at every precision pairing, n up to 10^6 + 3;
* richardson_apply over 130 calls bit-exact INCLUDING the update calls (w' from
  in-order fp32 dots, src/richardson.cpp:31-45);
* the small composed solves equal to the oracle's, bit for bit (outer count,
  residual history, solution);
* the full-size BASELINE configs against the recorded runs of the UNMODIFIED
  reference (tests/golden/reference_runs.json), residual histories digit for digit
  -- config 5 (n = 2e7), whose default tree reductions take 2 outer steps where
  the reference takes 3, included.
"""
import json
import os

import numpy as np
import pytest

from _util import F3R16, F3R32, TOL, normwise, rand_vec, small_problems

pytestmark = pytest.mark.gpu

PRECS = (0, 1, 2)


@pytest.mark.parametrize("n", [1, 31, 4097, 1_000_003])
def test_seq_dots_bit_exact(cuda, oracle, n):
    import paper_2505_20719_b200 as f
    with f.seq_reductions():
        for px in PRECS:
            for py in PRECS:
                x = rand_vec(oracle, px, n, 5)
                y = rand_vec(oracle, py, n, 6)
                for floor in (0, 1, 2):
                    got = f.dot_at_least(f.DenseVector(x, px), f.DenseVector(y, py), floor)
                    want = oracle.dot(x, px, y, py, floor)
                    assert got == want or (np.isnan(got) and np.isnan(want)), (px, py, floor, got, want)
            x = rand_vec(oracle, px, n, 8)
            got = f.norm2(f.DenseVector(x, px))
            want = oracle.norm2(x, px)
            assert got == want or (np.isinf(got) and np.isinf(want)), (px, got, want)


def test_seq_flag_is_scoped(cuda, oracle):
    """the context manager restores the default tree reductions"""
    import paper_2505_20719_b200 as f
    n = 1_000_003
    x = rand_vec(oracle, 1, n, 5)
    y = rand_vec(oracle, 1, n, 6)
    want = oracle.dot(x, 1, y, 1, 1)
    with f.seq_reductions():
        assert f.dot_at_least(f.DenseVector(x, 1), f.DenseVector(y, 1), 1) == want
    got = f.dot_at_least(f.DenseVector(x, 1), f.DenseVector(y, 1), 1)
    assert got != want  # 10^6 fp32 terms: the tree and the sequential order part
    assert abs(got - want) <= (n + 2) * 2.0 ** -24 * float(np.sum(np.abs(x * y)))


def test_seq_richardson_sequence_bit_exact(cuda, oracle):
    """130 calls of richardson_apply (updates at calls 64 and 128): every output,
    weight and counter bit-exact with the oracle, update calls included"""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import problems
    p = problems.problem(2, grid=16)
    a = (p.n, p.row_ptr, p.col_idx)
    v16 = oracle.round_vec(0, p.values)
    with f.seq_reductions():
        reps = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values))
        st = f.RichardsonState(reps.a16, 2, 64)
        om = np.ones(2)
        cnt = [1, 0, 0]
        for call in range(1, 131):
            v = rand_vec(oracle, 0, p.n, 100 + call)
            z_ref, om_ref, cnt_ref = oracle.richardson_apply(a, v16, 0, 2, 64, om, cnt, v)
            zd = f.DenseVector(p.n, 0)
            f.richardson_apply(st, f.DenseVector(v, 0), zd)
            w, counters = st._state()
            assert counters == cnt_ref, call
            assert w == list(om_ref), (call, w, om_ref)
            assert np.array_equal(zd.numpy(), z_ref), call
            om, cnt = om_ref, cnt_ref


@pytest.mark.parametrize("spec", [F3R16, F3R32])
def test_seq_small_solves_match_oracle(cuda, oracle, spec):
    """with the reference's reduction order (and its hypot, common.cuh ref_hypot)
    the whole nested solve is the reference's arithmetic: the same outer count,
    residual history and solution, bit for bit"""
    import paper_2505_20719_b200 as f
    for name, p in small_problems():
        with f.seq_reductions():
            reps = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values))
            s = f.build(f.parse_solver_spec(spec), reps, f.IdentityPrecond(p.n))
            run = s.run(p.b, f.RunOptions(tol=1e-10))
        ref = oracle.solve((p.n, p.row_ptr, p.col_idx), p.values, spec, p.b, tol=1e-10)
        rep = run.report
        assert rep.outer_iterations == ref.outer_iterations, (name, rep.outer_iterations, ref.outer_iterations)
        assert rep.final_true_residual <= 1e-10
        assert rep.residual_history == list(ref.residual_history), (name, rep.residual_history, ref.residual_history)
        assert np.array_equal(run.x, ref.x), (name, normwise(run.x, ref.x))


def _reference_run(config):
    path = os.path.join(os.path.dirname(__file__), "golden", "reference_runs.json")
    return json.load(open(path)).get(f"config{config}/fp16-f3r")


@pytest.mark.parametrize("config", [2, 3, 5])
def test_seq_full_config_vs_reference(cuda, config):
    """the full-size BASELINE config under sequential reductions against the recorded
    run of the UNMODIFIED reference: the same outer count (config 5: 3, where the
    default tree reductions take 2) and the same residual history"""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import problems
    ref = _reference_run(config)
    p = problems.problem(config)
    assert (p.n, p.nnz) == (ref["n"], ref["nnz"])
    with f.seq_reductions():
        reps = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values))
        s = f.build(f.parse_solver_spec(F3R16), reps, f.IdentityPrecond(p.n))
        rep = s.run(cuda.from_numpy(p.b).cuda(), f.RunOptions(tol=1e-10), want_x=False).report
    assert rep.converged and rep.final_true_residual <= 1e-10, rep
    assert rep.outer_iterations == ref["outer_iterations"], (rep.outer_iterations, rep.residual_history)
    # the reference's own arithmetic, so its own residual history, digit for digit
    assert rep.residual_history == ref["residual_history"], (rep.residual_history, ref["residual_history"])
    assert rep.final_true_residual == ref["final_true_residual"]
