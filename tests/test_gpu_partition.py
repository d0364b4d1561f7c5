"""Row-block partition on the device.

This box has one GPU, so the P ranks run as threads of one process on it
(LocalPartition): the same plans, ext layouts, halo gathers and rank-ordered
reductions as the NCCL transport, which is exercised here with P = 1."""
import numpy as np
import pytest

from _util import F3R16, F3R32, small_problems

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def probs():
    return small_problems()


def _csr(p):
    from paper_2505_20719_b200 import SparseCsr
    return SparseCsr(p.n, p.row_ptr, p.col_idx, p.values)


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("triple", [(0, 0, 0), (0, 1, 1), (1, 1, 1), (2, 2, 2), (2, 1, 2), (0, 2, 1)])
def test_partitioned_spmv_bit_exact(cuda, oracle, probs, P, triple):
    """halo exchange + rank-local SpMVs reproduce the reference's global SpMV
    bit for bit (stored-order row sums; every precision triple class)"""
    from paper_2505_20719_b200 import partition
    pa, px, py = triple
    for name, p in probs:
        x = np.random.default_rng(P).uniform(-1, 1, p.n)
        x = oracle.round_vec(px, x)
        want = oracle.spmv((p.n, p.row_ptr, p.col_idx), oracle.round_vec(pa, p.values), pa, x, px, py)
        got = partition.local_spmv(_csr(p), P, pa, px, py, x)
        assert np.array_equal(got, want), (name, P, triple)


def test_partitioned_spmv_u32_columns(cuda, oracle, probs, monkeypatch):
    from paper_2505_20719_b200 import partition
    monkeypatch.setenv("F3RG_COLUMNS", "u32")
    name, p = probs[4]
    x = oracle.round_vec(0, np.random.default_rng(3).uniform(-1, 1, p.n))
    want = oracle.spmv((p.n, p.row_ptr, p.col_idx), oracle.round_vec(0, p.values), 0, x, 0, 0)
    assert np.array_equal(partition.local_spmv(_csr(p), 3, 0, 0, 0, x), want)


def test_one_rank_partition_is_the_plain_solver_bitwise(cuda, probs):
    """P = 1 through the partitioned engine path (rank-local reductions + the
    one-CTA combine, Richardson update calls as phase launches) is bitwise the
    single-GPU solver"""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import partition
    for name, p in probs[:2]:
        reps = f.make_replicas(_csr(p))
        s = f.build(f.parse_solver_spec(F3R16), reps, f.IdentityPrecond(p.n))
        r1 = s.run(p.b, f.RunOptions(tol=TOL))
        lp = partition.LocalPartition(_csr(p), F3R16, 1)
        x, reps_p = lp.run(p.b, f.RunOptions(tol=TOL))
        assert reps_p[0].residual_history == r1.report.residual_history, name
        assert np.array_equal(x, r1.x), name
        assert reps_p[0].omegas_final == r1.report.omegas_final


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("spec", [F3R16, F3R32])
def test_partitioned_solve_matches_single(cuda, probs, P, spec):
    """P ranks: same outer count (+-10 %), converged to tol with the fp64 true
    residual, identical replicated state on every rank"""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import partition
    for name, p in probs:
        reps = f.make_replicas(_csr(p))
        s = f.build(f.parse_solver_spec(spec), reps, f.IdentityPrecond(p.n))
        r1 = s.run(p.b, f.RunOptions(tol=TOL)).report
        lp = partition.LocalPartition(_csr(p), spec, P)
        x, rr = lp.run(p.b, f.RunOptions(tol=TOL))
        for r in rr[1:]:  # replicated scalars: bitwise identical on all ranks
            assert r.residual_history == rr[0].residual_history and r.omegas_final == rr[0].omegas_final
            assert r.outer_iterations == rr[0].outer_iterations
        rep = rr[0]
        assert rep.converged and rep.final_true_residual <= TOL, (name, P, rep)
        assert abs(rep.outer_iterations - r1.outer_iterations) <= max(1, round(0.1 * r1.outer_iterations)), \
            (name, P, rep.outer_iterations, r1.outer_iterations)
        import scipy.sparse as sp
        a = sp.csr_matrix((p.values, p.col_idx, p.row_ptr), shape=(p.n, p.n))
        assert np.linalg.norm(p.b - a @ x) / np.linalg.norm(p.b) <= TOL * 1.0001


def test_partitioned_richardson_update_calls(cuda, probs):
    """the weight-update calls (call_count % 64 == 0) as phase launches: identical
    weights on every rank, close to the single-GPU run's. (The phase arithmetic
    itself is pinned bitwise by the P = 1 test above; across P the input vectors
    differ by the reduction order, and w' is a ratio of two such dots.)"""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import partition
    name, p = probs[1]  # poisson24: call 64 happens at residual ~1e-9, well above the noise floor
    reps = f.make_replicas(_csr(p))
    s = f.build(f.parse_solver_spec(F3R16), reps, f.IdentityPrecond(p.n))
    opts = f.RunOptions(tol=1e-18, max_outer_total=2)  # 64 Richardson calls; call 64 updates
    r1 = s.run(p.b, opts).report
    assert r1.precond_invocations == 2 * 32 * 2
    assert r1.omegas_final != [1.0, 1.0]
    for P in (2, 3):
        lp = partition.LocalPartition(_csr(p), F3R16, P)
        _, rr = lp.run(p.b, opts)
        assert rr[0].precond_invocations == r1.precond_invocations
        assert all(r.omegas_final == rr[0].omegas_final for r in rr)
        assert np.allclose(rr[0].omegas_final, r1.omegas_final, rtol=1e-2), (P, rr[0].omegas_final, r1.omegas_final)


def test_collectives_per_outer_iteration(cuda, probs):
    """SURVEY 8(e)'s collective count per outer iteration of fp16-F3R: 73 halo
    exchanges (1 + 8 + 32 z_j + 32 Richardson v) and 91 reductions (2 + 17 + 72).
    A Richardson call enqueues its update phases (2 halos + 2 reductions for m = 2)
    only where the device's call counter can make it an update call (one call in
    64), instead of on every call (then: +96 halos and +64 reductions per outer
    iteration). The same count on every rank."""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import partition
    name, p = probs[1]
    K = 4
    opts = f.RunOptions(tol=1e-18, max_outer_total=K)  # 128 Richardson calls: updates at 64 and 128
    lp = partition.LocalPartition(_csr(p), F3R16, 2)
    _, rr = lp.run(p.b, opts)
    assert rr[0].outer_iterations == K
    counts = [s.collectives() for s in lp.solvers]
    assert counts[0] == counts[1]
    halos, reds = counts[0]
    upd = 2  # update calls in the run
    # + the bnorm reduction, the cycle start, and the final true residual (halo + reduction)
    assert 73 * K + 2 * upd <= halos <= 73 * K + 2 * upd + 2, (halos, reds)
    assert 91 * K + 2 * upd <= reds <= 91 * K + 2 * upd + 3, (halos, reds)


def test_nccl_transport_one_rank(cuda, probs):
    """the NCCL transport (point-to-point halos, allgather) with one rank: bitwise
    the plain solver"""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import partition
    name, p = probs[0]
    try:
        uid = partition.nccl_unique_id()
    except f.UnsupportedError as e:
        pytest.skip(f"NCCL unavailable: {e}")
    reps = f.make_replicas(_csr(p))
    s = f.build(f.parse_solver_spec(F3R16), reps, f.IdentityPrecond(p.n))
    r1 = s.run(p.b, f.RunOptions(tol=TOL))
    npart = partition.NcclPartition(_csr(p), F3R16, 1, 0, uid)
    b = cuda.from_numpy(p.b).cuda()
    x = cuda.zeros(p.n, dtype=cuda.float64, device="cuda")
    rep = npart.run(b, x, f.RunOptions(tol=TOL))
    cuda.cuda.synchronize()
    assert rep.residual_history == r1.report.residual_history
    assert np.array_equal(x.cpu().numpy(), r1.x)


def test_partition_rejects_unsupported(cuda, probs):
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import partition
    name, p = probs[0]
    with pytest.raises(f.UnsupportedError):
        partition.LocalPartition(_csr(p), "F8:f64/f64 > R3:f16,c=64 > identity", 2)
    with pytest.raises(f.UnsupportedError):
        partition.LocalPartition(_csr(p), "R2:f64,c=64 > identity", 2)


@pytest.mark.parametrize("P", [2, 3])
def test_partitioned_ragged(cuda, oracle, P):
    """odd n (2431 rows, blocks of 811/810/810): halo pads, unaligned block sizes"""
    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import partition, problems
    p = problems.problem(1, grid=(17, 13, 11))
    x = oracle.round_vec(1, np.random.default_rng(5).uniform(-1, 1, p.n))
    want = oracle.spmv((p.n, p.row_ptr, p.col_idx), oracle.round_vec(0, p.values), 0, x, 1, 1)
    assert np.array_equal(partition.local_spmv(_csr(p), P, 0, 1, 1, x), want)
    lp = partition.LocalPartition(_csr(p), F3R16, P)
    _, rr = lp.run(p.b, f.RunOptions(tol=TOL))
    assert rr[0].converged and rr[0].final_true_residual <= TOL
