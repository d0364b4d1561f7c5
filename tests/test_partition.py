"""Row-block partition: the engine's C++ plans against a numpy
restatement, the structural properties the device path relies on, and the N > 1
host path exercised over torch.distributed (gloo, world size 2) on CPU."""
import os
import socket

import numpy as np
import pytest

from partition_ref import ext_to_global, partition_rows, plan


def _random_csr(n, per_row, seed, band=None):
    rng = np.random.default_rng(seed)
    rp, ci = [0], []
    for i in range(n):
        k = int(rng.integers(0, per_row + 1))
        if band:
            c = np.clip(i + rng.integers(-band, band + 1, size=k), 0, n - 1)
        else:
            c = rng.integers(0, n, size=k)
        c = np.unique(np.append(c, i))
        ci.extend(c.tolist())
        rp.append(len(ci))
    return np.array(rp, dtype=np.uint32), np.array(ci, dtype=np.uint32), rng.uniform(-1, 1, len(ci))


def _cases():
    from paper_2505_20719_b200 import problems
    out = []
    for cfg, grid in ((1, 8), (2, 8), (3, 6), (4, 8), (5, 3000)):
        p = problems.problem(cfg, grid=grid)
        out.append((f"cfg{cfg}", p.n, p.row_ptr, p.col_idx, p.values))
    for seed, (n, k, band) in enumerate(((97, 5, None), (300, 9, 12), (64, 0, None), (1000, 3, 400))):
        rp, ci, v = _random_csr(n, k, seed, band)
        out.append((f"rand{seed}", n, rp, ci, v))
    return out


CASES = _cases()


def test_split_rule_matches_reference():
    # src/ilu.cpp:47-54: base = n / P, remainder over the leading blocks
    assert partition_rows(10, 3) == [0, 4, 7, 10]
    assert partition_rows(8, 4) == [0, 2, 4, 6, 8]
    assert partition_rows(5, 5) == [0, 1, 2, 3, 4, 5]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_plan_matches_restatement(case, P):
    from paper_2505_20719_b200 import SparseCsr, partition
    name, n, rp, ci, v = case
    a = SparseCsr(n, rp, ci, v)
    for r in range(P):
        got = partition.part_plan(a, P, r)
        want = plan(n, rp, ci, P, r)
        for k in ("r0", "r1", "n_lo", "n_hi", "pad", "off", "n_ext", "ld", "nnz_begin"):
            assert getattr(got, k) == want[k], (k, r)
        assert np.array_equal(got.halo, want["halo"])
        assert np.array_equal(got.recv_off[got.recv_cnt > 0], want["recv_off"][want["recv_cnt"] > 0])
        assert np.array_equal(got.recv_cnt, want["recv_cnt"])
        for q in range(P):
            assert np.array_equal(got.send_idx[q], want["send_idx"][q]), (r, q)
        assert np.array_equal(got.local_rp, want["local_rp"])
        assert np.array_equal(got.local_ci, want["local_ci"])


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("P", [2, 4])
def test_plan_properties(case, P):
    """what the device path relies on: the ext layout maps back to the global
    columns in stored order (bit-identical SpMV), in-row gaps never widen (D16
    stays valid), owned rows 16-byte aligned, and every rank's receive runs are
    exactly what its peers send."""
    name, n, rp, ci, v = case
    plans = [plan(n, rp, ci, P, r) for r in range(P)]
    for r, p in enumerate(plans):
        n_own = p["r1"] - p["r0"]
        g = ext_to_global(p, n_own)
        lo, hi = rp[p["r0"]], rp[p["r1"]]
        assert np.array_equal(g[p["local_ci"]], ci[lo:hi].astype(np.int64))
        assert p["off"] % 8 == 0 and p["ld"] % 8 == 0 and p["ld"] >= p["n_ext"]
        lrp, lci = p["local_rp"], p["local_ci"].astype(np.int64)
        for i in range(n_own):
            row = lci[lrp[i]:lrp[i + 1]]
            grow = ci[lo + lrp[i]:lo + lrp[i + 1]].astype(np.int64)
            assert np.all(np.diff(row) > 0)
            assert np.all(np.diff(row) <= np.diff(grow))
        for q in range(P):
            if q == r:
                continue
            # what q sends to r == r's run from q
            sent = plans[q]["send_idx"][r] + plans[q]["r0"]
            run = g[p["recv_off"][q]:p["recv_off"][q] + p["recv_cnt"][q]]
            assert np.array_equal(sent, run)


# ---- N > 1 over torch.distributed (gloo, world size 2, CPU) -------------------------------
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, n, rp, ci, v, x, results):
    import torch
    import torch.distributed as dist
    import scipy.sparse as sp
    from paper_2505_20719_b200 import SparseCsr, partition
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = SparseCsr(n, rp, ci, v)
        p = partition.part_plan(a, world, rank)      # the engine's plan (C++)
        n_own = p.r1 - p.r0
        # 1. the send lists must be the peers' receive runs (global indices)
        for q in range(world):
            if q == rank:
                continue
            mine = torch.from_numpy((p.send_idx[q].astype(np.int64) + p.r0))
            cnt = torch.tensor([mine.numel()])
            other_cnt = torch.zeros(1, dtype=torch.long)
            reqs = [dist.isend(cnt, q), dist.irecv(other_cnt, q)]
            [r.wait() for r in reqs]
            other = torch.zeros(int(other_cnt.item()), dtype=torch.long)
            reqs = [dist.isend(mine, q), dist.irecv(other, q)]
            [r.wait() for r in reqs]
            lo = int(p.recv_off[q])
            want = ext_to_global({"n_ext": p.n_ext, "pad": p.pad, "off": p.off, "halo": p.halo,
                                  "n_lo": p.n_lo, "r0": p.r0, "r1": p.r1}, n_own)[lo:lo + int(p.recv_cnt[q])]
            assert np.array_equal(other.numpy(), want), "halo runs disagree"
        # 2. halo exchange of x + rank-local SpMV (stored-order row sums) = global SpMV
        ext = np.zeros(p.n_ext)
        ext[p.off:p.off + n_own] = x[p.r0:p.r1]
        for q in range(world):
            if q == rank:
                continue
            out = torch.from_numpy(x[p.r0:p.r1][p.send_idx[q]].copy())
            buf = torch.zeros(int(p.recv_cnt[q]), dtype=torch.float64)
            reqs = ([dist.isend(out, q)] if out.numel() else []) + ([dist.irecv(buf, q)] if buf.numel() else [])
            [r.wait() for r in reqs]
            ext[int(p.recv_off[q]):int(p.recv_off[q]) + buf.numel()] = buf.numpy()
        vals = v[p.nnz_begin:p.nnz_begin + len(p.local_ci)]
        aloc = sp.csr_matrix((vals, p.local_ci, p.local_rp), shape=(n_own, p.n_ext))
        y_own = torch.from_numpy(aloc @ ext)
        sizes = [partition_rows(n, world)[q + 1] - partition_rows(n, world)[q] for q in range(world)]
        parts = [torch.zeros(s, dtype=torch.float64) for s in sizes]
        dist.all_gather(parts, y_own)
        y = torch.cat(parts).numpy()
        # 3. rank-ordered combination of rank-local dot partials (the engine's Dist
        #    mode 2): every rank gets the same bits
        loc = torch.tensor([float(np.dot(y_own.numpy(), y_own.numpy()))], dtype=torch.float64)
        allp = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allp, loc)
        tot = 0.0
        for t in allp:
            tot = tot + float(t.item())
        results[rank] = (y, tot)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,grid", [(2, 8), (5, 2000), (3, 6)])
def test_gloo_world2_halo_spmv(cfg, grid):
    import torch.multiprocessing as mp
    import scipy.sparse as sp
    from paper_2505_20719_b200 import problems
    p = problems.problem(cfg, grid=grid)
    x = np.random.default_rng(7).uniform(-1, 1, p.n)
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, p.n, p.row_ptr, p.col_idx, p.values, x, results))
             for r in range(2)]
    [pr.start() for pr in procs]
    [pr.join(120) for pr in procs]
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    ref = sp.csr_matrix((p.values, p.col_idx, p.row_ptr), shape=(p.n, p.n)) @ x
    y0, t0 = results[0]
    y1, t1 = results[1]
    assert np.array_equal(y0, ref) and np.array_equal(y1, ref)   # bit-exact
    assert t0 == t1                                               # identical replicated scalar
