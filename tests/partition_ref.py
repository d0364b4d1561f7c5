"""Plain numpy restatement of the row-block partition plan (test infrastructure).

Follows the reference's block split (src/ilu.cpp:47-54) and DESIGN.md section 6's
ext layout; tests/test_partition.py checks the engine's C++ plans
(paper_2505_20719_b200/csrc/partition.cpp) against it entry by entry.
"""
import numpy as np


def partition_rows(n, P):
    base, rem = divmod(n, P)
    s = [0]
    for b in range(P):
        s.append(s[-1] + base + (1 if b < rem else 0))
    return s


def plan(n, rp, ci, P, rank):
    rp = np.asarray(rp, dtype=np.int64)
    ci = np.asarray(ci, dtype=np.int64)
    st = partition_rows(n, P)
    r0, r1 = st[rank], st[rank + 1]
    cols = ci[rp[r0]:rp[r1]]
    halo = np.unique(cols[(cols < r0) | (cols >= r1)])
    n_lo = int(np.searchsorted(halo, r0))
    n_hi = len(halo) - n_lo
    pad = (8 - n_lo % 8) % 8 if P > 1 else 0
    off = pad + n_lo
    n_own = r1 - r0
    n_ext = off + n_own + n_hi
    ld = (n_ext + 7) // 8 * 8 if P > 1 else n_ext
    owner = np.searchsorted(np.asarray(st), halo, side="right") - 1
    ext_of_halo = np.where(np.arange(len(halo)) < n_lo, pad + np.arange(len(halo)),
                           off + n_own + np.arange(len(halo)) - n_lo)
    recv_off = np.zeros(P, dtype=np.int64)
    recv_cnt = np.zeros(P, dtype=np.int64)
    for q in range(P):
        sel = np.nonzero(owner == q)[0]
        if len(sel):
            recv_off[q] = ext_of_halo[sel[0]]
            recv_cnt[q] = len(sel)
    send_idx = []
    for q in range(P):
        if q == rank:
            send_idx.append(np.zeros(0, dtype=np.int64))
            continue
        qc = ci[rp[st[q]]:rp[st[q + 1]]]
        need = np.unique(qc[(qc >= r0) & (qc < r1)]) - r0
        send_idx.append(need.astype(np.int64))
    lrp = rp[r0:r1 + 1] - rp[r0]
    lci = np.empty(len(cols), dtype=np.int64)
    lo = cols < r0
    hi = cols >= r1
    own = ~(lo | hi)
    lci[lo] = pad + np.searchsorted(halo[:n_lo], cols[lo])
    lci[own] = off + cols[own] - r0
    lci[hi] = off + n_own + np.searchsorted(halo[n_lo:], cols[hi])
    return dict(r0=r0, r1=r1, n_lo=n_lo, n_hi=n_hi, pad=pad, off=off, n_ext=n_ext, ld=ld, halo=halo,
                recv_off=recv_off, recv_cnt=recv_cnt, send_idx=send_idx, local_rp=lrp, local_ci=lci,
                nnz_begin=int(rp[r0]))


def ext_to_global(p, n_own):
    """global column of every ext index (-1 for the pad)"""
    g = np.full(p["n_ext"], -1, dtype=np.int64)
    g[p["pad"]:p["off"]] = p["halo"][:p["n_lo"]]
    g[p["off"]:p["off"] + n_own] = np.arange(p["r0"], p["r1"])
    g[p["off"] + n_own:] = p["halo"][p["n_lo"]:]
    return g
