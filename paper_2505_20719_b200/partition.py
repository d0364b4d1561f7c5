"""Row-block partition of the solve over P ranks.

Rows are split with the reference's rule (src/ilu.cpp:47-54: base = n/P, the
remainder spread over the leading blocks). Each rank owns its rows of A and of
every Krylov vector; SpMV inputs use the rank's ext layout
[pad | lo halo | owned | hi halo]; dots and norms are rank-local sums combined in
rank order, so all ranks hold bitwise-identical Hessenberg/Givens scalars and take
identical control decisions.

Two transports, one engine:
  LocalPartition  P ranks as threads of this process on the current device (the
                  one-GPU test vehicle: same plan, halo and reduction data flow)
  NcclPartition   one rank per process (torch.distributed launch), NCCL
                  point-to-point halos + allgather of the rank-local totals
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List

import numpy as np

from . import (ComposedSolver, DimensionError, RunOptions, SparseCsr, SolverSpec, _check, _Csr, _Report, lib)

IDENTITY = 2


class _PartInfo(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("r0", "r1", "n_lo", "n_hi", "pad", "off", "n_ext", "ld", "nnz_local",
                                          "nnz_begin", "n_send")]


def _csr(a: SparseCsr) -> _Csr:
    return _Csr(a.n, a.row_ptr.ctypes.data, a.col_idx.ctypes.data, a.values.ctypes.data)


@dataclass
class PartPlan:
    P: int
    rank: int
    r0: int
    r1: int
    n_lo: int
    n_hi: int
    pad: int
    off: int
    n_ext: int
    ld: int
    nnz_begin: int
    halo: np.ndarray          # global columns, ascending
    recv_off: np.ndarray      # [P] ext offset of each peer's run
    recv_cnt: np.ndarray      # [P]
    send_idx: List[np.ndarray]  # per peer: owned-local indices it needs, ascending
    local_rp: np.ndarray
    local_ci: np.ndarray      # ext columns


def part_plan(a: SparseCsr, P: int, rank: int) -> PartPlan:
    """rank `rank`'s plan as the engine builds it (C++ partition.cpp, host only)."""
    L = lib()
    c = _csr(a)
    info = _PartInfo()
    _check(L.f3rg_part_plan(C.byref(c), P, rank, C.byref(info), None, None, None, None, None, None, None))
    halo = np.zeros(max(1, info.n_lo + info.n_hi), dtype=np.uint32)
    roff = np.zeros(P, dtype=np.uint64)
    rcnt = np.zeros(P, dtype=np.uint64)
    scnt = np.zeros(P, dtype=np.uint64)
    sidx = np.zeros(max(1, info.n_send), dtype=np.uint32)
    lrp = np.zeros(info.r1 - info.r0 + 1, dtype=np.uint32)
    lci = np.zeros(max(1, info.nnz_local), dtype=np.uint32)
    _check(L.f3rg_part_plan(C.byref(c), P, rank, C.byref(info), halo.ctypes.data, roff.ctypes.data,
                            rcnt.ctypes.data, scnt.ctypes.data, sidx.ctypes.data, lrp.ctypes.data, lci.ctypes.data))
    splits = np.cumsum(scnt.astype(np.int64))[:-1]
    return PartPlan(P, rank, info.r0, info.r1, info.n_lo, info.n_hi, info.pad, info.off, info.n_ext, info.ld,
                    info.nnz_begin, halo[:info.n_lo + info.n_hi], roff, rcnt,
                    [v.copy() for v in np.split(sidx[:info.n_send], splits)], lrp, lci[:info.nnz_local])


def local_spmv(a: SparseCsr, P: int, pa: int, px: int, py: int, x: np.ndarray) -> np.ndarray:
    """y = A x computed as P rank-local SpMVs after a halo exchange (device)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(a.n)
    c = _csr(a)
    _check(lib().f3rg_local_spmv(C.byref(c), P, pa, px, py, x.ctypes.data, y.ctypes.data))
    return y


class _PartSolver(ComposedSolver):
    def __init__(self, comm, a: SparseCsr, spec: str, rank: int):  # noqa: D401 (no super().__init__)
        self.h = C.c_void_p()
        c = _csr(a)
        _check(lib().f3rg_solver_create_part(C.byref(self.h), comm, C.byref(c), spec.encode(), IDENTITY, rank))
        self.n = None


class LocalPartition:
    """P ranks of one process on the current device (threads + one stream)."""

    def __init__(self, a: SparseCsr, spec, P: int):
        text = spec.text if isinstance(spec, SolverSpec) else str(spec)
        self.a, self.P = a, int(P)
        self.comm = C.c_void_p()
        _check(lib().f3rg_comm_local(C.byref(self.comm), C.byref(_csr(a)), self.P))
        self.solvers = [_PartSolver(self.comm, a, text, r) for r in range(self.P)]

    def run(self, b: np.ndarray, opts: RunOptions = RunOptions()):
        b = np.ascontiguousarray(b, dtype=np.float64)
        if b.size != self.a.n:
            raise DimensionError("run: rhs length mismatch")
        x = np.zeros(self.a.n)
        reps = (_Report * self.P)()
        hs = (C.c_void_p * self.P)(*[s.h.value for s in self.solvers])
        _check(lib().f3rg_solve_local(self.comm, hs, b.ctypes.data, x.ctypes.data, C.byref(opts._c()), reps))
        return x, [s._report(reps[r]) for r, s in enumerate(self.solvers)]

    def reset(self) -> None:
        for s in self.solvers:
            s.reset()

    def __del__(self):
        for s in getattr(self, "solvers", []):
            s.__del__()
        self.solvers = []
        if getattr(self, "comm", None) and self.comm.value:
            lib().f3rg_comm_destroy(self.comm)
            self.comm = None


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib().f3rg_nccl_unique_id(buf))
    return bytes(buf)


class NcclPartition:
    """This process's rank of a P-rank NCCL partition (one GPU per process)."""

    def __init__(self, a: SparseCsr, spec, P: int, rank: int, unique_id: bytes):
        text = spec.text if isinstance(spec, SolverSpec) else str(spec)
        self.a, self.P, self.rank = a, int(P), int(rank)
        uid = (C.c_char * 128).from_buffer_copy(unique_id)
        self.comm = C.c_void_p()
        _check(lib().f3rg_comm_nccl(C.byref(self.comm), C.byref(_csr(a)), self.P, self.rank, uid))
        self.solver = _PartSolver(self.comm, a, text, self.rank)
        self.plan = part_plan(a, self.P, self.rank)

    def run(self, b_own, x_own, opts: RunOptions = RunOptions(), stream: int = 0):
        """b_own, x_own: CUDA fp64 tensors of this rank's rows."""
        r = _Report()
        _check(lib().f3rg_solve_part_device(self.solver.h, b_own.data_ptr(), x_own.data_ptr(), C.byref(opts._c()),
                                            C.byref(r), stream))
        return self.solver._report(r)

    def reset(self) -> None:
        self.solver.reset()

    def __del__(self):
        if getattr(self, "solver", None) is not None:
            self.solver.__del__()
            self.solver = None
        if getattr(self, "comm", None) and self.comm.value:
            lib().f3rg_comm_destroy(self.comm)
            self.comm = None
