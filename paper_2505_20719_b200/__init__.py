"""B200-native F3R hot path (arXiv 2505.20719): nested fp64 FGMRES > fp32 FGMRES >
fp16-matrix FGMRES > fp16 Richardson with adaptive weight, as hand-written sm_100a
CUDA behind a C ABI (include/f3rg.h, lib/libf3rg.so).

This module is the Python mirror of the reference's C++ interface for the path
(/root/reference/proj/include/f3r/*.hpp) -- same names, argument meaning and
error classes -- so tests read like the reference's own:

    reps = make_replicas(SparseCsr(n, row_ptr, col_idx, values))   # csr.hpp:72-81
    solver = build_f3r(F3rConfig(), reps, IdentityPrecond(n))       # nesting.hpp:93-95
    run = solver.run(b, RunOptions(tol=1e-10))                      # nesting.hpp:64
    run.report.outer_iterations, run.x

Device memory, streams and vectors are torch CUDA tensors (plumbing only); all
arithmetic runs in libf3rg.so. There is no CPU fallback: importing without the
built library, or calling without a GPU, raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# F3RG_LIB selects a tuning-sweep build (lib/variants/); default is the product library
LIB_PATH = os.environ.get("F3RG_LIB") or os.path.join(_HERE, "lib", "libf3rg.so")


# ---------------------------------------------------------------- errors (errors.hpp)
class F3rError(RuntimeError):
    """f3r::Error"""


class ParseError(F3rError):
    """f3r::ParseError -- malformed solver spec"""


class DimensionError(F3rError):
    """f3r::DimensionError -- size mismatch / invalid CSR"""


class FactorizationError(F3rError):
    """f3r::FactorizationError"""


class SolverError(F3rError):
    """f3r::SolverError -- structural solver failures (m < 1, precision increase, ...)"""


class UnsupportedError(SolverError):
    """Valid reference input that this device build does not implement (e.g. ILU(0) M)."""


class CudaError(F3rError):
    """CUDA runtime failure (no reference counterpart)."""


_ERRS = {2: DimensionError, 3: SolverError, 4: ParseError, 5: FactorizationError, 6: CudaError,
         7: UnsupportedError, 9: F3rError}


# ------------------------------------------------------------------ library loading
class _Report(C.Structure):
    _fields_ = [("converged", C.c_int32), ("outer_iterations", C.c_uint64), ("precond_invocations", C.c_uint64),
                ("final_true_residual", C.c_double), ("wall_seconds", C.c_double), ("n_history", C.c_uint64),
                ("n_levels", C.c_uint64), ("n_omegas", C.c_uint64), ("flag", C.c_char * 128)]


class _Csr(C.Structure):
    _fields_ = [("n", C.c_uint64), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p)]


class _IluCfg(C.Structure):
    _fields_ = [("nblocks", C.c_uint64), ("alpha", C.c_double), ("symmetric", C.c_int32),
                ("apply_precision", C.c_int32)]


class _RunOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_outer_restarts", C.c_int32), ("max_outer_total", C.c_uint64),
                ("reset_richardson_on_restart", C.c_int32)]


_lib = None


def lib():
    """Loads libf3rg.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2505_20719_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, u64, i32, dbl = C.c_void_p, C.c_uint64, C.c_int, C.c_double
    L.f3rg_last_error.restype = C.c_char_p
    L.f3rg_set_seq_reductions.argtypes = [i32]
    L.f3rg_matrix_stream_bytes.argtypes = [vp, i32]
    L.f3rg_matrix_stream_bytes.restype = u64
    L.f3rg_version.restype = C.c_char_p
    L.f3rg_matrix_create.argtypes = [C.POINTER(vp), C.POINTER(_Csr)]
    L.f3rg_matrix_destroy.argtypes = [vp]
    L.f3rg_matrix_rows.restype = u64
    L.f3rg_matrix_rows.argtypes = [vp]
    L.f3rg_matrix_nnz.restype = u64
    L.f3rg_matrix_nnz.argtypes = [vp]
    L.f3rg_matrix_values.argtypes = [vp, i32, vp]
    L.f3rg_matrix_engine.argtypes = [vp]
    L.f3rg_matrix_engine.restype = i32
    L.f3rg_wsell_pk_selfcheck.argtypes = [u64, vp, vp, C.c_uint32, vp]
    L.f3rg_wsell_pk_selfcheck.restype = i32
    L.f3rg_spec_canonical.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
    L.f3rg_solver_create.argtypes = [C.POINTER(vp), vp, C.c_char_p, i32]
    L.f3rg_solver_destroy.argtypes = [vp]
    L.f3rg_solver_id.restype = C.c_char_p
    L.f3rg_solver_id.argtypes = [vp]
    L.f3rg_solve.argtypes = [vp, vp, vp, C.POINTER(_RunOpts), C.POINTER(_Report)]
    L.f3rg_solve_device.argtypes = [vp, vp, vp, C.POINTER(_RunOpts), C.POINTER(_Report), C.c_size_t]
    L.f3rg_solver_history.argtypes = [vp, vp, u64]
    L.f3rg_solver_reset_state.argtypes = [vp, C.c_size_t]
    L.f3rg_solver_level_iterations.argtypes = [vp, vp, u64]
    L.f3rg_solver_omegas.argtypes = [vp, vp, u64]
    L.f3rg_solver_omega_count.restype = u64
    L.f3rg_solver_omega_count.argtypes = [vp]
    L.f3rg_krylov_solve.argtypes = [vp, i32, vp, vp, dbl, u64, C.POINTER(_Report), vp, u64]
    L.f3rg_krylov_solve_m.argtypes = [vp, vp, i32, vp, vp, dbl, u64, C.POINTER(_Report), vp, u64]
    # row-block partition (partition.py)
    L.f3rg_part_plan.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp]
    L.f3rg_comm_local.argtypes = [C.POINTER(vp), vp, i32]
    L.f3rg_nccl_unique_id.argtypes = [vp]
    L.f3rg_comm_nccl.argtypes = [C.POINTER(vp), vp, i32, i32, vp]
    L.f3rg_comm_destroy.argtypes = [vp]
    L.f3rg_solver_create_part.argtypes = [C.POINTER(vp), vp, vp, C.c_char_p, i32, i32]
    L.f3rg_solve_local.argtypes = [vp, vp, vp, vp, C.POINTER(_RunOpts), vp]
    L.f3rg_solve_part_device.argtypes = [vp, vp, vp, C.POINTER(_RunOpts), C.POINTER(_Report), C.c_size_t]
    L.f3rg_local_spmv.argtypes = [vp, i32, i32, i32, i32, vp, vp]
    L.f3rg_solver_set_profile.argtypes = [vp, i32]
    L.f3rg_solver_profile_entry.argtypes = [vp, u64, C.c_char_p, C.c_size_t, C.POINTER(dbl), C.POINTER(u64),
                                            C.POINTER(dbl)]
    L.f3rg_spmv.argtypes = [vp, i32, vp, i32, vp, i32, C.c_size_t]
    L.f3rg_dot.argtypes = [vp, i32, vp, i32, u64, i32, C.POINTER(dbl), C.c_size_t]
    L.f3rg_norm2.argtypes = [vp, i32, u64, C.POINTER(dbl), C.c_size_t]
    L.f3rg_axpy.argtypes = [dbl, vp, i32, vp, i32, u64, C.c_size_t]
    L.f3rg_add_scaled.argtypes = [vp, i32, dbl, vp, i32, vp, i32, u64, C.c_size_t]
    L.f3rg_copy.argtypes = [vp, i32, vp, i32, u64, C.c_size_t]
    L.f3rg_scale.argtypes = [dbl, vp, i32, u64, C.c_size_t]
    L.f3rg_fill.argtypes = [vp, i32, u64, dbl, C.c_size_t]
    L.f3rg_richardson_create.argtypes = [C.POINTER(vp), vp, i32, i32, u64]
    L.f3rg_richardson_destroy.argtypes = [vp]
    L.f3rg_richardson_set_omegas.argtypes = [vp, vp]
    L.f3rg_richardson_state.argtypes = [vp, vp, vp]
    L.f3rg_richardson_apply.argtypes = [vp, vp, vp, C.c_size_t]
    L.f3rg_richardson_set_precond.argtypes = [vp, vp]
    # primary preconditioner (ilu.hpp)
    L.f3rg_ilu_factorize.argtypes = [C.POINTER(vp), C.POINTER(_Csr), C.POINTER(_IluCfg)]
    L.f3rg_precond_identity.argtypes = [C.POINTER(vp), u64]
    L.f3rg_precond_destroy.argtypes = [vp]
    L.f3rg_precond_rows.restype = u64
    L.f3rg_precond_rows.argtypes = [vp]
    L.f3rg_precond_info.argtypes = [vp, C.POINTER(_IluCfg), vp, vp, u64]
    L.f3rg_precond_apply.argtypes = [vp, vp, i32, vp, i32, C.c_size_t]
    L.f3rg_ilu_factorize_host.argtypes = [C.POINTER(_Csr), C.POINTER(_IluCfg), C.POINTER(u64), C.POINTER(u64), vp, vp,
                                          vp, vp, vp, vp]
    L.f3rg_solver_create_m.argtypes = [C.POINTER(vp), vp, C.c_char_p, vp]
    L.f3rg_matrix_create_scaled.argtypes = [C.POINTER(vp), C.POINTER(_Csr), vp, vp, vp]
    L.f3rg_read_matrix_market.argtypes = [C.c_char_p, C.POINTER(vp)]
    L.f3rg_host_csr_view.argtypes = [vp, C.POINTER(_Csr)]
    L.f3rg_host_csr_nnz.restype = u64
    L.f3rg_host_csr_nnz.argtypes = [vp]
    L.f3rg_host_csr_destroy.argtypes = [vp]
    L.f3rg_write_matrix_market.argtypes = [C.c_char_p, C.POINTER(_Csr)]
    L.f3rg_fgmres_solve.argtypes = [vp, vp, i32, vp, vp, dbl, u64, C.POINTER(_Report), vp, u64]
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        msg = lib().f3rg_last_error().decode()
        raise _ERRS.get(rc, F3rError)(msg)


# ------------------------------------------------------------ precision (precision.hpp)
class Precision(enum.IntEnum):
    P16 = 0
    P32 = 1
    P64 = 2


def compute_precision(a: Precision, b: Precision) -> Precision:
    return Precision(max(int(a), int(b)))


def precision_name(p) -> str:
    return ("f16", "f32", "f64")[int(p)]


def _torch():
    import torch  # plumbing: device memory and streams
    return torch


def _prec_of(t) -> Precision:
    torch = _torch()
    m = {torch.float16: Precision.P16, torch.float32: Precision.P32, torch.float64: Precision.P64}
    if t.dtype not in m:
        raise DimensionError(f"unsupported dtype {t.dtype}")
    if not t.is_cuda:
        raise DimensionError("device vectors must be CUDA tensors")
    return m[t.dtype]


def torch_dtype(p):
    torch = _torch()
    return (torch.float16, torch.float32, torch.float64)[int(p)]


def _stream():
    torch = _torch()
    return torch.cuda.current_stream().cuda_stream


# ------------------------------------------------------------------ vectors (dense_vector.hpp)
class DenseVector:
    """Device vector with a runtime precision (reference DenseVector,
    include/f3r/dense_vector.hpp:25-57), backed by a torch CUDA tensor."""

    def __init__(self, n_or_tensor, precision: Precision = Precision.P64):
        torch = _torch()
        if isinstance(n_or_tensor, int):
            self.t = torch.zeros(n_or_tensor, dtype=torch_dtype(precision), device="cuda")
        elif isinstance(n_or_tensor, np.ndarray):
            self.t = torch.from_numpy(np.ascontiguousarray(n_or_tensor)).to(
                device="cuda", dtype=torch_dtype(precision))
        else:
            self.t = n_or_tensor.contiguous()
            _prec_of(self.t)

    def precision(self) -> Precision:
        return _prec_of(self.t)

    def size(self) -> int:
        return self.t.numel()

    def __len__(self):
        return self.t.numel()

    def numpy(self) -> np.ndarray:
        """exact widening to fp64"""
        return self.t.double().cpu().numpy()

    def ptr(self) -> int:
        return self.t.data_ptr()


def _vec(x) -> DenseVector:
    return x if isinstance(x, DenseVector) else DenseVector(x)


def fill(x: DenseVector, value: float) -> None:
    _check(lib().f3rg_fill(x.ptr(), x.precision(), x.size(), value, _stream()))


def copy_into(x: DenseVector, y: DenseVector) -> None:
    if x.size() != y.size():
        raise DimensionError(f"copy: length mismatch ({x.size()} vs {y.size()})")
    _check(lib().f3rg_copy(x.ptr(), x.precision(), y.ptr(), y.precision(), x.size(), _stream()))


def converted(x: DenseVector, p: Precision) -> DenseVector:
    out = DenseVector(x.size(), p)
    copy_into(x, out)
    return out


def scale_in_place(alpha: float, x: DenseVector) -> None:
    _check(lib().f3rg_scale(alpha, x.ptr(), x.precision(), x.size(), _stream()))


def axpy(alpha: float, x: DenseVector, y: DenseVector) -> None:
    if x.size() != y.size():
        raise DimensionError(f"axpy: length mismatch ({x.size()} vs {y.size()})")
    _check(lib().f3rg_axpy(alpha, x.ptr(), x.precision(), y.ptr(), y.precision(), x.size(), _stream()))


def add_scaled(x: DenseVector, alpha: float, y: DenseVector, out: DenseVector) -> None:
    if x.size() != y.size() or x.size() != out.size():
        raise DimensionError("add_scaled: length mismatch")
    _check(lib().f3rg_add_scaled(x.ptr(), x.precision(), alpha, y.ptr(), y.precision(), out.ptr(),
                                 out.precision(), x.size(), _stream()))


def dot_at_least(x: DenseVector, y: DenseVector, floor_precision: Precision) -> float:
    if x.size() != y.size():
        raise DimensionError(f"dot: length mismatch ({x.size()} vs {y.size()})")
    out = C.c_double()
    _check(lib().f3rg_dot(x.ptr(), x.precision(), y.ptr(), y.precision(), x.size(), int(floor_precision),
                          C.byref(out), _stream()))
    return out.value


class seq_reductions:
    """Validation mode: every dot / norm summed sequentially in index order, as the
    reference's dot_core (src/vector_ops.cpp:20-28), instead of the fixed-shape
    tree. Applies to kernels launched and solvers built inside the block:

        with seq_reductions():
            solver = build(spec, reps, M)
            run = solver.run(b, opts)
    """

    def __init__(self, on: bool = True):
        self.on = on
        self.old = None

    def __enter__(self):
        self.old = lib().f3rg_set_seq_reductions(1 if self.on else 0)
        return self

    def __exit__(self, *a):
        lib().f3rg_set_seq_reductions(self.old)


def dot(x: DenseVector, y: DenseVector) -> float:
    return dot_at_least(x, y, Precision.P16)


def norm2(x: DenseVector) -> float:
    out = C.c_double()
    _check(lib().f3rg_norm2(x.ptr(), x.precision(), x.size(), C.byref(out), _stream()))
    return out.value


# --------------------------------------------------------------------- matrices (csr.hpp)
class SparseCsr:
    """Host fp64 CSR with u32 indices (reference SparseCsr, include/f3r/csr.hpp:23-67).
    Validation happens when the device replicas are built (make_replicas)."""

    def __init__(self, n: int, row_ptr, col_idx, values):
        self.n = int(n)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.uint32)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.uint32)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        if self.row_ptr.size != self.n + 1:
            raise DimensionError("row_ptr length must be n+1")
        if self.values.size != self.col_idx.size:
            raise DimensionError("values length must equal nnz")

    def rows(self) -> int:
        return self.n

    def nnz(self) -> int:
        return int(self.col_idx.size)


class _DeviceMatrix:
    def __init__(self, a: SparseCsr, handle=None):
        L = lib()
        self.h = C.c_void_p()
        if handle is not None:
            self.h = handle
        else:
            csr = _Csr(a.n, a.row_ptr.ctypes.data, a.col_idx.ctypes.data, a.values.ctypes.data)
            _check(L.f3rg_matrix_create(C.byref(self.h), C.byref(csr)))
        self.n = a.n
        self.nnz_ = a.nnz()

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.f3rg_matrix_destroy(self.h)
            self.h = None


class ReplicaView:
    """One precision of PrecisionReplicas (what PrecisionReplicas::at returns)."""

    def __init__(self, dev: _DeviceMatrix, p: Precision):
        self.dev, self.p = dev, Precision(p)

    def precision(self) -> Precision:
        return self.p

    def rows(self) -> int:
        return self.dev.n

    def nnz(self) -> int:
        return self.dev.nnz_

    def values(self) -> np.ndarray:
        """replica values widened to fp64 (exact)"""
        out = np.zeros(self.dev.nnz_)
        _check(lib().f3rg_matrix_values(self.dev.h, self.p, out.ctypes.data))
        return out


class PrecisionReplicas:
    """reference PrecisionReplicas (include/f3r/csr.hpp:72-78): one device copy of the
    indices, fp64 / fp32 / fp16 value arrays (RNE demotions of a64)."""

    def __init__(self, a64: SparseCsr, _dev=None):
        self.host = a64
        self.dev = _dev if _dev is not None else _DeviceMatrix(a64)
        self.a64 = ReplicaView(self.dev, Precision.P64)
        self.a32 = ReplicaView(self.dev, Precision.P32)
        self.a16 = ReplicaView(self.dev, Precision.P16)

    def at(self, p: Precision) -> ReplicaView:
        return (self.a16, self.a32, self.a64)[int(p)]

    def rows(self) -> int:
        return self.dev.n

    def stream_bytes(self, p: Precision) -> int:
        """bytes one device pass over replica p streams (compressed column stream)"""
        return int(lib().f3rg_matrix_stream_bytes(self.dev.h, int(p)))

    def engine(self) -> int:
        """SpMV engine of the device layout: 0/1 row tiles, 2 row tiles over the
        row-sorted copy, 3 windowed SELL (f3rg_matrix_engine)"""
        return int(lib().f3rg_matrix_engine(self.dev.h))


def make_replicas(a64: SparseCsr) -> PrecisionReplicas:
    return PrecisionReplicas(a64)


@dataclass
class ScaledSystem:
    """reference ScaledSystem (include/f3r/scaling.hpp): the scaled matrix -- here its
    device replicas --, the scaled right-hand side and d"""
    replicas: PrecisionReplicas
    rhs: np.ndarray
    d: np.ndarray


def diagonal_scale(a: SparseCsr, b) -> ScaledSystem:
    """reference diagonal_scale(A, b) (src/scaling.cpp:11-38) computed on the device
    from the unscaled matrix, bit-identical; the replicas are built from the scaled
    values in the same pass. Raises FactorizationError on a missing / zero diagonal."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.size != a.n:
        raise DimensionError("diagonal scaling: rhs length mismatch")
    h = C.c_void_p()
    bs, d = np.zeros(a.n), np.zeros(a.n)
    csr = _Csr(a.n, a.row_ptr.ctypes.data, a.col_idx.ctypes.data, a.values.ctypes.data)
    _check(lib().f3rg_matrix_create_scaled(C.byref(h), C.byref(csr), b.ctypes.data, bs.ctypes.data, d.ctypes.data))
    dev = _DeviceMatrix(a, handle=h)
    vals = np.zeros(a.nnz())
    _check(lib().f3rg_matrix_values(h, 2, vals.ctypes.data))
    return ScaledSystem(PrecisionReplicas(SparseCsr(a.n, a.row_ptr, a.col_idx, vals), _dev=dev), bs, d)


def wsell_pk_selfcheck(n: int, row_ptr, col_idx, ctas: int = 148) -> dict:
    """Builds the packed windowed SELL layout (csrc/wsell_pk_layout.hpp) of a CSR pattern on
    the host and decodes every row back against the CSR (no GPU needed); raises
    DimensionError on the first mismatch. Returns the layout's slot / far / slice / padding counts."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.uint32)
    ci = np.ascontiguousarray(col_idx, dtype=np.uint32)
    stats = np.zeros(4, dtype=np.uint64)
    _check(lib().f3rg_wsell_pk_selfcheck(int(n), rp.ctypes.data, ci.ctypes.data, int(ctas), stats.ctypes.data))
    return {"slots": int(stats[0]), "far": int(stats[1]), "slices": int(stats[2]), "padding": int(stats[3])}


def read_matrix_market(path: str) -> SparseCsr:
    """reference read_matrix_market (src/matrix_market.cpp:33-113); raises ParseError"""
    L = lib()
    h = C.c_void_p()
    _check(L.f3rg_read_matrix_market(str(path).encode(), C.byref(h)))
    try:
        v = _Csr()
        _check(L.f3rg_host_csr_view(h, C.byref(v)))
        nnz = int(L.f3rg_host_csr_nnz(h))
        n = int(v.n)
        rp = np.ctypeslib.as_array(C.cast(v.row_ptr, C.POINTER(C.c_uint32)), shape=(n + 1,)).copy()
        ci = np.ctypeslib.as_array(C.cast(v.col_idx, C.POINTER(C.c_uint32)), shape=(max(nnz, 1),))[:nnz].copy()
        va = np.ctypeslib.as_array(C.cast(v.values, C.POINTER(C.c_double)), shape=(max(nnz, 1),))[:nnz].copy()
        return SparseCsr(n, rp, ci, va)
    finally:
        L.f3rg_host_csr_destroy(h)


def write_matrix_market(path: str, a: SparseCsr) -> None:
    """reference write_matrix_market (src/matrix_market.cpp:115-127)"""
    csr = _Csr(a.n, a.row_ptr.ctypes.data, a.col_idx.ctypes.data, a.values.ctypes.data)
    _check(lib().f3rg_write_matrix_market(str(path).encode(), C.byref(csr)))


def spmv(a: ReplicaView, x: DenseVector, y: DenseVector) -> None:
    """y = A x at compute_precision(A, x), stored at y's precision (src/csr.cpp:138-147)."""
    if x.size() != a.rows() or y.size() != a.rows():
        raise DimensionError("spmv: dimension mismatch")
    _check(lib().f3rg_spmv(a.dev.h, a.p, x.ptr(), x.precision(), y.ptr(), y.precision(), _stream()))


# ------------------------------------------------------------ preconditioner (ilu.hpp)
class Preconditioner:
    """reference Preconditioner (include/f3r/ilu.hpp:25-32): z = M r on the device."""
    kind = 2
    h = None

    def rows(self) -> int:
        return self.n

    def apply(self, r: DenseVector, z: DenseVector) -> None:
        """z ~= A^{-1} r at compute_precision(factors, r), stored at z's precision."""
        if r.size() != self.n or z.size() != self.n:
            raise DimensionError("preconditioner apply: size mismatch")
        _check(lib().f3rg_precond_apply(self._handle(), r.ptr(), r.precision(), z.ptr(), z.precision(), _stream()))

    def _handle(self):
        if self.h is None:
            self.h = C.c_void_p()
            _check(lib().f3rg_precond_identity(C.byref(self.h), self.n))
        return self.h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.f3rg_precond_destroy(self.h)
            self.h = None


class IdentityPrecond(Preconditioner):
    """reference IdentityPrecond (include/f3r/ilu.hpp:34-42): apply = copy_into."""
    kind = 2

    def __init__(self, n: int):
        self.n = int(n)


@dataclass
class IluConfig:
    """reference IluConfig (include/f3r/ilu.hpp:44-49)"""
    nblocks: int = 1
    alpha: float = 1.0
    symmetric: bool = False
    apply_precision: Precision = Precision.P64

    def _c(self):
        return _IluCfg(int(self.nblocks), float(self.alpha), int(bool(self.symmetric)), int(self.apply_precision))


class BlockJacobiIlu0(Preconditioner):
    """reference BlockJacobiIlu0 (include/f3r/ilu.hpp:51-84): block-Jacobi ILU(0) /
    IC(0), factorised on the host at fp64 (src/ilu.cpp:38-185); apply runs the two
    triangular sweeps on the device, bit-exact with the reference's sequential
    ones (src/ilu.cpp:187-263)."""

    def __init__(self, h, n: int, cfg: IluConfig):
        self.h, self.n, self._cfg = h, int(n), cfg
        self.kind = 1 if cfg.symmetric else 0

    @staticmethod
    def factorize(a: SparseCsr, cfg: IluConfig) -> "BlockJacobiIlu0":
        """Raises FactorizationError naming the block and row, as the reference."""
        h = C.c_void_p()
        csr = _Csr(a.n, a.row_ptr.ctypes.data, a.col_idx.ctypes.data, a.values.ctypes.data)
        _check(lib().f3rg_ilu_factorize(C.byref(h), C.byref(csr), C.byref(cfg._c())))
        return BlockJacobiIlu0(h, a.n, cfg)

    def config(self) -> IluConfig:
        return self._cfg

    def _info(self):
        cfg = _IluCfg()
        lev = np.zeros(2, dtype=np.uint32)
        br = np.zeros(int(self._cfg.nblocks) + 1, dtype=np.uint32)
        _check(lib().f3rg_precond_info(self.h, C.byref(cfg), lev.ctypes.data, br.ctypes.data, br.size))
        return lev, br

    def block_ranges(self) -> list:
        return [int(v) for v in self._info()[1]]

    def sweep_levels(self) -> tuple:
        """dependency depth of the forward and backward sweeps (the device critical path)"""
        lev = self._info()[0]
        return int(lev[0]), int(lev[1])


def ilu_factorize_host(a: SparseCsr, cfg: IluConfig):
    """The product's host factorisation alone (no GPU): ((lp, li, lv), (up, ui, uv)),
    the stored factors as the reference keeps them."""
    csr = _Csr(a.n, a.row_ptr.ctypes.data, a.col_idx.ctypes.data, a.values.ctypes.data)
    nl, nu = C.c_uint64(), C.c_uint64()
    L = lib()
    _check(L.f3rg_ilu_factorize_host(C.byref(csr), C.byref(cfg._c()), C.byref(nl), C.byref(nu), None, None, None,
                                     None, None, None))
    lp, up = np.zeros(a.n + 1, np.uint32), np.zeros(a.n + 1, np.uint32)
    li, ui = np.zeros(max(1, nl.value), np.uint32), np.zeros(max(1, nu.value), np.uint32)
    lv, uv = np.zeros(max(1, nl.value)), np.zeros(max(1, nu.value))
    _check(L.f3rg_ilu_factorize_host(C.byref(csr), C.byref(cfg._c()), None, None, lp.ctypes.data, li.ctypes.data,
                                     lv.ctypes.data, up.ctypes.data, ui.ctypes.data, uv.ctypes.data))
    return (lp, li[:nl.value], lv[:nl.value]), (up, ui[:nu.value], uv[:nu.value])


# ---------------------------------------------------------------- spec (solver_spec.hpp)
def canonical_spec(text: str) -> str:
    """parse_solver_spec(text).to_string() (src/solver_spec.cpp:147-212); raises ParseError."""
    buf = C.create_string_buffer(1024)
    _check(lib().f3rg_spec_canonical(text.encode(), buf, 1024))
    return buf.value.decode()


@dataclass
class SolverSpec:
    """A spec kept in the reference grammar; parse_solver_spec validates it."""
    text: str

    def to_string(self) -> str:
        return canonical_spec(self.text)


def parse_solver_spec(text: str) -> SolverSpec:
    canonical_spec(text)
    return SolverSpec(text)


class F3rMode(enum.Enum):
    FP64 = 0
    FP32 = 1
    FP16 = 2


@dataclass
class F3rConfig:
    """reference F3rConfig (include/f3r/nesting.hpp:84-91)"""
    m1: int = 100
    m2: int = 8
    m3: int = 4
    m4: int = 2
    c: int = 64
    mode: F3rMode = F3rMode.FP16


def f3r_spec(cfg: F3rConfig) -> SolverSpec:
    """reference f3r_spec (src/nesting.cpp:359-386), terminal = the primary
    preconditioner at the Richardson precision."""
    if cfg.mode == F3rMode.FP16:
        mid, low_m, low_v, rich = "f32", "f16", "f32", "f16"
    elif cfg.mode == F3rMode.FP32:
        mid, low_m, low_v, rich = "f32", "f32", "f32", "f32"
    else:
        mid, low_m, low_v, rich = "f64", "f64", "f64", "f64"
    return SolverSpec(f"F{cfg.m1}:f64/f64 > F{cfg.m2}:{mid}/{mid} > F{cfg.m3}:{low_m}/{low_v} > "
                      f"R{cfg.m4}:{rich},c={cfg.c} > ilu0(prec={rich})")


# --------------------------------------------------------------------- solver (nesting.hpp)
@dataclass
class RunOptions:
    """reference RunOptions (include/f3r/nesting.hpp:29-38)"""
    tol: float = 1e-8
    max_outer_restarts: int = 3
    max_outer_total: int = 300
    reset_richardson_on_restart: bool = False

    def _c(self):
        return _RunOpts(self.tol, self.max_outer_restarts, self.max_outer_total,
                        int(self.reset_richardson_on_restart))


@dataclass
class ConvergenceReport:
    """reference ConvergenceReport (include/f3r/report.hpp:18-30)"""
    converged: bool = False
    outer_iterations: int = 0
    precond_invocations: int = 0
    level_iterations: list = field(default_factory=list)
    residual_history: list = field(default_factory=list)
    final_true_residual: float = 0.0
    wall_seconds: float = 0.0
    omegas_final: list = field(default_factory=list)
    flag: str = ""
    solver_id: str = ""
    problem_id: str = ""


@dataclass
class RunResult:
    x: Optional[np.ndarray]
    report: ConvergenceReport


class ComposedSolver:
    """reference ComposedSolver (include/f3r/nesting.hpp:55-77): the whole nest runs
    on the GPU; one C-ABI call per solve."""

    def __init__(self, spec, a: PrecisionReplicas, m: Preconditioner):
        if m.rows() != a.rows():
            raise DimensionError("preconditioner size does not match the matrix")
        text = spec.text if isinstance(spec, SolverSpec) else str(spec)
        self.h = C.c_void_p()
        self._a, self._m = a, m
        _check(lib().f3rg_solver_create_m(C.byref(self.h), a.dev.h, text.encode(), m._handle()))
        self.n = a.rows()

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.f3rg_solver_destroy(self.h)
            self.h = None

    def id(self) -> str:
        return lib().f3rg_solver_id(self.h).decode()

    def _report(self, r: _Report) -> ConvergenceReport:
        L = lib()
        hist = np.zeros(max(1, r.n_history))
        L.f3rg_solver_history(self.h, hist.ctypes.data, r.n_history)
        lv = np.zeros(max(1, r.n_levels), dtype=np.uint64)
        L.f3rg_solver_level_iterations(self.h, lv.ctypes.data, r.n_levels)
        om = np.zeros(max(1, r.n_omegas))
        if r.n_omegas:
            _check(L.f3rg_solver_omegas(self.h, om.ctypes.data, r.n_omegas))
        return ConvergenceReport(bool(r.converged), int(r.outer_iterations), int(r.precond_invocations),
                                 [int(v) for v in lv[:r.n_levels]], list(hist[:r.n_history]),
                                 r.final_true_residual, r.wall_seconds, list(om[:r.n_omegas]), r.flag.decode(),
                                 self.id())

    def run(self, b, opts: RunOptions = RunOptions(), want_x: bool = True, out=None) -> RunResult:
        """b: host numpy fp64 array (host copies inside the call) or a CUDA fp64
        tensor (device-resident; x is returned as a CUDA tensor). With a host b,
        `out` (fp64 numpy array of length n, ideally in pinned memory) receives x."""
        r = _Report()
        if isinstance(b, np.ndarray):
            b = np.ascontiguousarray(b, dtype=np.float64)
            if b.size != self.n:
                raise DimensionError("run: rhs length mismatch")
            if out is not None and (out.dtype != np.float64 or out.size != self.n or not out.flags.c_contiguous):
                raise DimensionError("run: out must be a contiguous fp64 array of length n")
            x = (out if out is not None else np.zeros(self.n)) if want_x else None
            _check(lib().f3rg_solve(self.h, b.ctypes.data, x.ctypes.data if x is not None else None,
                                    C.byref(opts._c()), C.byref(r)))
            return RunResult(x, self._report(r))
        t = b.t if isinstance(b, DenseVector) else b
        if _prec_of(t) != Precision.P64 or t.numel() != self.n:
            raise DimensionError("run: rhs must be an fp64 vector of length n")
        torch = _torch()
        x = torch.empty(self.n, dtype=torch.float64, device=t.device) if want_x else None
        _check(lib().f3rg_solve_device(self.h, t.data_ptr(), x.data_ptr() if x is not None else None,
                                       C.byref(opts._c()), C.byref(r), _stream()))
        return RunResult(x, self._report(r))

    def reset(self) -> None:
        """Back to a freshly built solver (Richardson weights/counters persist across
        run() calls, as in the reference); stream-ordered, no host sync."""
        _check(lib().f3rg_solver_reset_state(self.h, _stream()))

    def innermost_omegas(self) -> list:
        """weights of the deepest Richardson level; empty when there is none"""
        cnt = int(lib().f3rg_solver_omega_count(self.h))
        om = np.zeros(max(1, cnt))
        if cnt:
            _check(lib().f3rg_solver_omegas(self.h, om.ctypes.data, cnt))
        return list(om[:cnt])

    def set_profile(self, on: bool = True) -> None:
        lib().f3rg_solver_set_profile(self.h, int(on))

    def collectives(self) -> tuple:
        """(halo exchanges, cross-rank reductions) the last profiled run enqueued"""
        h, r = C.c_uint64(), C.c_uint64()
        _check(lib().f3rg_solver_collectives(self.h, C.byref(h), C.byref(r)))
        return h.value, r.value

    def profile(self) -> list:
        """[(kernel, total_ms, launches, algorithmic_bytes)] of the last profiled run"""
        out, i = [], 0
        name = C.create_string_buffer(256)
        ms, ln, by = C.c_double(), C.c_uint64(), C.c_double()
        while lib().f3rg_solver_profile_entry(self.h, i, name, 256, C.byref(ms), C.byref(ln), C.byref(by)) == 0:
            out.append((name.value.decode(), ms.value, ln.value, by.value))
            i += 1
        return out


def build(spec, a: PrecisionReplicas, m: Preconditioner) -> ComposedSolver:
    return ComposedSolver(spec, a, m)


def build_f3r(cfg: F3rConfig, a: PrecisionReplicas, m: Preconditioner) -> ComposedSolver:
    return ComposedSolver(f3r_spec(cfg), a, m)


# ------------------------------------------------ competitor solvers (cg.hpp, src/cg.cpp)
@dataclass
class ReferenceSolveOptions:
    """reference ReferenceSolveOptions, include/f3r/cg.hpp:12-15"""
    tol: float = 1e-8
    max_precond_invocations: int = 19200


def _krylov_solve(which: int, a, m: Preconditioner, b, opts: ReferenceSolveOptions, x_out=None):
    dev = a.dev if isinstance(a, (PrecisionReplicas, ReplicaView)) else _DeviceMatrix(a)
    n = dev.n
    if m.rows() != n:
        raise DimensionError("preconditioner size does not match the matrix")
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.size != n:
        raise DimensionError("rhs length mismatch")
    if x_out is not None and (x_out.dtype != np.float64 or x_out.size != n):
        raise DimensionError("x_out must be an fp64 array of length n")
    r = _Report()
    hist = np.zeros(int(opts.max_precond_invocations) + 2)
    _check(lib().f3rg_krylov_solve_m(dev.h, None if isinstance(m, IdentityPrecond) else m._handle(), which,
                                     b.ctypes.data, x_out.ctypes.data if x_out is not None else None,
                                     float(opts.tol), int(opts.max_precond_invocations), C.byref(r),
                                     hist.ctypes.data, hist.size))
    return ConvergenceReport(bool(r.converged), int(r.outer_iterations), int(r.precond_invocations), [],
                             list(hist[:r.n_history]), r.final_true_residual, r.wall_seconds, [], r.flag.decode(),
                             "cg" if which == 0 else "bicgstab")


def cg_solve(a, m: Preconditioner, b, opts: ReferenceSolveOptions = ReferenceSolveOptions(), x_out=None):
    """reference cg_solve (include/f3r/cg.hpp:21-22, src/cg.cpp:22-75): fp64
    preconditioned CG on the device, M = identity or a BlockJacobiIlu0. Raises SolverError on an
    indefinite operator, as the reference. `x_out` optionally receives x."""
    return _krylov_solve(0, a, m, b, opts, x_out)


def bicgstab_solve(a, m: Preconditioner, b, opts: ReferenceSolveOptions = ReferenceSolveOptions(), x_out=None):
    """reference bicgstab_solve (include/f3r/cg.hpp:28-30, src/cg.cpp:77-171)."""
    return _krylov_solve(1, a, m, b, opts, x_out)


@dataclass
class FgmresOptions:
    """reference FgmresOptions, include/f3r/fgmres.hpp:41-44"""
    tol: float = 1e-8
    max_precond_invocations: int = 19200


def fgmres_restarted(a, m: Preconditioner, b, restart: int, opts: FgmresOptions = FgmresOptions(), x_out=None):
    """reference fgmres_restarted (include/f3r/fgmres.hpp:46-49, src/fgmres.cpp:163-222):
    fp64 FGMRES(restart) with the terminal preconditioner m, on the device."""
    dev = a.dev if isinstance(a, (PrecisionReplicas, ReplicaView)) else _DeviceMatrix(a)
    n = dev.n
    if m.rows() != n:
        raise DimensionError("preconditioner size does not match the matrix")
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.size != n:
        raise DimensionError("rhs length mismatch")
    r = _Report()
    hist = np.zeros(int(opts.max_precond_invocations) + 2)
    _check(lib().f3rg_fgmres_solve(dev.h, m._handle(), int(restart), b.ctypes.data,
                                   x_out.ctypes.data if x_out is not None else None, float(opts.tol),
                                   int(opts.max_precond_invocations), C.byref(r), hist.ctypes.data, hist.size))
    return ConvergenceReport(bool(r.converged), int(r.outer_iterations), int(r.precond_invocations), [],
                             list(hist[:r.n_history]), r.final_true_residual, r.wall_seconds, [], r.flag.decode(),
                             f"fgmres{int(restart)}")


# ------------------------------------------------------------- Richardson (richardson.hpp)
class RichardsonState:
    """Persistent Richardson state on the device (reference RichardsonState,
    include/f3r/richardson.hpp:26-46) bound to one replica; M = identity."""

    def __init__(self, a: ReplicaView, m: int, cycle: int):
        self.h = C.c_void_p()
        _check(lib().f3rg_richardson_create(C.byref(self.h), a.dev.h, int(a.p), int(m), int(cycle)))
        self.a, self.m_inner, self.cycle = a, int(m), int(cycle)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.f3rg_richardson_destroy(self.h)
            self.h = None

    @property
    def omegas(self) -> list:
        return self._state()[0]

    @omegas.setter
    def omegas(self, w: Sequence[float]):
        w = np.ascontiguousarray(w, dtype=np.float64)
        _check(lib().f3rg_richardson_set_omegas(self.h, w.ctypes.data))

    def _state(self):
        om = np.zeros(self.m_inner)
        cnt = np.zeros(3, dtype=np.uint64)
        _check(lib().f3rg_richardson_state(self.h, om.ctypes.data, cnt.ctypes.data))
        return list(om), [int(c) for c in cnt]

    @property
    def call_count(self) -> int:
        return self._state()[1][0]

    @property
    def update_count(self) -> int:
        return self._state()[1][1]

    @property
    def degenerate_events(self) -> int:
        return self._state()[1][2]


def richardson_apply(state: RichardsonState, v: DenseVector, z: DenseVector, m: Preconditioner = None) -> None:
    """reference richardson_apply (src/richardson.cpp:10-54) on the operator
    (A, M): M = identity by default, else the given preconditioner."""
    want = m.h if (m is not None and not isinstance(m, IdentityPrecond)) else None
    if getattr(state, "_m", None) is not want:
        _check(lib().f3rg_richardson_set_precond(state.h, want))
        state._m = want
    if v.precision() != state.a.p or z.precision() != state.a.p:
        raise DimensionError("richardson: vectors must be at the state's precision")
    if v.size() != state.a.rows() or z.size() != state.a.rows():
        raise DimensionError("richardson: dimension mismatch")
    _check(lib().f3rg_richardson_apply(state.h, v.ptr(), z.ptr(), _stream()))


__all__ = [
    "F3rError", "ParseError", "DimensionError", "FactorizationError", "SolverError", "UnsupportedError",
    "CudaError", "Precision", "compute_precision", "precision_name", "DenseVector", "fill", "copy_into",
    "converted", "scale_in_place", "axpy", "add_scaled", "dot", "dot_at_least", "norm2", "SparseCsr",
    "PrecisionReplicas", "make_replicas", "spmv", "Preconditioner", "IdentityPrecond", "IluConfig",
    "BlockJacobiIlu0", "ilu_factorize_host", "SolverSpec", "parse_solver_spec",
    "canonical_spec", "F3rMode", "F3rConfig", "f3r_spec", "RunOptions", "ConvergenceReport", "RunResult",
    "ComposedSolver", "build", "build_f3r", "RichardsonState", "richardson_apply", "lib", "FgmresOptions",
    "fgmres_restarted", "ReferenceSolveOptions", "cg_solve", "bicgstab_solve", "ScaledSystem", "diagonal_scale",
    "read_matrix_market", "write_matrix_market",
]
