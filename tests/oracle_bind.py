"""ctypes bindings for the CPU checkers under oracle/ -- TEST INFRASTRUCTURE ONLY.

Two libraries:
  * ``Oracle``    -- oracle/liboracle_f3r.so, our plain-C restatement (f3r_oracle.c);
  * ``Reference`` -- oracle/_ref/libf3r_ref.so, the UNMODIFIED reference sources
                     (/root/reference/proj/src) plus the ref_shim.cpp C-ABI veneer.
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module.
Vectors are float64 numpy arrays holding values representable at their
precision tag (0 = f16, 1 = f32, 2 = f64).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle_f3r.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libf3r_ref.so")

P16, P32, P64 = 0, 1, 2
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


@dataclass
class Report:
    converged: bool
    outer_iterations: int
    precond_invocations: int
    final_true_residual: float
    level_iterations: list
    residual_history: list
    omegas_final: list
    flag: str
    wall_seconds: float = 0.0
    solver_id: str = ""
    x: np.ndarray | None = field(default=None, repr=False)


class _OrLevel(C.Structure):
    _fields_ = [("kind", C.c_int), ("m", C.c_int), ("pa", C.c_int), ("pv", C.c_int), ("cycle", C.c_uint64),
                ("has_omega", C.c_int), ("omega", C.c_double)]


class _OrReport(C.Structure):
    _fields_ = [("converged", C.c_int), ("outer_iterations", C.c_uint64), ("precond_invocations", C.c_uint64),
                ("final_true_residual", C.c_double), ("n_levels", C.c_uint64),
                ("level_iterations", C.c_uint64 * 16), ("n_history", C.c_uint64), ("n_omegas", C.c_uint64),
                ("omegas", C.c_double * 64), ("flag", C.c_char * 128)]


class _RefReport(C.Structure):
    _fields_ = [("converged", C.c_int), ("outer_iterations", C.c_uint64), ("precond_invocations", C.c_uint64),
                ("final_true_residual", C.c_double), ("wall_seconds", C.c_double), ("n_levels", C.c_uint64),
                ("level_iterations", C.c_uint64 * 16), ("n_history", C.c_uint64), ("n_omegas", C.c_uint64),
                ("omegas", C.c_double * 64), ("flag", C.c_char * 128), ("id", C.c_char * 256)]


class Oracle:
    """Our C restatement of the reference algorithm (oracle/f3r_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle liboracle`)")
        L = self.lib = C.CDLL(path)
        L.or_half_from_double.restype = C.c_uint16
        L.or_half_from_double.argtypes = [C.c_double]
        L.or_half_from_float.restype = C.c_uint16
        L.or_half_from_float.argtypes = [C.c_float]
        L.or_float_from_half.restype = C.c_float
        L.or_float_from_half.argtypes = [C.c_uint16]
        L.or_round.restype = C.c_double
        L.or_round.argtypes = [C.c_int, C.c_double]
        L.or_spmv.argtypes = [C.c_uint64, _u32p, _u32p, _dp, C.c_int, _dp, C.c_int, _dp, C.c_int]
        L.or_dot.restype = C.c_double
        L.or_dot.argtypes = [_dp, C.c_int, _dp, C.c_int, C.c_uint64, C.c_int]
        L.or_norm2.restype = C.c_double
        L.or_norm2.argtypes = [_dp, C.c_int, C.c_uint64]
        L.or_axpy.argtypes = [C.c_double, _dp, C.c_int, _dp, C.c_int, C.c_uint64]
        L.or_add_scaled.argtypes = [_dp, C.c_int, C.c_double, _dp, C.c_int, _dp, C.c_int, C.c_uint64]
        L.or_copy.argtypes = [_dp, C.c_int, _dp, C.c_int, C.c_uint64]
        L.or_scale.argtypes = [C.c_double, _dp, C.c_int, C.c_uint64]
        L.or_parse_spec.restype = C.c_int
        L.or_parse_spec.argtypes = [C.c_char_p, C.POINTER(_OrLevel), C.c_int]
        L.or_solve.restype = C.c_int
        L.or_solve.argtypes = [C.c_uint64, _u32p, _u32p, _dp, C.POINTER(_OrLevel), C.c_int, _dp, C.c_double,
                               C.c_int, C.c_uint64, C.c_int, _dp, _dp, C.c_uint64, C.POINTER(_OrReport)]
        L.or_richardson_apply.argtypes = [C.c_uint64, _u32p, _u32p, _dp, C.c_int, C.c_int, C.c_uint64, _dp,
                                          C.POINTER(C.c_uint64), _dp, _dp]
        L.or_ilu_factorize.restype = C.c_int
        L.or_ilu_factorize.argtypes = [C.c_uint64, _u32p, _u32p, _dp, C.c_uint64, C.c_double, C.c_int, C.c_int,
                                       C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
        L.or_ilu_free.argtypes = [C.c_void_p]
        L.or_ilu_apply.argtypes = [C.c_void_p, _dp, C.c_int, _dp, C.c_int]
        L.or_ilu_count.restype = C.c_uint64
        L.or_ilu_count.argtypes = [C.c_void_p, C.c_int]
        L.or_ilu_export.argtypes = [C.c_void_p, C.c_int, _u32p, _u32p, _dp]
        L.or_solve_m.restype = C.c_int
        L.or_solve_m.argtypes = [C.c_uint64, _u32p, _u32p, _dp, C.POINTER(_OrLevel), C.c_int, C.c_void_p, _dp,
                                 C.c_double, C.c_int, C.c_uint64, C.c_int, _dp, _dp, C.c_uint64,
                                 C.POINTER(_OrReport)]
        L.or_richardson_apply_m.argtypes = [C.c_uint64, _u32p, _u32p, _dp, C.c_int, C.c_int, C.c_uint64,
                                            C.c_void_p, _dp, C.POINTER(C.c_uint64), _dp, _dp]
        L.or_fgmres_cycle.restype = C.c_int
        L.or_fgmres_cycle.argtypes = [C.c_uint64, _u32p, _u32p, _dp, C.c_int, C.c_int, _dp, _dp, C.c_int,
                                      C.c_double, C.c_int, C.c_int, C.POINTER(C.c_int), _dp, C.POINTER(C.c_int)]

    # -- scalars / rounding
    def half_from_double(self, x):
        return self.lib.or_half_from_double(float(x))

    def round(self, p, x):
        x = _f64(x)
        return np.array([self.lib.or_round(p, float(v)) for v in x.ravel()]).reshape(x.shape)

    def round_vec(self, p, x):
        """Vectorised demotion using numpy (only valid for f32/f64; f16 via the C path)."""
        x = _f64(x)
        if p == P64:
            return x.copy()
        if p == P32:
            return x.astype(np.float32).astype(np.float64)
        y = np.empty_like(x)
        self.lib.or_copy(x, P64, y, P16, x.size)
        return y

    # -- kernels
    def spmv(self, a, vals_p, pa, x, px, py):
        n, rp, ci = a
        y = np.zeros(n)
        self.lib.or_spmv(n, _u32(rp), _u32(ci), _f64(vals_p), pa, _f64(x), px, y, py)
        return y

    def dot(self, x, px, y, py, floor=P16):
        return self.lib.or_dot(_f64(x), px, _f64(y), py, len(x), floor)

    def norm2(self, x, px):
        return self.lib.or_norm2(_f64(x), px, len(x))

    def axpy(self, alpha, x, px, y, py):
        y = _f64(y).copy()
        self.lib.or_axpy(alpha, _f64(x), px, y, py, len(y))
        return y

    def add_scaled(self, x, px, alpha, y, py, po):
        out = np.zeros(len(x))
        self.lib.or_add_scaled(_f64(x), px, alpha, _f64(y), py, out, po, len(x))
        return out

    def copy(self, x, px, py):
        y = np.zeros(len(x))
        self.lib.or_copy(_f64(x), px, y, py, len(x))
        return y

    def scale(self, alpha, x, px):
        x = _f64(x).copy()
        self.lib.or_scale(alpha, x, px, len(x))
        return x

    def parse_spec(self, spec: str):
        levels = (_OrLevel * 16)()
        nl = self.lib.or_parse_spec(spec.encode(), levels, 16)
        if nl < 0:
            raise ValueError(f"oracle cannot parse spec {spec!r}")
        return levels, nl

    def ilu(self, a, vals64, nblocks, alpha=1.0, symmetric=False, prec=P64):
        """BlockJacobiIlu0::factorize (src/ilu.cpp:38-185) -> OracleIlu; raises
        FactorizationFailed carrying the reference's message."""
        n, rp, ci = a
        h = C.c_void_p()
        err = C.create_string_buffer(256)
        rc = self.lib.or_ilu_factorize(n, _u32(rp), _u32(ci), _f64(vals64), nblocks, alpha, int(symmetric), prec,
                                       C.byref(h), err, 256)
        if rc:
            raise FactorizationFailed(err.value.decode())
        return OracleIlu(self, h, n)

    def solve(self, a, vals64, spec, b, tol=1e-10, max_outer_restarts=3, max_outer_total=300,
              reset_richardson=False, hist_cap=4096, precond=None) -> Report:
        n, rp, ci = a
        levels, nl = self.parse_spec(spec)
        x = np.zeros(n)
        hist = np.zeros(hist_cap)
        rep = _OrReport()
        rc = self.lib.or_solve_m(n, _u32(rp), _u32(ci), _f64(vals64), levels, nl,
                                 precond.h if precond is not None else None, _f64(b), tol, max_outer_restarts,
                                 max_outer_total, int(reset_richardson), x, hist, hist_cap, C.byref(rep))
        if rc != 0:
            raise RuntimeError(f"oracle solve failed rc={rc}")
        return Report(bool(rep.converged), rep.outer_iterations, rep.precond_invocations, rep.final_true_residual,
                      list(rep.level_iterations[:rep.n_levels]), list(hist[:min(rep.n_history, hist_cap)]),
                      list(rep.omegas[:rep.n_omegas]), rep.flag.decode(), x=x)

    def richardson_apply(self, a, vals_p, p, m, cycle, omegas, counters, v, precond=None):
        n, rp, ci = a
        z = np.zeros(n)
        cnt = (C.c_uint64 * 3)(*counters)
        om = _f64(omegas).copy()
        self.lib.or_richardson_apply_m(n, _u32(rp), _u32(ci), _f64(vals_p), p, m, cycle,
                                       precond.h if precond is not None else None, om, cnt, _f64(v), z)
        return z, om, [cnt[0], cnt[1], cnt[2]]

    def fgmres_cycle(self, a, vals_pa, pa, pw, b, x, m, rel_tol=None, x_is_zero=True):
        n, rp, ci = a
        x = _f64(x).copy()
        it = C.c_int(0)
        est = np.zeros(m + 2)
        flags = (C.c_int * 3)()
        rc = self.lib.or_fgmres_cycle(n, _u32(rp), _u32(ci), _f64(vals_pa), pa, pw, _f64(b), x, m,
                                      0.0 if rel_tol is None else rel_tol, rel_tol is not None, int(x_is_zero),
                                      C.byref(it), est, flags)
        if rc:
            raise RuntimeError("oracle fgmres_cycle failed")
        return x, it.value, est[:it.value + 1], (flags[0], flags[1], flags[2])


class Reference:
    """The unmodified reference library (oracle/_ref/libf3r_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle ref` where /root/reference exists)")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_half_from_double.restype = C.c_uint16
        L.ref_half_from_double.argtypes = [C.c_double]
        L.ref_half_from_float.restype = C.c_uint16
        L.ref_half_from_float.argtypes = [C.c_float]
        L.ref_float_from_half.restype = C.c_float
        L.ref_float_from_half.argtypes = [C.c_uint16]
        L.ref_matrix_create.restype = C.c_void_p
        L.ref_matrix_create.argtypes = [C.c_uint64, _u32p, _u32p, _dp]
        L.ref_matrix_destroy.argtypes = [C.c_void_p]
        L.ref_matrix_values.argtypes = [C.c_void_p, C.c_int, _dp]
        L.ref_generate_stencil.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_diagonal_scale.argtypes = [C.c_uint64, _u32p, _u32p, _dp, C.c_void_p, _dp, C.c_void_p, _dp]
        L.ref_spmv.argtypes = [C.c_void_p, C.c_int, _dp, C.c_int, _dp, C.c_int]
        L.ref_dot.argtypes = [_dp, C.c_int, _dp, C.c_int, C.c_uint64, C.c_int, C.POINTER(C.c_double)]
        L.ref_norm2.argtypes = [_dp, C.c_int, C.c_uint64, C.POINTER(C.c_double)]
        L.ref_axpy.argtypes = [C.c_double, _dp, C.c_int, _dp, C.c_int, C.c_uint64]
        L.ref_add_scaled.argtypes = [_dp, C.c_int, C.c_double, _dp, C.c_int, _dp, C.c_int, C.c_uint64]
        L.ref_copy.argtypes = [_dp, C.c_int, _dp, C.c_int, C.c_uint64]
        L.ref_scale.argtypes = [C.c_double, _dp, C.c_int, C.c_uint64]
        L.ref_richardson_create.restype = C.c_void_p
        L.ref_richardson_create.argtypes = [C.c_int, C.c_uint64]
        L.ref_richardson_destroy.argtypes = [C.c_void_p]
        L.ref_richardson_record.argtypes = [C.c_void_p, C.c_int]
        L.ref_richardson_set_omegas.argtypes = [C.c_void_p, _dp]
        L.ref_richardson_state.argtypes = [C.c_void_p, _dp, C.POINTER(C.c_uint64)]
        L.ref_richardson_log.argtypes = [C.c_void_p, _dp, C.c_uint64, C.POINTER(C.c_uint64)]
        L.ref_richardson_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_int, _dp, _dp]
        L.ref_fgmres_cycle.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _dp, C.c_int, C.c_double, C.c_int,
                                       C.c_int, C.POINTER(C.c_int), _dp, C.POINTER(C.c_int)]
        L.ref_solve.argtypes = [C.c_void_p, C.c_char_p, _dp, C.c_double, C.c_int, C.c_uint64, C.c_int, C.c_void_p,
                                _dp, C.c_uint64, C.POINTER(_RefReport)]
        L.ref_spec_canonical.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64]
        L.ref_krylov_solve.argtypes = [C.c_void_p, C.c_int, _dp, C.c_double, C.c_uint64, C.c_void_p, _dp,
                                       C.c_uint64, C.POINTER(_RefReport)]
        L.ref_solve_m.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, _dp, C.c_double, C.c_int, C.c_uint64,
                                  C.c_int, C.c_void_p, _dp, C.c_uint64, C.POINTER(_RefReport)]
        L.ref_ilu_factorize.argtypes = [C.c_void_p, C.c_uint64, C.c_double, C.c_int, C.c_int,
                                        C.POINTER(C.c_void_p)]
        L.ref_ilu_destroy.argtypes = [C.c_void_p]
        L.ref_ilu_apply.argtypes = [C.c_void_p, _dp, C.c_int, _dp, C.c_int]
        L.ref_richardson_apply_m.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, _dp, _dp]
        L.ref_krylov_solve_m.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, _dp, C.c_double, C.c_uint64,
                                         C.c_void_p, _dp, C.c_uint64, C.POINTER(_RefReport)]
        L.ref_read_matrix_market.argtypes = [C.c_char_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_void_p,
                                             C.c_void_p, C.c_void_p]
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_max_threads.restype = C.c_int

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.lib.ref_last_error().decode()}")

    def set_threads(self, t):
        self.lib.ref_set_threads(int(t))

    def max_threads(self):
        return self.lib.ref_max_threads()

    def generate_stencil(self, lx, ly, lz, beta=0.0):
        n, nnz = C.c_uint64(), C.c_uint64()
        self._check(self.lib.ref_generate_stencil(lx, ly, lz, beta, C.byref(n), C.byref(nnz), None, None, None))
        rp = np.zeros(n.value + 1, np.uint32)
        ci = np.zeros(nnz.value, np.uint32)
        va = np.zeros(nnz.value)
        self._check(self.lib.ref_generate_stencil(lx, ly, lz, beta, C.byref(n), C.byref(nnz),
                                                  rp.ctypes.data, ci.ctypes.data, va.ctypes.data))
        return rp, ci, va

    def diagonal_scale(self, rp, ci, vals, b=None):
        n = len(rp) - 1
        vo = np.zeros(len(ci))
        d = np.zeros(n)
        bo = np.zeros(n) if b is not None else None
        bb = _f64(b) if b is not None else None
        self._check(self.lib.ref_diagonal_scale(n, _u32(rp), _u32(ci), _f64(vals),
                                                bb.ctypes.data if bb is not None else None, vo,
                                                bo.ctypes.data if bo is not None else None, d))
        return vo, bo, d

    class Matrix:
        def __init__(self, ref, rp, ci, vals):
            self.ref = ref
            self.n = len(rp) - 1
            self.h = ref.lib.ref_matrix_create(self.n, _u32(rp), _u32(ci), _f64(vals))
            if not self.h:
                raise RuntimeError(ref.lib.ref_last_error().decode())

        def __del__(self):
            if getattr(self, "h", None):
                self.ref.lib.ref_matrix_destroy(self.h)
                self.h = None

        def values(self, p):
            out = np.zeros(10 ** 0)
            # nnz from a dummy spmv is not exposed; the caller knows nnz
            raise NotImplementedError

    def matrix(self, rp, ci, vals):
        return Reference.Matrix(self, rp, ci, vals)

    def replica_values(self, m, p, nnz):
        out = np.zeros(nnz)
        self._check(self.lib.ref_matrix_values(m.h, p, out))
        return out

    def spmv(self, m, pa, x, px, py):
        y = np.zeros(m.n)
        self._check(self.lib.ref_spmv(m.h, pa, _f64(x), px, y, py))
        return y

    def dot(self, x, px, y, py, floor=P16):
        out = C.c_double()
        self._check(self.lib.ref_dot(_f64(x), px, _f64(y), py, len(x), floor, C.byref(out)))
        return out.value

    def norm2(self, x, px):
        out = C.c_double()
        self._check(self.lib.ref_norm2(_f64(x), px, len(x), C.byref(out)))
        return out.value

    def axpy(self, alpha, x, px, y, py):
        y = _f64(y).copy()
        self._check(self.lib.ref_axpy(alpha, _f64(x), px, y, py, len(y)))
        return y

    def add_scaled(self, x, px, alpha, y, py, po):
        out = np.zeros(len(x))
        self._check(self.lib.ref_add_scaled(_f64(x), px, alpha, _f64(y), py, out, po, len(x)))
        return out

    def copy(self, x, px, py):
        y = np.zeros(len(x))
        self._check(self.lib.ref_copy(_f64(x), px, y, py, len(x)))
        return y

    def scale(self, alpha, x, px):
        x = _f64(x).copy()
        self._check(self.lib.ref_scale(alpha, x, px, len(x)))
        return x

    def richardson(self, m, cycle):
        return _RefRichardson(self, m, cycle)

    def fgmres_cycle(self, mat, pa, pw, b, x, m, rel_tol=None, x_is_zero=True):
        x = _f64(x).copy()
        it = C.c_int(0)
        est = np.zeros(m + 2)
        flags = (C.c_int * 3)()
        self._check(self.lib.ref_fgmres_cycle(mat.h, pa, pw, _f64(b), x, m, 0.0 if rel_tol is None else rel_tol,
                                              rel_tol is not None, int(x_is_zero), C.byref(it), est, flags))
        return x, it.value, est[:it.value + 1], (flags[0], flags[1], flags[2])

    def ilu(self, mat, nblocks, alpha=1.0, symmetric=False, prec=P64):
        """the reference's BlockJacobiIlu0::factorize on mat's fp64 values"""
        h = C.c_void_p()
        rc = self.lib.ref_ilu_factorize(mat.h, nblocks, alpha, int(symmetric), prec, C.byref(h))
        if rc == 5:
            raise FactorizationFailed(self.lib.ref_last_error().decode())
        self._check(rc)
        return _RefIlu(self, h, mat.n)

    def solve(self, mat, spec, b, tol=1e-10, max_outer_restarts=3, max_outer_total=300, reset_richardson=False,
              want_x=True, hist_cap=4096, precond=None) -> Report:
        hist = np.zeros(hist_cap)
        rep = _RefReport()
        x = np.zeros(mat.n) if want_x else None
        self._check(self.lib.ref_solve_m(mat.h, spec.encode(), precond.h if precond is not None else None, _f64(b),
                                         tol, max_outer_restarts, max_outer_total, int(reset_richardson),
                                         x.ctypes.data if x is not None else None, hist, hist_cap, C.byref(rep)))
        return Report(bool(rep.converged), rep.outer_iterations, rep.precond_invocations, rep.final_true_residual,
                      list(rep.level_iterations[:rep.n_levels]), list(hist[:min(rep.n_history, hist_cap)]),
                      list(rep.omegas[:rep.n_omegas]), rep.flag.decode(), rep.wall_seconds, rep.id.decode(), x=x)

    def krylov_solve(self, mat, which, b, tol=1e-10, max_precond=19200, hist_cap=1 << 16, precond=None,
                     restart=64) -> Report:
        """reference cg_solve (which="cg") / bicgstab_solve ("bicgstab"), src/cg.cpp:22-171, or
        fgmres_restarted ("fgmres", src/fgmres.cpp:163-222); M = identity or `precond`"""
        hist = np.zeros(hist_cap)
        rep = _RefReport()
        w = {"cg": 0, "bicgstab": 1, "fgmres": 2}[which]
        self._check(self.lib.ref_krylov_solve_m(mat.h, w, precond.h if precond is not None else None, int(restart),
                                                _f64(b), tol, max_precond, None, hist, hist_cap, C.byref(rep)))
        return Report(bool(rep.converged), rep.outer_iterations, rep.precond_invocations, rep.final_true_residual,
                      [], list(hist[:min(rep.n_history, hist_cap)]), [], rep.flag.decode(), rep.wall_seconds,
                      rep.id.decode())

    def read_matrix_market(self, path):
        """(row_ptr, col_idx, values) of the reference reader; RuntimeError on ParseError"""
        n, nnz = C.c_uint64(), C.c_uint64()
        self._check(self.lib.ref_read_matrix_market(str(path).encode(), C.byref(n), C.byref(nnz), None, None, None))
        rp = np.zeros(n.value + 1, np.uint32)
        ci = np.zeros(max(1, nnz.value), np.uint32)
        va = np.zeros(max(1, nnz.value))
        self._check(self.lib.ref_read_matrix_market(str(path).encode(), C.byref(n), C.byref(nnz), rp.ctypes.data,
                                                    ci.ctypes.data, va.ctypes.data))
        return rp, ci[:nnz.value], va[:nnz.value]

    def spec_canonical(self, spec):
        buf = C.create_string_buffer(512)
        self._check(self.lib.ref_spec_canonical(spec.encode(), buf, 512))
        return buf.value.decode()


class _RefRichardson:
    def __init__(self, ref, m, cycle):
        self.ref, self.m = ref, m
        self.h = ref.lib.ref_richardson_create(m, cycle)
        ref.lib.ref_richardson_record(self.h, 1)

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_richardson_destroy(self.h)

    def apply(self, mat, p, v, precond=None):
        z = np.zeros(mat.n)
        if precond is None:
            self.ref._check(self.ref.lib.ref_richardson_apply(mat.h, self.h, p, _f64(v), z))
        else:
            self.ref._check(self.ref.lib.ref_richardson_apply_m(mat.h, self.h, p, precond.h, _f64(v), z))
        return z

    def state(self):
        om = np.zeros(self.m)
        cnt = (C.c_uint64 * 3)()
        self.ref.lib.ref_richardson_state(self.h, om, cnt)
        return om, [cnt[0], cnt[1], cnt[2]]

    def log(self):
        out = np.zeros(4096)
        ln = C.c_uint64()
        self.ref.lib.ref_richardson_log(self.h, out, 4096, C.byref(ln))
        return out[:ln.value]


class FactorizationFailed(RuntimeError):
    """f3r::FactorizationError raised by a checker's factorize"""


class OracleIlu:
    """A block-Jacobi ILU(0)/IC(0) factorised by the C oracle."""

    def __init__(self, oracle, h, n):
        self.o, self.h, self.n = oracle, h, n

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.or_ilu_free(self.h)
            self.h = None

    def apply(self, r, pr, pz):
        z = np.zeros(self.n)
        self.o.lib.or_ilu_apply(self.h, _f64(r), pr, z, pz)
        return z

    def factors(self, upper):
        """(ptr, idx, vals) of the stored lower (upper=0) or upper (1) factor"""
        nz = self.o.lib.or_ilu_count(self.h, int(upper))
        ptr = np.zeros(self.n + 1, np.uint32)
        idx = np.zeros(max(nz, 1), np.uint32)
        vals = np.zeros(max(nz, 1))
        self.o.lib.or_ilu_export(self.h, int(upper), ptr, idx, vals)
        return ptr, idx[:nz], vals[:nz]


class _RefIlu:
    def __init__(self, ref, h, n):
        self.ref, self.h, self.n = ref, h, n

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_ilu_destroy(self.h)
            self.h = None

    def apply(self, r, pr, pz):
        z = np.zeros(self.n)
        self.ref._check(self.ref.lib.ref_ilu_apply(self.h, _f64(r), pr, z, pz))
        return z


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def oracle_available() -> bool:
    return os.path.exists(ORACLE_SO)
