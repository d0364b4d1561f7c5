// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI veneer over the UNMODIFIED reference library (/root/reference/proj,
// compiled in place by oracle/Makefile into oracle/_ref/libf3r_ref.so). It lets
// the Python test-suite, the golden-vector generator and bench.py's CPU arm
// drive the reference through its own public C++ API (include/f3r/*.hpp):
//   - spmv / dot / dot_at_least / axpy / add_scaled / copy_into / scale_in_place
//     / norm2 / fill            (include/f3r/csr.hpp:83-85, include/f3r/dense_vector.hpp:62-97)
//   - generate_stencil, diagonal_scale, make_replicas
//                                (include/f3r/stencil.hpp:32, scaling.hpp:33-41, csr.hpp:80)
//   - richardson_apply + RichardsonState (include/f3r/richardson.hpp:26-53)
//   - fgmres_cycle               (include/f3r/fgmres.hpp:37-38)
//   - build / parse_solver_spec / ComposedSolver::run (include/f3r/nesting.hpp:55-77)
// Nothing here is product code; the product path never links this library.
// Vectors cross this boundary as double arrays holding values already
// representable at the stated precision (0 = f16, 1 = f32, 2 = f64).

#include <chrono>
#include <fstream>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "f3r/cg.hpp"
#include "f3r/csr.hpp"
#include "f3r/dense_vector.hpp"
#include "f3r/fgmres.hpp"
#include "f3r/ilu.hpp"
#include "f3r/matrix_market.hpp"
#include "f3r/nesting.hpp"
#include "f3r/operator.hpp"
#include "f3r/richardson.hpp"
#include "f3r/scaling.hpp"
#include "f3r/solver_spec.hpp"
#include "f3r/stencil.hpp"

using f3r::DenseVector;
using f3r::Precision;

namespace {

thread_local std::string g_err;

Precision prec(int p) { return p == 0 ? Precision::P16 : p == 1 ? Precision::P32 : Precision::P64; }

DenseVector make_vec(const double* v, std::size_t n, int p) {
  DenseVector out(n, prec(p));
  for (std::size_t i = 0; i < n; ++i) out.set(i, v[i]);
  return out;
}

void read_vec(const DenseVector& v, double* out) {
  for (std::size_t i = 0; i < v.size(); ++i) out[i] = v.at(i);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const f3r::DimensionError& e) {
    g_err = e.what();
    return 2;
  } catch (const f3r::SolverError& e) {
    g_err = e.what();
    return 3;
  } catch (const f3r::ParseError& e) {
    g_err = e.what();
    return 4;
  } catch (const f3r::FactorizationError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

// Test double mirroring tests/test_richardson.cpp:19-28: multiply = spmv,
// precondition = identity copy.
class MatrixIdentityOp final : public f3r::LinearOperator {
 public:
  explicit MatrixIdentityOp(const f3r::SparseCsr& a) : a_(&a) {}
  std::size_t size() const override { return a_->rows(); }
  void multiply(const DenseVector& x, DenseVector& y) const override { f3r::spmv(*a_, x, y); }
  void precondition(const DenseVector& v, DenseVector& z) override { f3r::copy_into(v, z); }

 private:
  const f3r::SparseCsr* a_;
};

struct RefMatrix {
  f3r::PrecisionReplicas reps;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

int ref_max_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

// ---- half -----------------------------------------------------------------
uint16_t ref_half_from_double(double x) { return f3r::Half(x).bits(); }
uint16_t ref_half_from_float(float x) { return f3r::Half(x).bits(); }
float ref_float_from_half(uint16_t h) { return static_cast<float>(f3r::Half::from_bits(h)); }

// ---- matrices -------------------------------------------------------------
// Builds the replicas (make_replicas) of a validated fp64 CSR; NULL on error.
void* ref_matrix_create(uint64_t n, const uint32_t* row_ptr, const uint32_t* col_idx, const double* vals) {
  RefMatrix* m = nullptr;
  const int rc = guarded([&] {
    const uint64_t nnz = row_ptr[n];
    f3r::SparseCsr a(n, std::vector<uint32_t>(row_ptr, row_ptr + n + 1),
                     std::vector<uint32_t>(col_idx, col_idx + nnz), std::vector<double>(vals, vals + nnz));
    m = new RefMatrix{f3r::make_replicas(std::move(a))};
  });
  return rc == 0 ? m : nullptr;
}

void ref_matrix_destroy(void* h) { delete static_cast<RefMatrix*>(h); }

// Replica values widened to double (exact), for replica parity checks.
int ref_matrix_values(void* h, int p, double* out) {
  return guarded([&] {
    const auto& a = static_cast<RefMatrix*>(h)->reps.at(prec(p));
    for (std::size_t k = 0; k < a.nnz(); ++k) out[k] = a.value_at(k);
  });
}

// generate_stencil: first call with row_ptr == NULL returns n, nnz.
int ref_generate_stencil(int lx, int ly, int lz, double beta, uint64_t* n_out, uint64_t* nnz_out,
                         uint32_t* row_ptr, uint32_t* col_idx, double* vals) {
  return guarded([&] {
    const f3r::SparseCsr a = f3r::generate_stencil({lx, ly, lz, beta});
    *n_out = a.rows();
    *nnz_out = a.nnz();
    if (row_ptr) {
      std::memcpy(row_ptr, a.row_ptr().data(), (a.rows() + 1) * sizeof(uint32_t));
      std::memcpy(col_idx, a.col_idx().data(), a.nnz() * sizeof(uint32_t));
      for (std::size_t k = 0; k < a.nnz(); ++k) vals[k] = a.value_at(k);
    }
  });
}

int ref_parse_stencil_name(const char* name, int* lx, int* ly, int* lz, double* beta) {
  return guarded([&] {
    const auto s = f3r::parse_stencil_name(name);
    *lx = s.log2_nx;
    *ly = s.log2_ny;
    *lz = s.log2_nz;
    *beta = s.beta;
  });
}

// diagonal_scale(A, b): scaled values, scaled rhs (b may be NULL) and d.
int ref_diagonal_scale(uint64_t n, const uint32_t* row_ptr, const uint32_t* col_idx, const double* vals,
                       const double* b, double* vals_out, double* b_out, double* d_out) {
  return guarded([&] {
    const uint64_t nnz = row_ptr[n];
    f3r::SparseCsr a(n, std::vector<uint32_t>(row_ptr, row_ptr + n + 1),
                     std::vector<uint32_t>(col_idx, col_idx + nnz), std::vector<double>(vals, vals + nnz));
    if (b) {
      const auto s = f3r::diagonal_scale(a, make_vec(b, n, 2));
      for (std::size_t k = 0; k < nnz; ++k) vals_out[k] = s.matrix.value_at(k);
      read_vec(s.rhs, b_out);
      std::memcpy(d_out, s.d.data(), n * sizeof(double));
    } else {
      const auto s = f3r::diagonal_scale(a);
      for (std::size_t k = 0; k < nnz; ++k) vals_out[k] = s.matrix.value_at(k);
      std::memcpy(d_out, s.d.data(), n * sizeof(double));
    }
  });
}

// ---- kernels ----------------------------------------------------------------
int ref_spmv(void* h, int pa, const double* x, int px, double* y, int py) {
  return guarded([&] {
    const auto& a = static_cast<RefMatrix*>(h)->reps.at(prec(pa));
    const std::size_t n = a.rows();
    DenseVector xv = make_vec(x, n, px);
    DenseVector yv(n, prec(py));
    f3r::spmv(a, xv, yv);
    read_vec(yv, y);
  });
}

int ref_dot(const double* x, int px, const double* y, int py, uint64_t n, int floor_p, double* out) {
  return guarded([&] {
    *out = f3r::dot_at_least(make_vec(x, n, px), make_vec(y, n, py), prec(floor_p));
  });
}

int ref_norm2(const double* x, int px, uint64_t n, double* out) {
  return guarded([&] { *out = f3r::norm2(make_vec(x, n, px)); });
}

int ref_axpy(double alpha, const double* x, int px, double* y, int py, uint64_t n) {
  return guarded([&] {
    DenseVector yv = make_vec(y, n, py);
    f3r::axpy(alpha, make_vec(x, n, px), yv);
    read_vec(yv, y);
  });
}

int ref_add_scaled(const double* x, int px, double alpha, const double* y, int py, double* out, int po,
                   uint64_t n) {
  return guarded([&] {
    DenseVector ov(n, prec(po));
    f3r::add_scaled(make_vec(x, n, px), alpha, make_vec(y, n, py), ov);
    read_vec(ov, out);
  });
}

int ref_copy(const double* x, int px, double* y, int py, uint64_t n) {
  return guarded([&] {
    DenseVector yv(n, prec(py));
    f3r::copy_into(make_vec(x, n, px), yv);
    read_vec(yv, y);
  });
}

int ref_scale(double alpha, double* x, int px, uint64_t n) {
  return guarded([&] {
    DenseVector xv = make_vec(x, n, px);
    f3r::scale_in_place(alpha, xv);
    read_vec(xv, x);
  });
}

// ---- Richardson (state persists across calls) ------------------------------
void* ref_richardson_create(int m, uint64_t cycle) { return new f3r::RichardsonState(m, cycle); }
void ref_richardson_destroy(void* s) { delete static_cast<f3r::RichardsonState*>(s); }
void ref_richardson_record(void* s, int on) { static_cast<f3r::RichardsonState*>(s)->record_updates = on != 0; }
int ref_richardson_set_omegas(void* s, const double* w) {
  auto* st = static_cast<f3r::RichardsonState*>(s);
  for (std::size_t k = 0; k < st->omegas.size(); ++k) st->omegas[k] = w[k];
  return 0;
}
// out: omegas[m]; counters[0..2] = call_count, update_count, degenerate_events
int ref_richardson_state(void* s, double* omegas, uint64_t* counters) {
  auto* st = static_cast<f3r::RichardsonState*>(s);
  for (std::size_t k = 0; k < st->omegas.size(); ++k) omegas[k] = st->omegas[k];
  counters[0] = st->call_count;
  counters[1] = st->update_count;
  counters[2] = st->degenerate_events;
  return 0;
}
int ref_richardson_log(void* s, double* out, uint64_t cap, uint64_t* len) {
  auto* st = static_cast<f3r::RichardsonState*>(s);
  *len = st->update_log.size();
  for (std::size_t i = 0; i < st->update_log.size() && i < cap; ++i) out[i] = st->update_log[i];
  return 0;
}
// One richardson_apply with A = replica at precision p (vectors at p), M = I.
int ref_richardson_apply(void* h, void* s, int p, const double* v, double* z) {
  return guarded([&] {
    const auto& a = static_cast<RefMatrix*>(h)->reps.at(prec(p));
    MatrixIdentityOp op(a);
    const std::size_t n = a.rows();
    DenseVector zv(n, prec(p));
    f3r::richardson_apply(op, make_vec(v, n, p), *static_cast<f3r::RichardsonState*>(s), zv);
    read_vec(zv, z);
  });
}

// ---- block-Jacobi ILU(0)/IC(0) (include/f3r/ilu.hpp:44-84) ------------------
// Factorises the fp64 replica of h. On success *out is a BlockJacobiIlu0*.
int ref_ilu_factorize(void* h, uint64_t nblocks, double alpha, int symmetric, int p, void** out) {
  *out = nullptr;
  return guarded([&] {
    f3r::IluConfig cfg;
    cfg.nblocks = nblocks;
    cfg.alpha = alpha;
    cfg.symmetric = symmetric != 0;
    cfg.apply_precision = prec(p);
    *out = new f3r::BlockJacobiIlu0(f3r::BlockJacobiIlu0::factorize(static_cast<RefMatrix*>(h)->reps.a64, cfg));
  });
}
void ref_ilu_destroy(void* m) { delete static_cast<f3r::BlockJacobiIlu0*>(m); }
// z = M r (Preconditioner::apply), r at pr, z at pz
int ref_ilu_apply(void* m, const double* r, int pr, double* z, int pz) {
  return guarded([&] {
    const auto* M = static_cast<f3r::BlockJacobiIlu0*>(m);
    const std::size_t n = M->rows();
    DenseVector zv(n, prec(pz));
    M->apply(make_vec(r, n, pr), zv);
    read_vec(zv, z);
  });
}

// richardson_apply on (A_p, M) -- the operator a RichardsonInner sees when its child
// is the PrimarySolver (src/nesting.cpp:46-83: multiply = spmv, precondition = M)
class MatrixPrecondOp final : public f3r::LinearOperator {
 public:
  MatrixPrecondOp(const f3r::SparseCsr& a, const f3r::Preconditioner& m) : a_(&a), m_(&m) {}
  std::size_t size() const override { return a_->rows(); }
  void multiply(const DenseVector& x, DenseVector& y) const override { f3r::spmv(*a_, x, y); }
  void precondition(const DenseVector& v, DenseVector& z) override { m_->apply(v, z); }

 private:
  const f3r::SparseCsr* a_;
  const f3r::Preconditioner* m_;
};
int ref_richardson_apply_m(void* h, void* s, int p, void* precond, const double* v, double* z) {
  return guarded([&] {
    const auto& a = static_cast<RefMatrix*>(h)->reps.at(prec(p));
    MatrixPrecondOp op(a, *static_cast<f3r::BlockJacobiIlu0*>(precond));
    const std::size_t n = a.rows();
    DenseVector zv(n, prec(p));
    f3r::richardson_apply(op, make_vec(v, n, p), *static_cast<f3r::RichardsonState*>(s), zv);
    read_vec(zv, z);
  });
}

// ---- one FGMRES cycle against (A_pa, M = identity), vectors at pw ------------
int ref_fgmres_cycle(void* h, int pa, int pw, const double* b, double* x, int m, double rel_tol, int use_tol,
                     int x_is_zero, int* iterations, double* estimates /* m+1 */, int* flags /* happy, diverged, step */) {
  return guarded([&] {
    const auto& a = static_cast<RefMatrix*>(h)->reps.at(prec(pa));
    f3r::IdentityPrecond ident(a.rows());
    f3r::PreconditionedMatrix op(a, ident);
    const std::size_t n = a.rows();
    DenseVector xv = make_vec(x, n, pw);
    const auto res = f3r::fgmres_cycle(op, make_vec(b, n, pw), xv, m,
                                       use_tol ? std::optional<double>(rel_tol) : std::nullopt, x_is_zero != 0);
    read_vec(xv, x);
    *iterations = res.iterations;
    for (std::size_t i = 0; i < res.estimates.size(); ++i) estimates[i] = res.estimates[i];
    flags[0] = res.happy_breakdown;
    flags[1] = res.diverged;
    flags[2] = res.divergence_step;
  });
}

// ---- composed solve ---------------------------------------------------------
struct RefReport {
  int converged;
  uint64_t outer_iterations;
  uint64_t precond_invocations;
  double final_true_residual;
  double wall_seconds;
  uint64_t n_levels;
  uint64_t level_iterations[16];
  uint64_t n_history;
  uint64_t n_omegas;
  double omegas[64];
  char flag[128];
  char id[256];
};

// Solves with `spec` (the reference grammar) and M = IdentityPrecond.
// history: capacity hist_cap; x_out may be NULL.
int ref_solve_m(void* h, const char* spec, void* precond, const double* b, double tol, int max_outer_restarts,
                uint64_t max_outer_total, int reset_richardson, double* x_out, double* history, uint64_t hist_cap,
                RefReport* rep);
int ref_solve(void* h, const char* spec, const double* b, double tol, int max_outer_restarts,
              uint64_t max_outer_total, int reset_richardson, double* x_out, double* history, uint64_t hist_cap,
              RefReport* rep) {
  return ref_solve_m(h, spec, nullptr, b, tol, max_outer_restarts, max_outer_total, reset_richardson, x_out, history,
                     hist_cap, rep);
}

// Same with M = a BlockJacobiIlu0 from ref_ilu_factorize (nullptr: IdentityPrecond).
int ref_solve_m(void* h, const char* spec, void* precond, const double* b, double tol, int max_outer_restarts,
                uint64_t max_outer_total, int reset_richardson, double* x_out, double* history, uint64_t hist_cap,
                RefReport* rep) {
  return guarded([&] {
    auto* m = static_cast<RefMatrix*>(h);
    const std::size_t n = m->reps.a64.rows();
    f3r::IdentityPrecond ident(n);
    const f3r::Preconditioner& M =
        precond ? static_cast<const f3r::Preconditioner&>(*static_cast<f3r::BlockJacobiIlu0*>(precond)) : ident;
    auto solver = f3r::build(f3r::parse_solver_spec(spec), m->reps, M);
    f3r::RunOptions opts;
    opts.tol = tol;
    opts.max_outer_restarts = max_outer_restarts;
    opts.max_outer_total = max_outer_total;
    opts.reset_richardson_on_restart = reset_richardson != 0;
    const DenseVector bv = make_vec(b, n, 2);
    const auto t0 = std::chrono::steady_clock::now();
    auto run = solver.run(bv, opts);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const auto& r = run.report;
    std::memset(rep, 0, sizeof(*rep));
    rep->converged = r.converged;
    rep->outer_iterations = r.outer_iterations;
    rep->precond_invocations = r.precond_invocations;
    rep->final_true_residual = r.final_true_residual;
    rep->wall_seconds = secs;
    rep->n_levels = r.level_iterations.size();
    for (std::size_t i = 0; i < r.level_iterations.size() && i < 16; ++i) rep->level_iterations[i] = r.level_iterations[i];
    rep->n_history = r.residual_history.size();
    for (std::size_t i = 0; i < r.residual_history.size() && i < hist_cap; ++i) history[i] = r.residual_history[i];
    rep->n_omegas = r.omegas_final.size();
    for (std::size_t i = 0; i < r.omegas_final.size() && i < 64; ++i) rep->omegas[i] = r.omegas_final[i];
    std::strncpy(rep->flag, r.flag.c_str(), sizeof(rep->flag) - 1);
    std::strncpy(rep->id, solver.id().c_str(), sizeof(rep->id) - 1);
    if (x_out) read_vec(run.x, x_out);
  });
}

// The reference's competitor solvers (src/cg.cpp:22-171) with M = IdentityPrecond:
// which = 0 cg_solve, 1 bicgstab_solve. Same report layout as ref_solve.
int ref_krylov_solve_m(void* h, int which, void* precond, int restart, const double* b, double tol,
                       uint64_t max_precond, double* x_out, double* history, uint64_t hist_cap, RefReport* rep);
int ref_krylov_solve(void* h, int which, const double* b, double tol, uint64_t max_precond, double* x_out,
                     double* history, uint64_t hist_cap, RefReport* rep) {
  return ref_krylov_solve_m(h, which, nullptr, 64, b, tol, max_precond, x_out, history, hist_cap, rep);
}

// which = 2: fgmres_restarted(a, M, b, restart, FgmresOptions) (src/fgmres.cpp:163-222);
// precond: a BlockJacobiIlu0 from ref_ilu_factorize, nullptr = IdentityPrecond
int ref_krylov_solve_m(void* h, int which, void* precond, int restart, const double* b, double tol,
                       uint64_t max_precond, double* x_out, double* history, uint64_t hist_cap, RefReport* rep) {
  return guarded([&] {
    auto* m = static_cast<RefMatrix*>(h);
    const std::size_t n = m->reps.a64.rows();
    f3r::IdentityPrecond ident(n);
    const f3r::Preconditioner& M =
        precond ? static_cast<const f3r::Preconditioner&>(*static_cast<f3r::BlockJacobiIlu0*>(precond)) : ident;
    f3r::ReferenceSolveOptions opts;
    opts.tol = tol;
    opts.max_precond_invocations = max_precond;
    f3r::FgmresOptions fo;
    fo.tol = tol;
    fo.max_precond_invocations = max_precond;
    const DenseVector bv = make_vec(b, n, 2);
    const auto t0 = std::chrono::steady_clock::now();
    const f3r::ConvergenceReport r = which == 0   ? f3r::cg_solve(m->reps.a64, M, bv, opts)
                                     : which == 1 ? f3r::bicgstab_solve(m->reps.a64, M, bv, opts)
                                                  : f3r::fgmres_restarted(m->reps.a64, M, bv, restart, fo);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::memset(rep, 0, sizeof(*rep));
    rep->converged = r.converged;
    rep->outer_iterations = r.outer_iterations;
    rep->precond_invocations = r.precond_invocations;
    rep->final_true_residual = r.final_true_residual;
    rep->wall_seconds = secs;
    rep->n_history = r.residual_history.size();
    for (std::size_t i = 0; i < r.residual_history.size() && i < hist_cap; ++i) history[i] = r.residual_history[i];
    std::strncpy(rep->flag, r.flag.c_str(), sizeof(rep->flag) - 1);
    std::strncpy(rep->id, r.solver_id.c_str(), sizeof(rep->id) - 1);
    (void)x_out;
  });
}

// read_matrix_market(std::ifstream(path)) (src/matrix_market.cpp:33-113); call with
// null arrays for n / nnz, then again with arrays
int ref_read_matrix_market(const char* path, uint64_t* n, uint64_t* nnz, uint32_t* rp, uint32_t* ci, double* v) {
  return guarded([&] {
    std::ifstream in(path);
    const f3r::SparseCsr a = f3r::read_matrix_market(in);
    *n = a.rows();
    *nnz = a.nnz();
    if (rp) std::memcpy(rp, a.row_ptr().data(), (a.rows() + 1) * 4);
    if (ci) std::memcpy(ci, a.col_idx().data(), a.nnz() * 4);
    if (v) std::memcpy(v, a.values_as<double>().data(), a.nnz() * 8);
  });
}

// Canonical to_string() of a parsed spec (grammar round-trip).
int ref_spec_canonical(const char* spec, char* out, uint64_t cap) {
  return guarded([&] {
    const std::string s = f3r::parse_solver_spec(spec).to_string();
    std::strncpy(out, s.c_str(), cap - 1);
    out[cap - 1] = 0;
  });
}

}  // extern "C"
