// f3r_gpu.hpp -- header-only C++ face of the C ABI in f3rg.h, shaped like the
// reference's solve API so a reference maintainer can swap the CPU ComposedSolver
// for the device one with a handful of lines (INTEGRATION.md shows the adapter).
//
//   reference (include/f3r/...)                   this header
//   SparseCsr + make_replicas  csr.hpp:23-81       f3r_gpu::DeviceReplicas
//   ComposedSolver(spec, replicas, M)              f3r_gpu::ComposedSolver(spec, replicas[, M])
//     nesting.hpp:55-77
//   IdentityPrecond / BlockJacobiIlu0::factorize   f3r_gpu::DevicePreconditioner::identity /
//     ilu.hpp:34-84                                ::factorize (config fields as IluConfig)
//   RunOptions  nesting.hpp:29-38                  f3r_gpu::RunOptions (same fields)
//   ConvergenceReport  report.hpp:18-30            f3r_gpu::ConvergenceReport (same fields)
//   RunResult{x, report}  nesting.hpp:46-49        f3r_gpu::RunResult{x (fp64), report}
//   counters(), innermost_omegas(), id()           same names
//   ParseError / DimensionError / SolverError /    rethrown as f3r:: classes when the
//   FactorizationError  errors.hpp:12-38           reference's errors.hpp is included
//                                                  first, else as f3r_gpu:: mirrors
//
// Depends on f3rg.h only; link with -lf3rg (paper_2505_20719_b200/lib/libf3rg.so).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "f3rg.h"

namespace f3r_gpu {

#ifdef F3R_ERRORS_HPP
using Error = ::f3r::Error;
using ParseError = ::f3r::ParseError;
using DimensionError = ::f3r::DimensionError;
using FactorizationError = ::f3r::FactorizationError;
using SolverError = ::f3r::SolverError;
#else
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ParseError : Error {
  using Error::Error;
};
struct DimensionError : Error {
  using Error::Error;
};
struct FactorizationError : Error {
  using Error::Error;
};
struct SolverError : Error {
  using Error::Error;
};
#endif
// failures with no reference counterpart (CUDA runtime, unsupported on the device)
struct DeviceError : std::runtime_error {
  int code;
  DeviceError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void check(int rc) {
  if (rc == F3RG_OK) return;
  const std::string msg = f3rg_last_error();
  switch (rc) {
    case F3RG_EPARSE: throw ParseError(msg);
    case F3RG_EDIMENSION: throw DimensionError(msg);
    case F3RG_EFACTORIZATION: throw FactorizationError(msg);
    case F3RG_ESOLVER: throw SolverError(msg);
    default: throw DeviceError(rc, msg);
  }
}

struct RunOptions {
  double tol = 1e-8;
  int max_outer_restarts = 3;
  std::uint64_t max_outer_total = 300;
  bool reset_richardson_on_restart = false;
};

struct ConvergenceReport {
  bool converged = false;
  std::uint64_t outer_iterations = 0;
  std::uint64_t precond_invocations = 0;
  std::vector<std::uint64_t> level_iterations;
  std::vector<double> residual_history;
  double final_true_residual = 0.0;
  double wall_seconds = 0.0;
  std::vector<double> omegas_final;
  std::string flag;
  std::string solver_id;
  std::string problem_id;
};

struct NestingCounters {
  std::vector<std::uint64_t> level_invocations;  // not tracked per level on the device: empty
  std::vector<std::uint64_t> level_iterations;
  std::uint64_t precond_invocations = 0;
};

struct RunResult {
  std::vector<double> x;  // fp64, like the reference's RunResult::x
  ConvergenceReport report;
};

// The fp64 CSR uploaded once with its fp32 / fp16 replicas (RNE demotions, as
// make_replicas, src/csr.cpp:130-136) and one shared index copy.
class DeviceReplicas {
 public:
  DeviceReplicas(std::uint64_t n, const std::uint32_t* row_ptr, const std::uint32_t* col_idx,
                 const double* values) {
    f3rg_csr c{n, row_ptr, col_idx, values};
    f3rg_matrix* m = nullptr;
    check(f3rg_matrix_create(&m, &c));
    m_.reset(m);
  }
  // any CSR with rows(), row_ptr(), col_idx() and fp64 values_as<double>() -- i.e. the
  // reference's f3r::SparseCsr (its a64 replica) -- without including its headers
  template <class Csr>
  static DeviceReplicas from(const Csr& a64) {
    return DeviceReplicas(a64.rows(), a64.row_ptr().data(), a64.col_idx().data(),
                          a64.template values_as<double>().data());
  }
  std::uint64_t rows() const { return f3rg_matrix_rows(m_.get()); }
  std::uint64_t nnz() const { return f3rg_matrix_nnz(m_.get()); }
  const f3rg_matrix* handle() const { return m_.get(); }

 private:
  struct Del {
    void operator()(f3rg_matrix* m) const { f3rg_matrix_destroy(m); }
  };
  std::unique_ptr<f3rg_matrix, Del> m_;
};

// The primary preconditioner M on the device: IdentityPrecond, or block-Jacobi
// ILU(0)/IC(0) factorised on the host at fp64 exactly as BlockJacobiIlu0::factorize
// (src/ilu.cpp:38-185) and applied by bit-exact device sweeps. Throws
// FactorizationError with the reference's message.
class DevicePreconditioner {
 public:
  static DevicePreconditioner identity(std::uint64_t n) {
    f3rg_precond* m = nullptr;
    check(f3rg_precond_identity(&m, n));
    return DevicePreconditioner(m);
  }
  static DevicePreconditioner factorize(std::uint64_t n, const std::uint32_t* row_ptr, const std::uint32_t* col_idx,
                                        const double* values, std::uint64_t nblocks, double alpha, bool symmetric,
                                        int apply_precision) {
    f3rg_csr c{n, row_ptr, col_idx, values};
    f3rg_ilu_config cfg{nblocks, alpha, symmetric ? 1 : 0, apply_precision};
    f3rg_precond* m = nullptr;
    check(f3rg_ilu_factorize(&m, &c, &cfg));
    return DevicePreconditioner(m);
  }
  // the reference's SparseCsr (a64) and IluConfig, without including their headers
  template <class Csr, class Cfg>
  static DevicePreconditioner factorize(const Csr& a64, const Cfg& cfg) {
    return factorize(a64.rows(), a64.row_ptr().data(), a64.col_idx().data(), a64.template values_as<double>().data(),
                     cfg.nblocks, cfg.alpha, cfg.symmetric, static_cast<int>(cfg.apply_precision));
  }
  std::uint64_t rows() const { return f3rg_precond_rows(m_.get()); }
  const f3rg_precond* handle() const { return m_.get(); }

 private:
  explicit DevicePreconditioner(f3rg_precond* m) : m_(m, f3rg_precond_destroy) {}
  std::shared_ptr<f3rg_precond> m_;
};

// ComposedSolver over device replicas. `spec` is the reference grammar
// (src/solver_spec.cpp), e.g. "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 >
// identity". The replicas must outlive the solver (nesting.hpp:51-54). Like the
// reference, Richardson weights persist across run() calls; reset() restores the
// state of a freshly built solver.
class ComposedSolver {
 public:
  ComposedSolver(const std::string& spec, const DeviceReplicas& a) : n_(a.rows()) {
    f3rg_solver* s = nullptr;
    check(f3rg_solver_create(&s, a.handle(), spec.c_str(), F3RG_PRECOND_IDENTITY));
    s_.reset(s);
    id_ = f3rg_solver_id(s);
  }
  // with a primary preconditioner (the device keeps its own reference to it)
  ComposedSolver(const std::string& spec, const DeviceReplicas& a, const DevicePreconditioner& m) : n_(a.rows()) {
    f3rg_solver* s = nullptr;
    check(f3rg_solver_create_m(&s, a.handle(), spec.c_str(), m.handle()));
    s_.reset(s);
    id_ = f3rg_solver_id(s);
  }

  // b, x: host fp64 arrays of length rows() (x may be null); copies happen inside
  ConvergenceReport run(const double* b, double* x, const RunOptions& o = {}) {
    f3rg_run_options ro{o.tol, o.max_outer_restarts, o.max_outer_total, o.reset_richardson_on_restart ? 1 : 0};
    f3rg_report r{};
    check(f3rg_solve(s_.get(), b, x, &ro, &r));
    return report(r);
  }
  RunResult run(const std::vector<double>& b, const RunOptions& o = {}) {
    if (b.size() != n_) throw DimensionError("ComposedSolver::run: rhs size mismatch");
    RunResult out;
    out.x.assign(n_, 0.0);
    out.report = run(b.data(), out.x.data(), o);
    return out;
  }
  // b, x: DEVICE fp64 arrays; stream: a cudaStream_t cast to uintptr_t (0 = own stream)
  ConvergenceReport run_device(const double* b, double* x, const RunOptions& o = {}, std::uintptr_t stream = 0) {
    f3rg_run_options ro{o.tol, o.max_outer_restarts, o.max_outer_total, o.reset_richardson_on_restart ? 1 : 0};
    f3rg_report r{};
    check(f3rg_solve_device(s_.get(), b, x, &ro, &r, stream));
    return report(r);
  }

  void reset(std::uintptr_t stream = 0) { check(f3rg_solver_reset_state(s_.get(), stream)); }
  const NestingCounters& counters() const { return counters_; }
  std::vector<double> innermost_omegas() {
    std::vector<double> w(f3rg_solver_omega_count(s_.get()));
    if (!w.empty()) check(f3rg_solver_omegas(s_.get(), w.data(), w.size()));
    return w;
  }
  const std::string& id() const { return id_; }

 private:
  ConvergenceReport report(const f3rg_report& r) {
    ConvergenceReport c;
    c.converged = r.converged != 0;
    c.outer_iterations = r.outer_iterations;
    c.precond_invocations = r.precond_invocations;
    c.final_true_residual = r.final_true_residual;
    c.wall_seconds = r.wall_seconds;
    c.flag = r.flag;
    c.solver_id = id_;
    c.residual_history.resize(r.n_history);
    check(f3rg_solver_history(s_.get(), c.residual_history.data(), r.n_history));
    c.level_iterations.resize(r.n_levels);
    check(f3rg_solver_level_iterations(s_.get(), reinterpret_cast<std::uint64_t*>(c.level_iterations.data()),
                                       r.n_levels));
    c.omegas_final.resize(r.n_omegas);
    if (r.n_omegas) check(f3rg_solver_omegas(s_.get(), c.omegas_final.data(), r.n_omegas));
    counters_.level_iterations = c.level_iterations;
    counters_.precond_invocations += r.precond_invocations;
    return c;
  }
  struct Del {
    void operator()(f3rg_solver* s) const { f3rg_solver_destroy(s); }
  };
  std::unique_ptr<f3rg_solver, Del> s_;
  std::uint64_t n_;
  std::string id_;
  NestingCounters counters_;
};

}  // namespace f3r_gpu
