/* f3r_gpu_adapter.hpp -- the drop-in a reference maintainer adds: f3r::GpuComposedSolver,
 * a class with the constructor and run() of f3r::ComposedSolver
 * (/root/reference/proj/include/f3r/nesting.hpp:55-77) that solves the whole nest on
 * the B200 through include/f3r_gpu.hpp (the C ABI include/f3rg.h underneath).
 *
 * Code that builds replicas, specs and options through the reference API switches
 * solvers by changing one type:
 *
 *     #include "f3r/errors.hpp"     // first: the adapter then throws f3r::ParseError & co.
 *     #include "f3r/nesting.hpp"
 *     #include "f3r_gpu_adapter.hpp"
 *     ...
 *     f3r::GpuComposedSolver solver(f3r::parse_solver_spec(text), replicas, M);
 *     f3r::RunResult r = solver.run(b, opts);
 *
 * Header-only; needs the reference's include directory on the path and links
 * -lf3rg. The M handed in is mirrored on the device:
 * IdentityPrecond as the identity, a BlockJacobiIlu0 refactorised from the fp64
 * replica with its own config (deterministic, identical factors). */
#ifndef F3R_GPU_ADAPTER_HPP
#define F3R_GPU_ADAPTER_HPP

#include <string>
#include <utility>
#include <vector>

#include "f3r/csr.hpp"
#include "f3r/dense_vector.hpp"
#include "f3r/ilu.hpp"
#include "f3r/nesting.hpp"
#include "f3r/solver_spec.hpp"
#include "f3r_gpu.hpp"

namespace f3r {

class GpuComposedSolver {
 public:
  GpuComposedSolver(const SolverSpec& spec, const PrecisionReplicas& a, const Preconditioner& m)
      : dev_(f3r_gpu::DeviceReplicas::from(a.a64)), m_(device_m(a, m)), s_(spec.to_string(), dev_, m_) {}
  RunResult run(const DenseVector& b, const RunOptions& o = {}) {
    const auto& b64 = b.data<double>();  // the outermost level is fp64 on this path
    f3r_gpu::RunOptions go{o.tol, o.max_outer_restarts, o.max_outer_total, o.reset_richardson_on_restart};
    std::vector<double> x(b64.size(), 0.0);
    const auto g = s_.run(b64.data(), x.data(), go);
    RunResult r{DenseVector(std::move(x)), {}};
    r.report.converged = g.converged;
    r.report.outer_iterations = g.outer_iterations;
    r.report.precond_invocations = g.precond_invocations;
    r.report.level_iterations = g.level_iterations;
    r.report.residual_history = g.residual_history;
    r.report.final_true_residual = g.final_true_residual;
    r.report.wall_seconds = g.wall_seconds;
    r.report.omegas_final = g.omegas_final;
    r.report.flag = g.flag;
    r.report.solver_id = g.solver_id;
    return r;
  }
  std::vector<double> innermost_omegas() { return s_.innermost_omegas(); }
  const std::string& id() const { return s_.id(); }

 private:
  // the same M on the device: a BlockJacobiIlu0 is refactorised there from the fp64
  // replica with its own config (the factorisation is deterministic and identical)
  static f3r_gpu::DevicePreconditioner device_m(const PrecisionReplicas& a, const Preconditioner& m) {
    if (m.rows() != a.a64.rows()) throw DimensionError("preconditioner size mismatch");
    if (const auto* bj = dynamic_cast<const BlockJacobiIlu0*>(&m))
      return f3r_gpu::DevicePreconditioner::factorize(a.a64, bj->config());
    return f3r_gpu::DevicePreconditioner::identity(m.rows());
  }
  f3r_gpu::DeviceReplicas dev_;
  f3r_gpu::DevicePreconditioner m_;
  f3r_gpu::ComposedSolver s_;
};

}  // namespace f3r

#endif  // F3R_GPU_ADAPTER_HPP
