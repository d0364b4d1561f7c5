// dropin_reference_api.cpp -- TEST: a program written against the reference's own
// C++ API (f3r::generate_stencil, diagonal_scale, make_replicas, IdentityPrecond,
// build(parse_solver_spec(...)), ComposedSolver::run) that swaps in the device
// solver through the adapter a reference maintainer would add (INTEGRATION.md
// "C++"), then solves the same system both ways and prints one JSON line.
//
// Built by `make -C oracle dropin` against the reference headers and the reference
// library compiled from its sources (oracle/_ref/libf3r_ref.so); the binary lands
// in oracle/_ref/ and is run by tests/test_dropin.py on the GPU box.
//
// usage: dropin_reference_api <log2_n> <beta> [spec] [identity|ic0|ilu0]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>

#include "f3r/errors.hpp"  // first: f3r_gpu then rethrows the reference's exception classes
#include "f3r/csr.hpp"
#include "f3r/dense_vector.hpp"
#include "f3r/ilu.hpp"
#include "f3r/nesting.hpp"
#include "f3r/scaling.hpp"
#include "f3r/solver_spec.hpp"
#include "f3r/stencil.hpp"
#include "f3r_gpu_adapter.hpp"  // f3r::GpuComposedSolver, the shipped drop-in

int main(int argc, char** argv) {
  const int lg = argc > 1 ? std::atoi(argv[1]) : 5;
  const double beta = argc > 2 ? std::atof(argv[2]) : 0.0;
  const std::string spec_text =
      argc > 3 ? argv[3] : "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > identity";

  // reference problem setup (27-point stencil, x_true = 1, unit-diagonal scaling)
  f3r::SparseCsr a = f3r::generate_stencil(f3r::StencilSpec{lg, lg, lg, beta});
  f3r::DenseVector ones(std::vector<double>(a.rows(), 1.0));
  f3r::DenseVector b(a.rows(), f3r::Precision::P64);
  f3r::spmv(a, ones, b);
  f3r::ScaledSystem sys = f3r::diagonal_scale(a, b);
  f3r::PrecisionReplicas reps = f3r::make_replicas(std::move(sys.matrix));
  const std::string mkind = argc > 4 ? argv[4] : "identity";
  std::unique_ptr<f3r::Preconditioner> mp;
  if (mkind == "identity") {
    mp = std::make_unique<f3r::IdentityPrecond>(reps.a64.rows());
  } else {  // the reference bench's default M: 4 blocks, alpha 1, fp16 factors
    f3r::IluConfig cfg;
    cfg.nblocks = 4;
    cfg.symmetric = mkind == "ic0";
    cfg.apply_precision = f3r::Precision::P16;
    mp = std::make_unique<f3r::BlockJacobiIlu0>(f3r::BlockJacobiIlu0::factorize(reps.a64, cfg));
  }
  const f3r::Preconditioner& m = *mp;
  const f3r::SolverSpec spec = f3r::parse_solver_spec(spec_text);
  f3r::RunOptions opts;
  opts.tol = 1e-10;

  f3r::ComposedSolver cpu = f3r::build(spec, reps, m);
  const f3r::RunResult rc = cpu.run(sys.rhs, opts);

  f3r::GpuComposedSolver gpu(spec, reps, m);
  const f3r::RunResult rg = gpu.run(sys.rhs, opts);

  double dx = 0.0, xn = 0.0;
  for (std::size_t i = 0; i < rc.x.size(); ++i) {
    const double d = rc.x.at(i) - rg.x.at(i);
    dx += d * d;
    xn += rc.x.at(i) * rc.x.at(i);
  }
  // error path: a malformed spec must surface as the reference's own ParseError
  bool parse_error = false;
  try {
    f3r_gpu::ComposedSolver bad("F8:f32/f32 >", f3r_gpu::DeviceReplicas::from(reps.a64));
  } catch (const f3r::ParseError&) {
    parse_error = true;
  }
  std::printf(
      "{\"n\": %zu, \"nnz\": %zu, \"id_cpu\": \"%s\", \"id_gpu\": \"%s\", "
      "\"cpu\": {\"converged\": %d, \"outer\": %llu, \"res\": %.6e, \"s\": %.4f}, "
      "\"gpu\": {\"converged\": %d, \"outer\": %llu, \"res\": %.6e, \"s\": %.4f}, "
      "\"x_rel_diff\": %.6e, \"parse_error_is_f3r\": %d}\n",
      reps.a64.rows(), reps.a64.nnz(), cpu.id().c_str(), gpu.id().c_str(), rc.report.converged ? 1 : 0,
      (unsigned long long)rc.report.outer_iterations, rc.report.final_true_residual, rc.report.wall_seconds,
      rg.report.converged ? 1 : 0, (unsigned long long)rg.report.outer_iterations, rg.report.final_true_residual,
      rg.report.wall_seconds, std::sqrt(dx / xn), parse_error ? 1 : 0);
  return 0;
}
