// krylov.cuh -- the reference's fp64 competitor solvers on the device (reference
// src/cg.cpp:22-171: cg_solve, bicgstab_solve) with M = identity or a block-Jacobi
// ILU(0)/IC(0) (its sweeps run between these kernels, trsv.cuh), on the same SpMV
// engine. Every scalar recurrence (alpha, beta, rho, omega, breakdown and stop
// tests) runs in the last CTA of the kernel that completes its reduction, so the
// host enqueues a batch of iterations and synchronises once per batch; a stop
// flag gates the rest of the batch. Element-wise updates follow the reference's
// per-element sequences (axpy: y = fl(fl(a x) + y); add_scaled: out = fl(x +
// fl(a y))); reductions are tree-ordered like every dot on the device.
#pragma once

#include "common.cuh"
#include "levels.cuh"
#include "spmv.cuh"

namespace f3rg {

template <int NV>
__device__ __forceinline__ bool reduce_f64(double (&v)[NV], Sync& sync, double* scratch, double* tot) {
  block_sum<P64, NV>(v, scratch);
  if (threadIdx.x == 0)
    for (int k = 0; k < NV; ++k) sync.partials[(size_t)blockIdx.x * kMaxPart + k] = v[k];
  if (!last_block(sync.counter)) return false;
  reduce_partials<P64, NV>(sync.partials, gridDim.x, kMaxPart, tot, scratch);
  return true;
}

// relative residual after an iteration (both solvers): history, tolerance, cap
__device__ __forceinline__ void record_iteration(KState* S, double rr) {
  S->it += 1;
  const double rel = __ddiv_rn(__dsqrt_rn(rr), S->bnorm);
  if (S->it < S->hist_cap) S->hist[S->it] = rel;
  S->rr = rr;
  if (rel < S->tol) S->stop = KS_TOL;
  else if (S->precond >= S->max_precond) S->stop = KS_CAPPED;
}

// y = A x (fp64) with the dot (u, y) in the epilogue; u row-local
struct EpiDotF64 {
  const double* u;
  double* y;
  double d;
  double ui;
  __device__ __forceinline__ void prefetch(uint32_t i) { ui = __ldg(u + i); }
  __device__ __forceinline__ void row(uint32_t i, double acc) {
    y[i] = acc;
    d = __dadd_rn(d, __dmul_rn(ui, acc));
  }
};
// t = A s with (t, t), (t, s), (s, s)
struct EpiBiT {
  const double* s;
  double* t;
  double tt, ts, ss;
  double si;
  __device__ __forceinline__ void prefetch(uint32_t i) { si = __ldg(s + i); }
  __device__ __forceinline__ void row(uint32_t i, double acc) {
    t[i] = acc;
    tt = __dadd_rn(tt, __dmul_rn(acc, acc));
    ts = __dadd_rn(ts, __dmul_rn(acc, si));
    ss = __dadd_rn(ss, __dmul_rn(si, si));
  }
};

// ---- CG ---------------------------------------------------------------------------
// q = A p, pq = (p, q); alpha = rz / pq, or stop on pq <= 0 (src/cg.cpp:49-52)
template <int IDX>
__global__ void __launch_bounds__(tile_threads(IDX), tile_minb(IDX)) k_cg_spmv(CsrDev A, TilesDev T, const double* p, double* q,
                                                               KState* S, Sync sync) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ double scratch[tile_scratch(IDX)];
  __shared__ double tot[1];
  if (S->stop) return;
  GatherPlain<P64, P64> g{p};
  EpiDotF64 e{p, q, 0.0, 0.0};
  spmv_tiles<P64, P64, IDX>(A, T, g, e, smem);
  double v[1] = {e.d};
  if (!reduce_f64<1>(v, sync, scratch, tot)) return;
  if (threadIdx.x == 0) {
    const double pq = tot[0];
    if (pq <= 0.0) S->stop = KS_INDEFINITE;
    else S->alpha = __ddiv_rn(S->rz, pq);
  }
}

// x += alpha p; r -= alpha q; ||r|| -> history / stop (src/cg.cpp:53-62)
__global__ void __launch_bounds__(256) k_cg_update(double* x, double* r, const double* p, const double* q, uint64_t n,
                                                   KState* S, Sync sync) {
  pdl_wait();
  __shared__ double scratch[64];
  __shared__ double tot[1];
  if (S->stop) return;
  const double a = S->alpha, na = -a;
  double v[1] = {0.0};
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    x[i] = __dadd_rn(__dmul_rn(a, p[i]), x[i]);
    const double ri = __dadd_rn(__dmul_rn(na, q[i]), r[i]);
    r[i] = ri;
    v[0] = __dadd_rn(v[0], __dmul_rn(ri, ri));
  }
  pdl_trigger();
  if (!reduce_f64<1>(v, sync, scratch, tot)) return;
  if (threadIdx.x == 0) record_iteration(S, tot[0]);
  // the post-check part of the iteration (z = r, rz, beta) runs in k_cg_next so
  // that a failed true-residual check can resume exactly where the reference does
}

// after the checks: z = M r = r, rz' = (r, z) = (r, r), beta = rz'/rz (src/cg.cpp:69-75)
__global__ void k_cg_next(KState* S) {
  pdl_wait();
  if (S->stop) return;
  S->precond += 1;
  S->beta = __ddiv_rn(S->rr, S->rz);
  S->rz = S->rr;
}

// with M: rz' = (r, z), z = M r computed by the sweeps; beta = rz'/rz (src/cg.cpp:69-72)
__global__ void __launch_bounds__(256) k_cg_rz(const double* r, const double* z, uint64_t n, KState* S, Sync sync) {
  pdl_wait();
  __shared__ double scratch[64];
  __shared__ double tot[1];
  if (S->stop) return;
  double v[1] = {0.0};
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    v[0] = __dadd_rn(v[0], __dmul_rn(r[i], z[i]));
  pdl_trigger();
  if (!reduce_f64<1>(v, sync, scratch, tot)) return;
  if (threadIdx.x == 0) {
    S->precond += 1;
    S->beta = __ddiv_rn(tot[0], S->rz);
    S->rz = tot[0];
  }
}

// p = z + beta p (add_scaled(z, beta, p, p); z = r when M = identity)
__global__ void __launch_bounds__(256) k_cg_p(double* p, const double* r, uint64_t n, const KState* S) {
  pdl_wait();
  if (S->stop) return;
  const double b = S->beta;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    p[i] = __dadd_rn(r[i], __dmul_rn(b, p[i]));
}

// ---- BiCGStab -----------------------------------------------------------------------
// rho' = (rhat, r) with the breakdown test |rho'| <= eps ||rhat|| ||r||; beta, rho
// (src/cg.cpp:107-115)
__global__ void __launch_bounds__(256) k_bi_rho(const double* rhat, const double* r, uint64_t n, KState* S,
                                                Sync sync) {
  pdl_wait();
  __shared__ double scratch[64 * 3];
  __shared__ double tot[3];
  if (S->stop) return;
  double v[3] = {0.0, 0.0, 0.0};
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double h = rhat[i], ri = r[i];
    v[0] = __dadd_rn(v[0], __dmul_rn(h, ri));
    v[1] = __dadd_rn(v[1], __dmul_rn(h, h));
    v[2] = __dadd_rn(v[2], __dmul_rn(ri, ri));
  }
  pdl_trigger();
  if (!reduce_f64<3>(v, sync, scratch, tot)) return;
  if (threadIdx.x == 0) {
    const double rho_new = tot[0];
    const double lim = __dmul_rn(__dmul_rn(1e-14, __dsqrt_rn(tot[1])), __dsqrt_rn(tot[2]));
    if (fabs(rho_new) <= lim) {
      S->stop = KS_BREAKDOWN;
      return;
    }
    S->beta = __dmul_rn(__ddiv_rn(rho_new, S->rho), __ddiv_rn(S->alpha, S->omega));
    S->rho = rho_new;
  }
}

// p = r + beta (p - omega v): axpy(-omega, v, p); add_scaled(r, beta, p, p)
__global__ void __launch_bounds__(256) k_bi_p(double* p, const double* v, const double* r, uint64_t n,
                                              const KState* S) {
  pdl_wait();
  if (S->stop) return;
  const double no = -S->omega, b = S->beta;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double pi = __dadd_rn(__dmul_rn(no, v[i]), p[i]);
    p[i] = __dadd_rn(r[i], __dmul_rn(b, pi));
  }
}

// phat = M p = p; v = A phat; (rhat, v); alpha = rho / (rhat, v) (src/cg.cpp:120-129)
template <int IDX>
__global__ void __launch_bounds__(tile_threads(IDX), tile_minb(IDX)) k_bi_v(CsrDev A, TilesDev T, const double* p, double* v,
                                                            const double* rhat, KState* S, Sync sync) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ double scratch[tile_scratch(IDX)];
  __shared__ double tot[1];
  if (S->stop) return;
  GatherPlain<P64, P64> g{p};
  EpiDotF64 e{rhat, v, 0.0, 0.0};
  spmv_tiles<P64, P64, IDX>(A, T, g, e, smem);
  double d[1] = {e.d};
  if (!reduce_f64<1>(d, sync, scratch, tot)) return;
  if (threadIdx.x == 0) {
    S->precond += 1;
    const double rv = tot[0];
    if (fabs(rv) < 1e-14) S->stop = KS_BREAKDOWN;
    else S->alpha = __ddiv_rn(S->rho, rv);
  }
}

// s = r - alpha v (add_scaled(r, -alpha, v, s))
__global__ void __launch_bounds__(256) k_bi_s(double* s, const double* r, const double* v, uint64_t n,
                                              const KState* S) {
  pdl_wait();
  if (S->stop) return;
  const double na = -S->alpha;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    s[i] = __dadd_rn(r[i], __dmul_rn(na, v[i]));
}

// shat = M s = s; t = A shat; omega = (t, s) / (t, t), or the t = 0 cases
// (src/cg.cpp:131-147)
template <int IDX>
__global__ void __launch_bounds__(tile_threads(IDX), tile_minb(IDX)) k_bi_t(CsrDev A, TilesDev T, const double* s,
                                                            const double* shat, double* t, KState* S, Sync sync) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ double scratch[tile_scratch(IDX) * 3];
  __shared__ double tot[3];
  if (S->stop) return;
  GatherPlain<P64, P64> g{shat};
  EpiBiT e{s, t, 0.0, 0.0, 0.0, 0.0};
  spmv_tiles<P64, P64, IDX>(A, T, g, e, smem);
  double d[3] = {e.tt, e.ts, e.ss};
  if (!reduce_f64<3>(d, sync, scratch, tot)) return;
  if (threadIdx.x == 0) {
    S->precond += 1;
    const double tt = tot[0];
    if (tt == 0.0) {
      if (__ddiv_rn(__dsqrt_rn(tot[2]), S->bnorm) < S->tol) S->omega = 0.0;
      else S->stop = KS_BREAKDOWN;
    } else {
      S->omega = __ddiv_rn(tot[1], tt);
    }
  }
}

// x += alpha phat; x += omega shat; r = s - omega t; ||r|| (src/cg.cpp:148-160)
__global__ void __launch_bounds__(256) k_bi_update(double* x, double* r, const double* p, const double* s,
                                                   const double* shat, const double* t, uint64_t n, KState* S,
                                                   Sync sync) {
  pdl_wait();
  __shared__ double scratch[64];
  __shared__ double tot[1];
  if (S->stop) return;
  const double a = S->alpha, w = S->omega, nw = -w;
  double v[1] = {0.0};
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double si = s[i];
    double xi = __dadd_rn(__dmul_rn(a, p[i]), x[i]);
    x[i] = __dadd_rn(__dmul_rn(w, shat[i]), xi);
    const double ri = __dadd_rn(si, __dmul_rn(nw, t[i]));
    r[i] = ri;
    v[0] = __dadd_rn(v[0], __dmul_rn(ri, ri));
  }
  pdl_trigger();
  if (!reduce_f64<1>(v, sync, scratch, tot)) return;
  if (threadIdx.x == 0) record_iteration(S, tot[0]);
}

// after a failed true-residual check: continue exactly as the reference's loop
// (cap test, then -- CG only -- the post-check part of the iteration)
__global__ void k_krylov_resume(KState* S) {
  pdl_wait();
  if (S->stop != KS_TOL) return;
  S->stop = S->precond >= S->max_precond ? KS_CAPPED : KS_RUN;
}

}  // namespace f3rg
