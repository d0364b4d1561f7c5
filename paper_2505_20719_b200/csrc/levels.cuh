// levels.cuh -- device kernels of one FGMRES level (reference src/fgmres.cpp:21-148
// and src/nesting.cpp:46-112), all Hessenberg / Givens / least-squares work kept on
// the device so an inner level never synchronises with the host.
//
// Per Arnoldi step j of a level with basis precision W:
//   [child solve on v_j]                 -> z_j  (child's output precision, exact)
//   k_spmv_dots : w = A z_j (C = promote(A, W), rounded to W) fused with the
//                 classical Gram-Schmidt projections h_i = (w, v_i), i <= j
//                 (fp16-F3R: j+1 <= 8 always; larger j adds k_multi_dot passes)
//   k_cgs       : w -= sum_i h_i v_i (sequential axpys per element, as the
//                 reference), ||w||, divergence test, Givens update, estimate
// and per invocation:
//   k_level_start : demote the parent's v_j (cast, src/nesting.cpp:60), ||b||,
//                   v_0 scale -- the Arnoldi start (src/fgmres.cpp:29-54)
//   k_level_finish: back-substitution + x += Z y (src/fgmres.cpp:133-146)
//
// Basis storage: slot j+1 holds the UN-normalised w written by k_cgs together with
// its scale fl_W(1/||w||) (reference scale_in_place, a reciprocal multiply); the
// first kernel that reads v_{j+1} row-locally applies the scale and writes the
// normalised values back, so normalisation costs no extra pass over HBM.
#pragma once

#include "common.cuh"
#include "spmv.cuh"

#include <type_traits>

namespace f3rg {

constexpr int kMaxPart = 16;  // partial slots per block
constexpr int kStageMax = 128;  // Hessenberg columns up to this length are staged in shared memory


struct Gate {
  const int* dead;  // per-level "stopped early" flags
  int n;            // kernel is skipped if any dead[0..n-1] != 0
  __device__ __forceinline__ bool closed() const {
    for (int i = 0; i < n; ++i)
      if (dead[i]) return true;
    return false;
  }
};



struct Sync {
  double* partials;   // gridDim.x * kMaxPart
  unsigned* counter;  // last-block counter
  int seq;            // sequential index-order reductions (validation mode, common.cuh seq_sums)
};

// Cross-rank completion of a reduction under the row-block partition (P > 1,
// SURVEY.md 8(e)); DESIGN.md section 6.
//   mode 0: one rank -- the last CTA runs the tail on its own totals
//   mode 1: the last CTA publishes its rank-local totals to loc[0..NV) and stops
//   mode 2: one CTA combines all[r * kMaxPart + k], r = 0..P-1, in rank order at
//           the reduction precision, then runs the tail (the body is skipped)
// Every rank combines the same P values in the same order, so the replicated
// scalars (Hessenberg column, norms, Givens state) are bitwise equal on all ranks.
struct Dist {
  int mode;
  int P;
  double* loc;
  const double* all;
};

template <int C>
__device__ void combine_ranks(const Dist& d, int nv, double* out) {
  if (threadIdx.x == 0)
    for (int k = 0; k < nv; ++k) {
      T_<C> acc = Ar<C>::zero();
      for (int r = 0; r < d.P; ++r) acc = Ar<C>::add(acc, cvt<C>(d.all[(size_t)r * kMaxPart + k]));
      out[k] = Ar<C>::wide(acc);
    }
  __syncthreads();
}

// mode 1: hand the rank-local totals over and report "stop here"
__device__ __forceinline__ bool publish_local(const Dist& d, int nv, const double* tot) {
  if (d.mode != 1) return false;
  if (threadIdx.x == 0)
    for (int k = 0; k < nv; ++k) d.loc[k] = tot[k];
  return true;
}

// ------------------------------------------------------------------------------
// v_0 of an invocation: dst = demote(src * s) (s optional); optionally write the
// scaled source back (materialising the parent's normalised basis vector); norm.
template <int PS, int PW>
__global__ void __launch_bounds__(256) k_level_start(void* src, const double* src_scale, int writeback, void* dst,
                                                     uint64_t n, LevelState* L, int* dead, Gate gate, int level,
                                                     unsigned long long* cnt, Sync sync, const IoSlot* io, Dist dist) {
  pdl_wait();
  __shared__ double scratch[64];
  __shared__ double tot[1];
  if (gate.closed()) return;
  if (dist.mode != 2) {
    if (io) {
      src = io->src;
      src_scale = io->src_scale;
    }
    const T_<PS> s = src_scale ? cvt<PS>(*src_scale) : Ar<PS>::one();
    T_<PW> acc[1] = {Ar<PW>::zero()};
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t i0 = 0;
    if (!writeback && aligned16(src) && aligned16(dst)) {
      // 8 elements per thread and round: 16-byte transactions, same per-element
      // arithmetic (each thread's running sum just covers 8 neighbours per round)
      const uint64_t ng = n / kGroup;
      for (uint64_t g = tid; g < ng; g += stride) {
        T_<PS> v[kGroup];
        T_<PW> d[kGroup];
        ld8<PS>(src, g, v);
#pragma unroll
        for (int k = 0; k < kGroup; ++k) {
          d[k] = cvt<PW>(src_scale ? Ar<PS>::mul(s, v[k]) : v[k]);
          acc[0] = Ar<PW>::add(acc[0], Ar<PW>::mul(d[k], d[k]));
        }
        st8<PW>(dst, g, d);
      }
      i0 = ng * kGroup;
    }
    for (uint64_t i = i0 + tid; i < n; i += stride) {
      T_<PS> v = ld<PS>(src, i);
      if (src_scale) {
        v = Ar<PS>::mul(s, v);
        if (writeback) st<PS>(src, i, v);
      }
      const T_<PW> d = cvt<PW>(v);
      st<PW>(dst, i, d);
      acc[0] = Ar<PW>::add(acc[0], Ar<PW>::mul(d, d));
    }
    pdl_trigger();
    block_sum<PW, 1>(acc, scratch);
    if (threadIdx.x == 0) sync.partials[(size_t)blockIdx.x * kMaxPart] = Ar<PW>::wide(acc[0]);
    if (!last_block(sync.counter)) return;
    if (sync.seq) {
      seq_sums<PW>(n, 1, [&](uint64_t i, int) {
        const T_<PW> d = ldcg<PW>(dst, i);
        return Ar<PW>::mul(d, d);
      }, tot);
    } else {
      reduce_partials<PW, 1>(sync.partials, gridDim.x, kMaxPart, tot, scratch);
    }
    if (publish_local(dist, 1, tot)) return;
  } else {
    combine_ranks<PW>(dist, 1, tot);
  }
  if (threadIdx.x == 0) {
    using A = Ar<PW>;
    const T_<PW> beta = A::sqrt(cvt<PW>(tot[0]));  // norm2 at the storage precision
    L->beta = A::wide(beta);
    L->bnorm = A::wide(beta);
    L->k = 0;
    L->happy = L->diverged = L->tol_hit = 0;
    L->div_step = -1;
    L->estimate = A::wide(beta);
    L->g[0] = A::wide(beta);
    L->scale[0] = A::wide(A::div(A::one(), beta));
    const bool stop = A::wide(beta) == 0.0 || !A::finite(beta);
    if (stop) L->diverged = !A::finite(beta);
    dead[level] = stop ? 1 : 0;
    cnt[CNT_INV + level] += 1;
  }
}

// z_j = v_j for a level whose child is the identity primary preconditioner
// (src/ilu.cpp:33-36): materialise the normalised basis vector into the Z slot.
template <int PW>
__global__ void __launch_bounds__(256) k_copy_scaled(void* v, const double* scale, void* z, uint64_t n, Gate gate,
                                                     unsigned long long* cnt) {
  pdl_wait();
  if (gate.closed()) return;
  const T_<PW> s = scale ? cvt<PW>(*scale) : Ar<PW>::one();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    T_<PW> x = ld<PW>(v, i);
    if (scale) x = Ar<PW>::mul(s, x);
    st<PW>(z, i, x);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[CNT_PRECOND] += 1;
}

// ------------------------------------------------------------------------------
// w = A z (rounded to W) fused with h_i = (w, v_i) for i < min(j+1, 8).
// fixed-size register "array" addressed only with compile-time indices
template <class T>
struct Reg8 {
  T r0, r1, r2, r3, r4, r5, r6, r7;
  template <int K>
  __device__ __forceinline__ T& at() {
    if constexpr (K == 0) return r0;
    else if constexpr (K == 1) return r1;
    else if constexpr (K == 2) return r2;
    else if constexpr (K == 3) return r3;
    else if constexpr (K == 4) return r4;
    else if constexpr (K == 5) return r5;
    else if constexpr (K == 6) return r6;
    else return r7;
  }
};
template <int K, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (K < N) {
    f(std::integral_constant<int, K>{});
    static_for<K + 1, N>(f);
  }
}

// Basis slots hold UN-normalised vectors; slot k's normalisation factor
// s_k = fl_W(1/||w_k||) (reference scale_in_place, src/fgmres.cpp:88-92) lives in
// L->scale[k] and every consumer forms v_k(i) = fl_W(s_k * w_k(i)) in registers --
// bit-identical to the reference's materialised v_k, without a write-back pass.
template <int C, int PW, int ND>
struct EpiDots {
  void* w;
  void* V;
  uint64_t ld;  // slot stride
  T_<PW> sk[ND];  // s_k
  T_<PW> d[ND];   // partial (w, v_k)
  T_<PW> vk[ND];  // prefetched raw w_k(i)
  __device__ __forceinline__ void prefetch(uint32_t i) {
#pragma unroll
    for (int k = 0; k < ND; ++k) vk[k] = ::f3rg::ld<PW>(V, (uint64_t)k * ld + i);
  }
  __device__ __forceinline__ void row(uint32_t i, T_<C> acc) {
    const T_<PW> wi = cvt<PW>(acc);
#pragma unroll
    for (int k = 0; k < ND; ++k) d[k] = Ar<PW>::add(d[k], Ar<PW>::mul(wi, Ar<PW>::mul(sk[k], vk[k])));
    st<PW>(w, i, wi);
  }
};

template <int PA, int PZ, int PW, int ND, int IDX>
__device__ __forceinline__ void spmv_dots_body(const CsrDev& A, const TilesDev& T, const void* z, void* V, uint64_t ld,
                                               int j, LevelState* L, Sync& sync, double* dots, int defer,
                                               uint8_t* smem, double* scratch, double* res, const Dist& dist) {
  constexpr int C = pmax(PA, PW);
  GatherPlain<PZ, C> g{z};
  EpiDots<C, PW, ND> e;
  e.w = static_cast<uint8_t*>(V) + (size_t)(j + 1) * ld * sizeof(T_<PW>);
  e.V = V;
  e.ld = ld;
#pragma unroll
  for (int k = 0; k < ND; ++k) e.d[k] = Ar<PW>::zero(), e.sk[k] = cvt<PW>(L->scale[k]);
  spmv_tiles<PA, C, IDX>(A, T, g, e, smem);
  T_<PW> dd[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) dd[k] = e.d[k];
  block_sum<PW, ND>(dd, scratch);
  if (threadIdx.x == 0)
    for (int k = 0; k < 8; ++k) dots[(size_t)blockIdx.x * kMaxPart + k] = k < ND ? Ar<PW>::wide(dd[k]) : 0.0;
  if (defer) return;
  if (!last_block(sync.counter)) return;
  if (sync.seq) {  // h_k = dot(w, v_k) in index order, v_k = fl(s_k w_k) (src/fgmres.cpp:71-73)
    const uint64_t n = A.n;
    seq_sums<PW>(n, ND, [&](uint64_t i, int k) {
      const T_<PW> vk = Ar<PW>::mul(cvt<PW>(L->scale[k]), ldcg<PW>(V, (uint64_t)k * ld + i));
      return Ar<PW>::mul(ldcg<PW>(e.w, i), vk);
    }, res);
  } else {
    reduce_partials<PW, ND>(dots, gridDim.x, kMaxPart, res, scratch);
  }
  if (publish_local(dist, ND, res)) return;
  if (threadIdx.x == 0)
    for (int k = 0; k < ND; ++k) L->H[(size_t)j * (L->m + 1) + k] = res[k];
}

// w = A z (rounded to W) fused with the projections h_k = (w, v_k), k < min(j+1, 8)
// (the projection count is a compile-time parameter of the epilogue: runtime
// predication there cost ~140 instructions per row). defer != 0: only per-CTA
// partials are written (to `dots`); the following k_cgs reduces them.
// V: slot 0 of the basis (owned rows); ld: slot stride; z: the SpMV input (ext layout)
template <int PA, int PZ, int PW, int IDX>
__global__ void __launch_bounds__(tile_threads(IDX), tile_minb(IDX)) k_spmv_dots(CsrDev A, TilesDev T, const void* z, void* V, uint64_t ld, int j,
                                                   LevelState* L, Gate gate, Sync sync, double* dots, int defer,
                                                   Dist dist) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ double scratch[tile_scratch(IDX)];
  __shared__ double res[8];
  if (gate.closed()) return;
  if (dist.mode == 2) {
    const int nd = j + 1 < 8 ? j + 1 : 8;
    combine_ranks<PW>(dist, nd, res);
    if (threadIdx.x == 0)
      for (int k = 0; k < nd; ++k) L->H[(size_t)j * (L->m + 1) + k] = res[k];
    return;
  }
  switch (j + 1 < 8 ? j + 1 : 8) {
#define F3RG_ND(K) \
  case K: spmv_dots_body<PA, PZ, PW, K, IDX>(A, T, z, V, ld, j, L, sync, dots, defer, smem, scratch, res, dist); break;
    F3RG_ND(1) F3RG_ND(2) F3RG_ND(3) F3RG_ND(4) F3RG_ND(5) F3RG_ND(6) F3RG_ND(7)
    default: spmv_dots_body<PA, PZ, PW, 8, IDX>(A, T, z, V, ld, j, L, sync, dots, defer, smem, scratch, res, dist);
#undef F3RG_ND
  }
}

// remaining projections h_k, k in [k0, min(k0+8, j+1)), for long outer cycles
template <int PW>
__global__ void __launch_bounds__(256) k_multi_dot(const void* V, uint64_t n, uint64_t ldv, int j, int k0,
                                                   LevelState* L, Gate gate, Sync sync, Dist dist) {
  pdl_wait();
  __shared__ double scratch[8 * 8];
  __shared__ double res[8];
  if (gate.closed()) return;
  const int nd = (j + 1 - k0) < 8 ? (j + 1 - k0) : 8;
  if (dist.mode == 2) {
    combine_ranks<PW>(dist, nd, res);
    if (threadIdx.x == 0)
      for (int k = 0; k < nd; ++k) L->H[(size_t)j * (L->m + 1) + k0 + k] = res[k];
    return;
  }
  T_<PW> d[8], s[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    d[k] = Ar<PW>::zero();
    s[k] = k < nd ? cvt<PW>(L->scale[k0 + k]) : Ar<PW>::zero();
  }
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const T_<PW> wi = ld<PW>(V, (uint64_t)(j + 1) * ldv + i);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < nd)
        d[k] = Ar<PW>::add(d[k], Ar<PW>::mul(wi, Ar<PW>::mul(s[k], ld<PW>(V, (uint64_t)(k0 + k) * ldv + i))));
  }
  block_sum<PW, 8>(d, scratch);
  if (threadIdx.x == 0)
    for (int k = 0; k < 8; ++k) sync.partials[(size_t)blockIdx.x * kMaxPart + k] = Ar<PW>::wide(d[k]);
  if (!last_block(sync.counter)) return;
  if (sync.seq) {
    seq_sums<PW>(n, nd, [&](uint64_t i, int k) {
      const T_<PW> vk = Ar<PW>::mul(cvt<PW>(L->scale[k0 + k]), ldcg<PW>(V, (uint64_t)(k0 + k) * ldv + i));
      return Ar<PW>::mul(ldcg<PW>(V, (uint64_t)(j + 1) * ldv + i), vk);
    }, res);
  } else {
    reduce_partials<PW, 8>(sync.partials, gridDim.x, kMaxPart, res, scratch);
  }
  if (publish_local(dist, nd, res)) return;
  if (threadIdx.x == 0)
    for (int k = 0; k < nd; ++k) L->H[(size_t)j * (L->m + 1) + k0 + k] = res[k];
}

// ------------------------------------------------------------------------------
// CGS subtraction + norm + Givens (src/fgmres.cpp:74-129). With dots != nullptr the
// projections are first reduced from k_spmv_dots' per-CTA partials (every CTA in
// the same fixed order -> identical h in all CTAs; CTA 0 records the H column).
// `outer` levels never set their dead flag (the host decides) and report through
// `info`.
// NJ = min(j + 1, 8) is a kernel template parameter (one instantiation per
// projection count): the small-NJ kernels then need few registers, run more CTAs
// per SM and keep two rounds of 16-byte loads in flight per thread.
// shared memory of the CGS body (declared by the calling kernel: one copy however
// many cgs_body instantiations a kernel holds)
struct CgsSmem {
  double scratch[64];
  double hs[128];
  double tot[8];
  double hc[kStageMax + 1], cs[kStageMax], sn[kStageMax], gj_tol[3];
};

template <int PW, int NJ>
__device__ __forceinline__ void cgs_body(void* V, uint64_t n, uint64_t ldv, int j, LevelState* L, int* dead,
                                         int level, int outer, int use_tol, StepInfo* info, Sync sync,
                                         const double* dots, int dots_G, Dist dist, CgsSmem& sm) {
  double* scratch = sm.scratch;
  double* hs = sm.hs;
  double* tot = sm.tot;
  using A = Ar<PW>;
  const int m1 = L->m + 1;
  double* h = L->H + (size_t)j * m1;
  const int nh = j + 1 <= 128 ? j + 1 : 128;
  if (dist.mode != 2) {
  // the projections: reduced here from k_spmv_dots' partials (deferred) or read
  // from H; called after each thread has issued its first streaming loads so the
  // reduction's latency hides under them
  auto get_h = [&]() {
    if (dots) {  // j + 1 <= 8 here
      reduce_partials<PW, 8>(dots, dots_G, kMaxPart, tot, scratch);
      for (int k = threadIdx.x; k < nh; k += blockDim.x) hs[k] = -tot[k];
      if (blockIdx.x == 0 && threadIdx.x < nh) h[threadIdx.x] = tot[threadIdx.x];
    } else {
      for (int k = threadIdx.x; k < nh; k += blockDim.x) hs[k] = -h[k];
    }
    __syncthreads();
  };
  T_<PW> acc[1] = {A::zero()};
  T_<PW>* w = static_cast<T_<PW>*>(V) + (size_t)(j + 1) * ldv;
  constexpr int VE = 16 / (int)sizeof(T_<PW>);
  constexpr bool DEEP = NJ <= 4;  // two load rounds in flight
  T_<PW> a[NJ], sc[NJ];
  auto update = [&](uint64_t i, T_<PW> wi, const T_<PW>* vv) {
#pragma unroll
    for (int u = 0; u < NJ; ++u) wi = A::add(A::mul(a[u], A::mul(sc[u], vv[u])), wi);
    for (int k = NJ; k <= j; ++k) {  // long outer cycles only
      const T_<PW> v = A::mul(cvt<PW>(L->scale[k]), ld<PW>(V, (uint64_t)k * ldv + i));
      wi = A::add(A::mul(k < 128 ? cvt<PW>(hs[k]) : cvt<PW>(-h[k]), v), wi);
    }
    acc[0] = A::add(acc[0], A::mul(wi, wi));
    return wi;
  };
  auto coefficients = [&]() {
#pragma unroll
    for (int u = 0; u < NJ; ++u) a[u] = cvt<PW>(hs[u]), sc[u] = cvt<PW>(L->scale[u]);
  };
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  if (n % VE == 0 && ldv % VE == 0) {
    const uint64_t nv = n / VE;
    const uint4* w4 = reinterpret_cast<const uint4*>(w);
    struct Round {
      uint4 v[NJ];
      uint4 w;
    };
    auto load = [&](Round& r, uint64_t e) {
#pragma unroll
      for (int u = 0; u < NJ; ++u)
        r.v[u] = reinterpret_cast<const uint4*>(static_cast<const T_<PW>*>(V) + (uint64_t)u * ldv)[e];
      r.w = w4[e];
    };
    auto process = [&](const Round& r, uint64_t e) {
      T_<PW> wv[VE];
      memcpy(wv, &r.w, 16);
#pragma unroll
      for (int l = 0; l < VE; ++l) {
        T_<PW> vv[NJ];
#pragma unroll
        for (int u = 0; u < NJ; ++u)
          memcpy(&vv[u], reinterpret_cast<const char*>(&r.v[u]) + l * sizeof(T_<PW>), sizeof(T_<PW>));
        wv[l] = update(e * VE + l, wv[l], vv);
      }
      uint4 out;
      memcpy(&out, wv, 16);
      reinterpret_cast<uint4*>(w)[e] = out;
    };
    if constexpr (DEEP) {
      Round r0, r1;
      uint64_t e = tid;
      if (e < nv) load(r0, e);
      if (e + stride < nv) load(r1, e + stride);
      get_h();
      coefficients();
      while (e < nv) {
        process(r0, e);
        if (e + 2 * stride < nv) load(r0, e + 2 * stride);
        e += stride;
        if (e >= nv) break;
        process(r1, e);
        if (e + 2 * stride < nv) load(r1, e + 2 * stride);
        e += stride;
      }
    } else {
      Round r0;
      uint64_t e = tid;
      if (e < nv) load(r0, e);
      get_h();
      coefficients();
      for (; e < nv;) {
        process(r0, e);
        e += stride;
        if (e < nv) load(r0, e);
      }
    }
  } else {
    get_h();
    coefficients();
    for (uint64_t i = tid; i < n; i += stride) {
      T_<PW> vv[NJ];
#pragma unroll
      for (int u = 0; u < NJ; ++u) vv[u] = ld<PW>(V, (uint64_t)u * ldv + i);
      w[i] = update(i, w[i], vv);
    }
  }
  pdl_trigger();
  block_sum<PW, 1>(acc, scratch);
  if (threadIdx.x == 0) sync.partials[(size_t)blockIdx.x * kMaxPart] = A::wide(acc[0]);
  if (!last_block(sync.counter)) return;
  }  // dist.mode != 2
  // Givens tail: one parallel round trip stages the small state (column j of H,
  // the previous rotations, g_j) in shared memory, overlapped with the partials
  // reduction; thread 0 then runs the serial recurrence out of shared memory
  // instead of a chain of dependent global loads
  double* hc = sm.hc;
  double* cs = sm.cs;
  double* sn = sm.sn;
  double* gj_tol = sm.gj_tol;
  const bool staged = j < kStageMax;
  if (staged) {
    for (int i = threadIdx.x; i <= j; i += blockDim.x) hc[i] = __ldcg(h + i);
    for (int i = threadIdx.x; i < j; i += blockDim.x) cs[i] = __ldcg(L->cs + i), sn[i] = __ldcg(L->sn + i);
    if (threadIdx.x == 0) gj_tol[0] = __ldcg(L->g + j), gj_tol[1] = L->tol, gj_tol[2] = L->bnorm;
  }
  if (dist.mode != 2) {
    if (sync.seq) {  // ||w||^2 in index order (norm2, src/fgmres.cpp:77)
      T_<PW>* w = static_cast<T_<PW>*>(V) + (size_t)(j + 1) * ldv;
      seq_sums<PW>(n, 1, [&](uint64_t i, int) {
        const T_<PW> wi = ldcg<PW>(w, i);
        return A::mul(wi, wi);
      }, tot);
    } else {
      reduce_partials<PW, 1>(sync.partials, gridDim.x, kMaxPart, tot, scratch);  // ends with __syncthreads
    }
    if (publish_local(dist, 1, tot)) return;
  } else {
    combine_ranks<PW>(dist, 1, tot);
  }
  if (threadIdx.x != 0) return;
  double* hh = staged ? hc : h;
  const double* csr = staged ? cs : L->cs;
  const double* snr = staged ? sn : L->sn;

  const T_<PW> wnorm = A::sqrt(cvt<PW>(tot[0]));
  hh[j + 1] = A::wide(wnorm);
  bool bad = !A::finite(wnorm);
  for (int i = 0; i <= j + 1; ++i) bad = bad || !isfinite(hh[i]);
  bool stop = false;
  if (bad) {
    L->diverged = 1;
    L->div_step = j;
    stop = true;
  } else {
    const bool happy = A::wide(wnorm) == 0.0;
    if (!happy) L->scale[j + 1] = A::wide(A::div(A::one(), wnorm));
    // apply the accumulated rotations to column j, then generate the new one
    for (int i = 0; i < j; ++i) {
      const T_<PW> c = cvt<PW>(csr[i]), s = cvt<PW>(snr[i]);
      const T_<PW> hi = cvt<PW>(hh[i]), hi1 = cvt<PW>(hh[i + 1]);
      const T_<PW> t = A::add(A::mul(c, hi), A::mul(s, hi1));
      hh[i + 1] = A::wide(A::add(A::mul(A::neg(s), hi), A::mul(c, hi1)));
      hh[i] = A::wide(t);
    }
    const T_<PW> hj = cvt<PW>(hh[j]), hj1 = cvt<PW>(hh[j + 1]);
    const T_<PW> rho = A::hypot(hj, hj1);
    T_<PW> c, s;
    if (A::wide(rho) == 0.0) {
      c = A::one();
      s = A::zero();
    } else {
      c = A::div(hj, rho);
      s = A::div(hj1, rho);
    }
    L->cs[j] = A::wide(c);
    L->sn[j] = A::wide(s);
    hh[j] = A::wide(rho);
    hh[j + 1] = 0.0;
    const T_<PW> gj = cvt<PW>(staged ? gj_tol[0] : L->g[j]);
    const double gj1 = A::wide(A::mul(A::neg(s), gj));
    L->g[j + 1] = gj1;
    L->g[j] = A::wide(A::mul(c, gj));
    L->k = j + 1;
    const double est = fabs(gj1);
    L->estimate = est;
    if (happy) {
      L->happy = 1;
      stop = true;
    } else if (use_tol && est < (staged ? gj_tol[1] * gj_tol[2] : L->tol * L->bnorm)) {
      L->tol_hit = 1;
      stop = true;
    }
  }
  if (staged)
    for (int i = 0; i <= j + 1; ++i) h[i] = hc[i];
  if (!outer && stop) dead[level] = 1;
  if (info) {
    info->estimate = L->estimate;
    info->k = L->k;
    info->happy = L->happy;
    info->diverged = L->diverged;
    info->div_step = L->div_step;
    info->tol_hit = L->tol_hit;
  }
}

template <int PW, int NJ>
__global__ void __launch_bounds__(256, NJ <= 2 ? 4 : NJ <= 4 ? 3 : 2) k_cgs(void* V, uint64_t n, uint64_t ldv, int j, LevelState* L, int* dead,
                                             Gate gate, int level, int outer, int use_tol, StepInfo* info, Sync sync,
                                             const double* dots, int dots_G, Dist dist) {
  pdl_wait();
  __shared__ CgsSmem sm;
  if (gate.closed()) return;
  cgs_body<PW, NJ>(V, n, ldv, j, L, dead, level, outer, use_tol, info, sync, dots, dots_G, dist, sm);
}


// ------------------------------------------------------------------------------
// Back-substitution (in W) + x (+)= sum_l y_l z_l, sequential axpys per element
// (src/fgmres.cpp:133-146). x_is_zero: inner levels start from fill(out, 0).
template <int PZ, int PW, int PX>
__global__ void __launch_bounds__(256) k_level_finish(const void* Z, uint64_t n, uint64_t ldz, LevelState* L, void* x,
                                                      int x_is_zero, Gate gate, int level, unsigned long long* cnt,
                                                      int count_iterations, const IoSlot* io) {
  pdl_wait();
  __shared__ double ys[1024];
  if (gate.closed()) return;
  if (io) x = io->dst;
  using A = Ar<PW>;
  const int k = L->k;
  const int m1 = L->m + 1;
  // inner levels (k <= 16): stage the triangle of H and g in shared memory with one
  // parallel round trip, so thread 0's back-substitution never waits on global loads
  constexpr int KS = 16;
  __shared__ double Hs[KS * KS], gs[KS];
  const bool staged = k <= KS;
  if (staged) {
    const double* H = L->H;
    for (int t = threadIdx.x; t < k * k; t += blockDim.x) {
      const int l = t / k, i = t - l * k;
      if (l >= i) Hs[l * KS + i] = H[(size_t)l * m1 + i];
    }
    if (threadIdx.x < k) gs[threadIdx.x] = L->g[threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (int i = k - 1; i >= 0; --i) {
      T_<PW> acc = cvt<PW>(staged ? gs[i] : L->g[i]);
      for (int l = i + 1; l < k; ++l)
        acc = A::sub(acc, A::mul(cvt<PW>(staged ? Hs[l * KS + i] : L->H[(size_t)l * m1 + i]), cvt<PW>(ys[l])));
      ys[i] = A::wide(A::div(acc, cvt<PW>(staged ? Hs[i * KS + i] : L->H[(size_t)i * m1 + i])));
    }
    if (blockIdx.x == 0) {
      for (int i = 0; i < k; ++i) L->y[i] = ys[i];
      if (count_iterations) cnt[CNT_IT + level] += (unsigned long long)k;
    }
  }
  __syncthreads();
  constexpr int C = pmax(PW, PX);  // axpy(y, z, x): compute at promote(z, x)
  using AC = Ar<C>;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  // first <= 8 coefficients in registers, loop specialised on their count
  auto body = [&](auto K_) {
    constexpr int K = decltype(K_)::value;
    T_<C> yy[K > 0 ? K : 1];
#pragma unroll
    for (int u = 0; u < K; ++u) yy[u] = cvt<C>(ys[u]);
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t i0 = 0;
    if (k <= K && ldz % kGroup == 0 && aligned16(Z) && aligned16(x)) {
      // 8 elements per thread and round (16-byte transactions), same sequential
      // per-element axpy order as below
      const uint64_t ng = n / kGroup;
      for (uint64_t g = tid; g < ng; g += stride) {
        T_<PX> xv[kGroup];
        if (x_is_zero) {
#pragma unroll
          for (int e = 0; e < kGroup; ++e) xv[e] = cvt<PX>(0.0);
        } else {
          ld8<PX>(x, g, xv);
        }
#pragma unroll
        for (int u = 0; u < K; ++u) {
          T_<PZ> zz[kGroup];
          ld8<PZ>(static_cast<const T_<PZ>*>(Z) + (uint64_t)u * ldz, g, zz);
#pragma unroll
          for (int e = 0; e < kGroup; ++e) xv[e] = cvt<PX>(AC::add(AC::mul(yy[u], cvt<C>(zz[e])), cvt<C>(xv[e])));
        }
        st8<PX>(x, g, xv);
      }
      i0 = ng * kGroup;
    }
    for (uint64_t i = i0 + tid; i < n; i += stride) {
      T_<PZ> zz[K > 0 ? K : 1];
#pragma unroll
      for (int u = 0; u < K; ++u) zz[u] = ld<PZ>(Z, (uint64_t)u * ldz + i);
      T_<PX> xi = x_is_zero ? cvt<PX>(0.0) : ld<PX>(x, i);
#pragma unroll
      for (int u = 0; u < K; ++u) xi = cvt<PX>(AC::add(AC::mul(yy[u], cvt<C>(zz[u])), cvt<C>(xi)));
      for (int l = K; l < k; ++l)  // long outer cycles only
        xi = cvt<PX>(AC::add(AC::mul(cvt<C>(ys[l]), cvt<C>(ld<PZ>(Z, (uint64_t)l * ldz + i))), cvt<C>(xi)));
      st<PX>(x, i, xi);
    }
  };
  switch (k < 8 ? k : 8) {
    case 0: body(std::integral_constant<int, 0>{}); break;
    case 1: body(std::integral_constant<int, 1>{}); break;
    case 2: body(std::integral_constant<int, 2>{}); break;
    case 3: body(std::integral_constant<int, 3>{}); break;
    case 4: body(std::integral_constant<int, 4>{}); break;
    case 5: body(std::integral_constant<int, 5>{}); break;
    case 6: body(std::integral_constant<int, 6>{}); break;
    case 7: body(std::integral_constant<int, 7>{}); break;
    default: body(std::integral_constant<int, 8>{}); break;
  }
}

// ------------------------------------------------------------------------------
// r = b - A x (restart residual / true residual, src/fgmres.cpp:31-38,
// src/nesting.cpp:165-173) with ||r||^2 partials. ax is rounded to W first,
// exactly as op.multiply(x, ax) followed by add_scaled(b, -1, ax, r).
template <int C, int PW>
struct EpiResidual {
  const double* b;  // fp64 right-hand side
  void* r;
  T_<PW> acc;
  double bi;
  __device__ __forceinline__ void prefetch(uint32_t i) { bi = __ldg(b + i); }
  __device__ __forceinline__ void row(uint32_t i, T_<C> y) {
    constexpr int CR = pmax(P64, PW);  // promote(b=f64, ax=W, r=W)
    const T_<CR> ax = cvt<CR>(cvt<PW>(y));
    const T_<PW> ri = cvt<PW>(Ar<CR>::add(cvt<CR>(bi), Ar<CR>::neg(ax)));
    st<PW>(r, i, ri);
    acc = Ar<PW>::add(acc, Ar<PW>::mul(ri, ri));
  }
};

// result: L (if non-null) gets the Arnoldi start like k_level_start; norm2 (W) is
// also written to *out_norm.
// x: ext layout (gathered); b, r: owned rows
template <int PA, int PX, int PW, int IDX>
__global__ void __launch_bounds__(tile_threads(IDX), tile_minb(IDX)) k_residual(CsrDev A, TilesDev T, const void* x, const double* b, void* r,
                                                  LevelState* L, double* out_norm, Sync sync, Dist dist) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ double scratch[tile_scratch(IDX)];
  __shared__ double tot[1];
  if (dist.mode != 2) {
    constexpr int C = pmax(PA, PX);
    GatherPlain<PX, C> g{x};
    EpiResidual<C, PW> e{b, r, Ar<PW>::zero(), 0.0};
    spmv_tiles<PA, C, IDX>(A, T, g, e, smem);
    T_<PW> acc[1] = {e.acc};
    block_sum<PW, 1>(acc, scratch);
    if (threadIdx.x == 0) sync.partials[(size_t)blockIdx.x * kMaxPart] = Ar<PW>::wide(acc[0]);
    if (!last_block(sync.counter)) return;
    if (sync.seq) {
      seq_sums<PW>(A.n, 1, [&](uint64_t i, int) {
        const T_<PW> ri = ldcg<PW>(r, i);
        return Ar<PW>::mul(ri, ri);
      }, tot);
    } else {
      reduce_partials<PW, 1>(sync.partials, gridDim.x, kMaxPart, tot, scratch);
    }
    if (publish_local(dist, 1, tot)) return;
  } else {
    combine_ranks<PW>(dist, 1, tot);
  }
  if (threadIdx.x == 0) {
    using AW = Ar<PW>;
    const T_<PW> beta = AW::sqrt(cvt<PW>(tot[0]));
    if (out_norm) *out_norm = AW::wide(beta);
    if (L) {
      L->beta = AW::wide(beta);
      L->k = 0;
      L->happy = L->diverged = L->tol_hit = 0;
      L->div_step = -1;
      L->estimate = AW::wide(beta);
      L->g[0] = AW::wide(beta);
      L->scale[0] = AW::wide(AW::div(AW::one(), beta));
    }
  }
}

}  // namespace f3rg
