// richardson.cuh -- the innermost weighted-Richardson solve (reference
// src/richardson.cpp:10-54, include/f3r/richardson.hpp:26-53) with the identity
// primary preconditioner, as ONE kernel per invocation.
//
// Non-update calls (63 of every 64 with c = 64) take the fused sweep: with z0 = 0
// and M = I, z1 = fl(fl(w0*v) + 0) is an element-wise function of v, so the m = 2
// solve  z2 = z1 + w1 (v - A z1)  is a single SpMV pass that recomputes z1 on the
// fly for every gathered column. The residual and z1 never touch HBM: the pass
// reads v (the parent's basis vector, demoted in-register), A16 + indices and
// writes z2 -- SURVEY.md Appendix A.1's exact per-element sequence.
//
// Update calls (call_count % c == 0) compute w' = (r, A r) / (A r, A r) at >= fp32
// with device-side reductions and grid barriers (the kernel is launched
// cooperatively so all CTAs are co-resident); the weight bookkeeping (cumulative
// average with l = call_count/c - 1, degenerate fallback) runs on the device, so
// no call ever synchronises with the host.
#pragma once

#include "common.cuh"
#include "levels.cuh"
#include "spmv.cuh"

namespace f3rg {


// gather chunk of the Richardson passes: with the P16 stream a chunk's values ride
// in registers next to its gathers, and chunks of 16 spill in this kernel
// (measured ~2 % slower than 8)
#ifndef F3RG_RICH_CHUNK
#define F3RG_RICH_CHUNK 9
#endif
#ifndef F3RG_WSELL_Z1  // windowed engine: materialise z1 before the plain Richardson pass (A/B: 0)
#define F3RG_WSELL_Z1 1
#endif
constexpr int rich_chunk(int idx) { return idx == 2 ? F3RG_RICH_CHUNK : 0; }  // short shape: its own chunk

// Right-hand side of the call: v_i = demote(s * parent_v_i) (s optional). v is in
// the ext layout (row-block partition): gathers index it by ext column, row-local
// reads by owned row + off (off = 0 on a single rank).
template <int PV, int PW>
struct RhsView {
  const void* v;
  T_<PV> s;
  bool scaled;
  uint64_t off;
  __device__ __forceinline__ T_<PV> raw(uint64_t c) const { return ldg<PV>(v, c); }
  __device__ __forceinline__ T_<PV> raw_row(uint64_t i) const { return ldg<PV>(v, i + off); }
  __device__ __forceinline__ T_<PW> row(uint64_t i) const { return apply(raw_row(i)); }
  // s = 1 when unscaled: fl(1 * x) == x exactly (no flush-to-zero), so no select
  __device__ __forceinline__ T_<PW> apply(T_<PV> x) const { return cvt<PW>(Ar<PV>::mul(s, x)); }
  __device__ __forceinline__ T_<PW> operator()(uint64_t i) const { return apply(raw(i)); }
};

// z1 = fl(fl(w0 * v) + 0) -- axpy into a zero-filled z; the +0 only turns -0 into
// +0. As a SpMV operand the sign of a zero z1 cannot matter: the row accumulator
// starts at +0 and an RNE sum is -0 only if both addends are -0, so it is never
// -0 and acc + (+-0) == acc. The gather therefore skips the +0 (bit-exact); the
// epilogue, where z1 is added to a possibly -0 term, keeps it.
template <int PV, int PW, int C>
struct GatherZ1 {
  using Raw = T_<PV>;
  RhsView<PV, PW> rhs;
  T_<PW> w0;
  uint64_t pol = 0;  // L2 policy of the windowed engine's ring fills / far gathers (0: plain loads)
  __device__ __forceinline__ void set_policy(uint64_t) {}
  __device__ __forceinline__ void set_ring_policy(uint64_t p) { pol = p; }
  __device__ __forceinline__ Raw load(uint32_t c) const { return pol ? ldg_hint<PV>(rhs.v, c, pol) : rhs.raw(c); }
  __device__ __forceinline__ T_<C> value(Raw r) const { return cvt<C>(Ar<PW>::mul(w0, rhs.apply(r))); }
  // windowed engine: the ring holds z1 itself (wsell.cuh WsRing)
  using RingT = T_<PW>;
  __device__ __forceinline__ RingT ring_put(Raw r) const { return Ar<PW>::mul(w0, rhs.apply(r)); }
  __device__ __forceinline__ T_<C> ring_get(RingT z) const { return cvt<C>(z); }
};

// the right-hand side itself as the SpMV operand (update call, step 0: p = r = v)
template <int PV, int PW, int C>
struct GatherRhs {
  using Raw = T_<PV>;
  RhsView<PV, PW> rhs;
  uint64_t pol = 0;
  __device__ __forceinline__ void set_policy(uint64_t) {}
  __device__ __forceinline__ void set_ring_policy(uint64_t p) { pol = p; }
  __device__ __forceinline__ Raw load(uint32_t c) const { return pol ? ldg_hint<PV>(rhs.v, c, pol) : rhs.raw(c); }
  __device__ __forceinline__ T_<C> value(Raw r) const { return cvt<C>(rhs.apply(r)); }
  using RingT = T_<PW>;
  __device__ __forceinline__ RingT ring_put(Raw r) const { return rhs.apply(r); }
  __device__ __forceinline__ T_<C> ring_get(RingT z) const { return cvt<C>(z); }
};

// one fused step k >= 1: r = v - A z_k ; z_{k+1} = z_k + w_k r  (M = I, p = r)
template <int PV, int PW, int C, bool Z1_ON_THE_FLY>
struct EpiStep {
  RhsView<PV, PW> rhs;
  T_<PW> w0, wk;
  const void* zk;  // materialised z_k (when not on the fly)
  void* out;
  T_<PV> vraw;  // raw loads only in prefetch: their latency hides behind the row sum
  T_<PW> zi;
  __device__ __forceinline__ void prefetch(uint32_t i) {
    vraw = rhs.raw_row(i);
    if constexpr (!Z1_ON_THE_FLY) zi = ldcg<PW>(zk, i);
  }
  __device__ __forceinline__ void row(uint32_t i, T_<C> acc) {
    using A = Ar<PW>;
    const T_<PW> s = cvt<PW>(acc);
    const T_<PW> vi = rhs.apply(vraw);
    const T_<PW> r = A::add(vi, A::neg(s));  // add_scaled(v, -1, s): C = wp, -1*s exact
    if constexpr (Z1_ON_THE_FLY) zi = A::add(A::mul(w0, vi), A::zero());
    st<PW>(out, i, A::add(A::mul(wk, r), zi));
  }
};

// update-call phase B: s = A p (rounded to wp), (r, s) and (s, s) at >= fp32
template <int PV, int PW, int C, int CD>
struct EpiDotsRs {
  RhsView<PV, PW> rhs;
  const void* R;  // p = r (nullptr: r = v)
  T_<CD> num, den;
  T_<PW> rr;
  T_<PV> vraw;
  void* S = nullptr;  // sequential reductions: s materialised for the in-order recomputation
  __device__ __forceinline__ void prefetch(uint32_t i) {
    if (R) rr = ldcg<PW>(R, i);
    else vraw = rhs.raw_row(i);
  }
  __device__ __forceinline__ void row(uint32_t i, T_<C> acc) {
    const T_<PW> s = cvt<PW>(acc);
    if (S) st<PW>(S, i, s);
    const T_<PW> r = R ? rr : rhs.apply(vraw);
    num = Ar<CD>::add(num, Ar<CD>::mul(cvt<CD>(r), cvt<CD>(s)));
    den = Ar<CD>::add(den, Ar<CD>::mul(cvt<CD>(s), cvt<CD>(s)));
  }
};

// update-call phase A: r_k = v - A z_k (materialised)
template <int PV, int PW, int C>
struct EpiResid {
  RhsView<PV, PW> rhs;
  void* R;
  T_<PV> vraw;
  __device__ __forceinline__ void prefetch(uint32_t i) { vraw = rhs.raw_row(i); }
  __device__ __forceinline__ void row(uint32_t i, T_<C> acc) {
    const T_<PW> s = cvt<PW>(acc);
    st<PW>(R, i, Ar<PW>::add(rhs.apply(vraw), Ar<PW>::neg(s)));
  }
};

// flags & 1 (row-block partition, P > 1): plain calls only, no bookkeeping -- update
// calls and the per-call bookkeeping run as k_rich_phase launches with the
// cross-rank exchanges between them
template <int PA, int PW, int PV, int IDX>
__global__ void __launch_bounds__(tile_threads(IDX), tile_minb(IDX)) k_richardson(CsrDev A, TilesDev T, const void* v, const double* v_scale,
                                                    void* out, uint64_t n, RichState* RS, Gate gate, int level,
                                                    unsigned long long* cnt, Sync sync, unsigned* bar_count,
                                                    unsigned* bar_gen, const IoSlot* io, uint64_t voff, int flags) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ double scratch[tile_scratch(IDX)];
  __shared__ double red[2];
  if (gate.closed()) return;
  if (io) {
    v = io->src;
    v_scale = io->src_scale;
    out = io->dst;
  }
  constexpr int C = pmax(PA, PW);    // SpMV accumulator (multiply(z, scratch))
  constexpr int CD = pmax(P32, PW);  // w' inner products: dot_at_least(.., P32)
  using AW = Ar<PW>;
  const int m = RS->m;
  const unsigned long long call = RS->calls[0];
  const bool update = RS->cycle != 0ull && (call % RS->cycle) == 0ull;
  if ((flags & 1) && update) return;
  RhsView<PV, PW> rhs{v, v_scale ? cvt<PV>(*v_scale) : Ar<PV>::one(), v_scale != nullptr, voff};
  const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;

  if (!update) {
    const T_<PW> w0 = cvt<PW>(RS->omegas[0]);
    if (m == 1) {
      for (uint64_t i = gtid; i < n; i += gstride) st<PW>(out, i, AW::add(AW::mul(w0, rhs.row(i)), AW::zero()));
    } else {
      // step 1 with z1 on the fly, then steps 2..m-1 ping-ponging through scratch.
      // Gather-bound matrices (config 5: the gather-bound tile shape, IDX bit 3, and
      // the windowed engine, bit 4), m = 2 on one rank: z1 is materialised at the
      // storage precision first, so the scattered gathers read 2-byte z1 (through L1,
      // or as the windowed engine's ring element with no per-entry transform left)
      // instead of the wider v (same z1 bits; the +0 is immaterial as an SpMV
      // operand, see GatherZ1)
      bool done = false;
      if constexpr (idx_gather(IDX) || (idx_wsell(IDX) && F3RG_WSELL_Z1)) {
        if (m == 2 && !(flags & 1) && voff == 0) {
          // eight independent loads per thread and round: one load per round left the pass
          // latency-bound (ncu: 117 us of the 911 us call for 120 MB of traffic)
          {
            constexpr int UN = 8;
            uint64_t i = gtid;
            for (; i + (UN - 1) * gstride < n; i += UN * gstride) {
              T_<PV> r[UN];
#pragma unroll
              for (int u = 0; u < UN; ++u) r[u] = rhs.raw_row(i + u * gstride);
#pragma unroll
              for (int u = 0; u < UN; ++u)
                st<PW>(RS->Za, i + u * gstride, AW::add(AW::mul(w0, rhs.apply(r[u])), AW::zero()));
            }
            for (; i < n; i += gstride) st<PW>(RS->Za, i, AW::add(AW::mul(w0, rhs.row(i)), AW::zero()));
          }
          grid_barrier(bar_count, bar_gen);
          GatherCA<PW, C> g{RS->Za};
          EpiStep<PV, PW, C, false> e{rhs, w0, cvt<PW>(RS->omegas[1]), RS->Za, out, {}, {}};
          spmv_tiles<PA, C, IDX, rich_chunk(IDX)>(A, T, g, e, smem);
          done = true;
        }
      }
      if (!done) {
        GatherZ1<PV, PW, C> g{rhs, w0};
        EpiStep<PV, PW, C, true> e{rhs, w0, cvt<PW>(RS->omegas[1]), nullptr, m == 2 ? out : RS->Za, {}, {}};
        spmv_tiles<PA, C, IDX, rich_chunk(IDX)>(A, T, g, e, smem);
      }
      for (int k = 2; k < m; ++k) {
        grid_barrier(bar_count, bar_gen);
        const void* zk = (k % 2 == 0) ? RS->Za : RS->Zb;
        void* zn = (k + 1 == m) ? out : ((k % 2 == 0) ? RS->Zb : RS->Za);
        GatherCG<PW, C> g{zk};
        EpiStep<PV, PW, C, false> e{rhs, w0, cvt<PW>(RS->omegas[k]), zk, zn, {}, {}};
        spmv_tiles<PA, C, IDX, rich_chunk(IDX)>(A, T, g, e, smem);
      }
    }
  } else {
    // generic adaptive-weight call: for each step k
    //   A (k>0): r = v - A z_k      B: s = A r, (r,s), (s,s) -> w'      C: z += w' r
    for (int k = 0; k < m; ++k) {
      if (k > 0) {
        GatherCG<PW, C> g{RS->Za};
        EpiResid<PV, PW, C> e{rhs, RS->R, {}};
        spmv_tiles<PA, C, IDX, rich_chunk(IDX)>(A, T, g, e, smem);
        grid_barrier(bar_count, bar_gen);
      }
      {
        EpiDotsRs<PV, PW, C, CD> e{rhs, k > 0 ? RS->R : nullptr, Ar<CD>::zero(), Ar<CD>::zero(), {}, {}};
        if (sync.seq) e.S = RS->Zb;
        if (k == 0) {
          GatherRhs<PV, PW, C> g{rhs};
          spmv_tiles<PA, C, IDX, rich_chunk(IDX)>(A, T, g, e, smem);
        } else {
          GatherCG<PW, C> g{RS->R};
          spmv_tiles<PA, C, IDX, rich_chunk(IDX)>(A, T, g, e, smem);
        }
        T_<CD> acc[2] = {e.num, e.den};
        block_sum<CD, 2>(acc, scratch);
        if (threadIdx.x == 0) {
          sync.partials[(size_t)blockIdx.x * kMaxPart + 0] = Ar<CD>::wide(acc[0]);
          sync.partials[(size_t)blockIdx.x * kMaxPart + 1] = Ar<CD>::wide(acc[1]);
        }
        grid_barrier(bar_count, bar_gen);
        // every CTA reduces the partials in the same fixed order -> identical w'
        reduce_partials<CD, 2>(sync.partials, gridDim.x, kMaxPart, red, scratch);
        if (sync.seq) {  // (r, s), (s, s) in index order (dot_at_least, src/richardson.cpp:32-33)
          grid_barrier(bar_count, bar_gen);  // every CTA is done with the partials
          if (blockIdx.x == 0) {
            seq_sums<CD>(n, 2, [&](uint64_t i, int q) {
              const T_<CD> sv = cvt<CD>(ldcg<PW>(RS->Zb, i));
              const T_<CD> rv = q ? sv : cvt<CD>(k > 0 ? ldcg<PW>(RS->R, i) : rhs.row(i));
              return Ar<CD>::mul(rv, sv);
            }, red);
            if (threadIdx.x == 0) sync.partials[0] = red[0], sync.partials[1] = red[1];
          }
          grid_barrier(bar_count, bar_gen);
          if (threadIdx.x == 0) red[0] = __ldcg(sync.partials), red[1] = __ldcg(sync.partials + 1);
          __syncthreads();
        }
      }
      const double num = red[0], den = red[1];
      double wk;
      int fresh;
      if (den == 0.0 || !isfinite(num) || !isfinite(den)) {
        wk = RS->omegas[k];
        fresh = 0;
      } else {
        wk = Ar<CD>::wide(Ar<CD>::div(cvt<CD>(num), cvt<CD>(den)));
        fresh = 1;
      }
      const T_<PW> wh = cvt<PW>(wk);
      void* zn = (k + 1 == m) ? out : RS->Za;
      for (uint64_t i = gtid; i < n; i += gstride) {
        const T_<PW> p = k > 0 ? ldcg<PW>(RS->R, i) : rhs.row(i);
        const T_<PW> zi = k > 0 ? ldcg<PW>(RS->Za, i) : AW::zero();
        st<PW>(zn, i, AW::add(AW::mul(wh, p), zi));
      }
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        RS->wused[k] = wk;
        RS->wupd[k] = fresh;
      }
      if (k + 1 < m) grid_barrier(bar_count, bar_gen);
      __syncthreads();
    }
  }
  if (flags & 1) return;  // bookkeeping: k_rich_phase PHASE_BOOK
  // bookkeeping once every CTA is done reading the state
  // update calls publish wused/wupd across CTAs (full fence); plain calls only count
  if (!(update ? last_block(sync.counter) : last_block_light(sync.counter))) return;
  if (threadIdx.x == 0) {
    if (update) {
      const double l = (double)(call / RS->cycle - 1ull);
      for (int k = 0; k < m; ++k) {
        if (RS->wupd[k]) {
          RS->omegas[k] = __ddiv_rn(__dadd_rn(__dmul_rn(l, RS->omegas[k]), RS->wused[k]), __dadd_rn(l, 1.0));
        } else {
          RS->calls[2] += 1ull;
        }
      }
      RS->calls[1] += 1ull;
    }
    RS->calls[0] = call + 1ull;
    cnt[CNT_INV + level] += 1ull;
    cnt[CNT_IT + level] += (unsigned long long)m;
    cnt[CNT_PRECOND] += (unsigned long long)m;
  }
}


// ---- row-block partition (P > 1): one Richardson call as a launch sequence ------
// The cooperative kernel's grid barriers become kernel boundaries, so the halo
// exchanges (z_k, r) and the cross-rank (r, s), (s, s) reductions can sit between
// them. The engine enqueues the sequence for EVERY call (the update decision
// call_count % c == 0 is made here on the device, exactly as in k_richardson);
// on plain calls every update phase returns at once and k_richardson (flags & 1)
// did the sweep. Same arithmetic, same per-element order as k_richardson.
enum { PH_RESID = 0, PH_DOTS = 1, PH_UPDATE = 2, PH_BOOK = 3 };

template <int PA, int PW, int PV, int IDX>
__global__ void __launch_bounds__(tile_threads(IDX), tile_minb(IDX)) k_rich_phase(CsrDev A, TilesDev T, int phase, int k, const void* v,
                                                    const double* v_scale, uint64_t off, void* out, uint64_t n,
                                                    RichState* RS, void* R, void* Za, Gate gate, int level,
                                                    unsigned long long* cnt, Sync sync, Dist dist) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ double scratch[tile_scratch(IDX)];
  __shared__ double tot[2];
  if (gate.closed()) return;
  constexpr int C = pmax(PA, PW);
  constexpr int CD = pmax(P32, PW);
  using AW = Ar<PW>;
  const int m = RS->m;
  const unsigned long long call = RS->calls[0];
  const bool update = RS->cycle != 0ull && (call % RS->cycle) == 0ull;
  RhsView<PV, PW> rhs{v, v_scale ? cvt<PV>(*v_scale) : Ar<PV>::one(), v_scale != nullptr, off};
  T_<PW>* Rown = static_cast<T_<PW>*>(R) + off;
  T_<PW>* Zown = static_cast<T_<PW>*>(Za) + off;
  if (phase == PH_RESID) {  // r = v - A z_k
    if (!update) return;
    GatherCG<PW, C> g{Za};
    EpiResid<PV, PW, C> e{rhs, Rown, {}};
    spmv_tiles<PA, C, IDX, rich_chunk(IDX)>(A, T, g, e, smem);
  } else if (phase == PH_DOTS) {  // s = A p, rank-local (r, s), (s, s)
    if (!update) return;
    EpiDotsRs<PV, PW, C, CD> e{rhs, k > 0 ? Rown : nullptr, Ar<CD>::zero(), Ar<CD>::zero(), {}, {}};
    if (k == 0) {
      GatherRhs<PV, PW, C> g{rhs};
      spmv_tiles<PA, C, IDX, rich_chunk(IDX)>(A, T, g, e, smem);
    } else {
      GatherCG<PW, C> g{R};
      spmv_tiles<PA, C, IDX, rich_chunk(IDX)>(A, T, g, e, smem);
    }
    T_<CD> acc[2] = {e.num, e.den};
    block_sum<CD, 2>(acc, scratch);
    if (threadIdx.x == 0) {
      sync.partials[(size_t)blockIdx.x * kMaxPart + 0] = Ar<CD>::wide(acc[0]);
      sync.partials[(size_t)blockIdx.x * kMaxPart + 1] = Ar<CD>::wide(acc[1]);
    }
    if (!last_block(sync.counter)) return;
    reduce_partials<CD, 2>(sync.partials, gridDim.x, kMaxPart, tot, scratch);
    publish_local(dist, 2, tot);
  } else if (phase == PH_UPDATE) {  // w' from the rank-ordered totals; z += w' p
    if (!update) return;
    combine_ranks<CD>(dist, 2, tot);
    const double num = tot[0], den = tot[1];
    double wk;
    int fresh;
    if (den == 0.0 || !isfinite(num) || !isfinite(den)) {
      wk = RS->omegas[k];
      fresh = 0;
    } else {
      wk = Ar<CD>::wide(Ar<CD>::div(cvt<CD>(num), cvt<CD>(den)));
      fresh = 1;
    }
    const T_<PW> wh = cvt<PW>(wk);
    void* zn = (k + 1 == m) ? out : static_cast<void*>(Zown);
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gstride) {
      const T_<PW> p = k > 0 ? ldcg<PW>(Rown, i) : rhs.row(i);
      const T_<PW> zi = k > 0 ? ldcg<PW>(Zown, i) : AW::zero();
      st<PW>(zn, i, AW::add(AW::mul(wh, p), zi));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      RS->wused[k] = wk;
      RS->wupd[k] = fresh;
    }
  } else if (blockIdx.x == 0 && threadIdx.x == 0) {  // PH_BOOK, one thread: as k_richardson's tail
    if (update) {
      const double l = (double)(call / RS->cycle - 1ull);
      for (int q = 0; q < m; ++q) {
        if (RS->wupd[q]) {
          RS->omegas[q] = __ddiv_rn(__dadd_rn(__dmul_rn(l, RS->omegas[q]), RS->wused[q]), __dadd_rn(l, 1.0));
        } else {
          RS->calls[2] += 1ull;
        }
      }
      RS->calls[1] += 1ull;
    }
    RS->calls[0] = call + 1ull;
    cnt[CNT_INV + level] += 1ull;
    cnt[CNT_IT + level] += (unsigned long long)m;
    cnt[CNT_PRECOND] += (unsigned long long)m;
  }
}


// ---- Richardson with a block-Jacobi ILU(0)/IC(0) primary preconditioner -----------
// One call of richardson_apply (src/richardson.cpp:10-54) with op.precondition = M
// (the PrimarySolver's apply, src/nesting.cpp:70-83) as a launch sequence:
//   RM_START  r = converted(v)                            (:19)
//   per step k:  [k > 0] RM_RESID  r = v - A z_k          (:24-27)
//                forward + backward sweep  p = M r         (:28, trsv.cuh); on plain
//                calls the backward sweep also does z_{k+1} = z_k + fl(w_k) p (:49)
//                RM_DOTS / RM_UPDATE  (update calls only, decided here on the device
//                from call_count % c): s = A p, w' = (r,s)/(s,s) at >= fp32, z += w' p
//   RM_BOOK   weight averaging and counters              (:42-52)
enum { RM_START = 0, RM_RESID = 1, RM_DOTS = 2, RM_UPDATE = 3, RM_BOOK = 4 };

template <int PA, int PW, int PV, int IDX>
__global__ void __launch_bounds__(tile_threads(IDX), tile_minb(IDX)) k_richm_phase(CsrDev A, TilesDev T, int phase, int k,
                                                                     const void* v, const double* v_scale,
                                                                     void* out, uint64_t n, RichState* RS, void* R,
                                                                     void* P, void* Za, Gate gate, int level,
                                                                     unsigned long long* cnt, Sync sync) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ double scratch[tile_scratch(IDX)];
  __shared__ double tot[2];
  if (gate.closed()) return;
  constexpr int C = pmax(PA, PW);
  constexpr int CD = pmax(P32, PW);
  using AW = Ar<PW>;
  const int m = RS->m;
  const unsigned long long call = RS->calls[0];
  const bool update = RS->cycle != 0ull && (call % RS->cycle) == 0ull;
  RhsView<PV, PW> rhs{v, v_scale ? cvt<PV>(*v_scale) : Ar<PV>::one(), v_scale != nullptr, 0};
  const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (phase == RM_START) {
    for (uint64_t i = gtid; i < n; i += gstride) st<PW>(R, i, rhs.row(i));
  } else if (phase == RM_RESID) {
    GatherCG<PW, C> g{Za};
    EpiResid<PV, PW, C> e{rhs, R, {}};
    spmv_tiles<PA, C, IDX, rich_chunk(IDX)>(A, T, g, e, smem);
  } else if (phase == RM_DOTS) {
    if (!update) return;
    GatherCG<PW, C> g{P};
    EpiDotsRs<PV, PW, C, CD> e{rhs, R, Ar<CD>::zero(), Ar<CD>::zero(), {}, {}};
    if (sync.seq) e.S = RS->Zb;
    spmv_tiles<PA, C, IDX, rich_chunk(IDX)>(A, T, g, e, smem);
    T_<CD> acc[2] = {e.num, e.den};
    block_sum<CD, 2>(acc, scratch);
    if (threadIdx.x == 0) {
      sync.partials[(size_t)blockIdx.x * kMaxPart + 0] = Ar<CD>::wide(acc[0]);
      sync.partials[(size_t)blockIdx.x * kMaxPart + 1] = Ar<CD>::wide(acc[1]);
    }
    if (!last_block(sync.counter)) return;
    if (sync.seq) {
      seq_sums<CD>(n, 2, [&](uint64_t i, int q) {
        const T_<CD> sv = cvt<CD>(ldcg<PW>(RS->Zb, i));
        return Ar<CD>::mul(q ? sv : cvt<CD>(ldcg<PW>(R, i)), sv);
      }, tot);
    } else {
      reduce_partials<CD, 2>(sync.partials, gridDim.x, kMaxPart, tot, scratch);
    }
    if (threadIdx.x == 0) {
      const double num = tot[0], den = tot[1];
      if (den == 0.0 || !isfinite(num) || !isfinite(den)) {
        RS->wused[k] = RS->omegas[k];
        RS->wupd[k] = 0;
      } else {
        RS->wused[k] = Ar<CD>::wide(Ar<CD>::div(cvt<CD>(num), cvt<CD>(den)));
        RS->wupd[k] = 1;
      }
    }
  } else if (phase == RM_UPDATE) {
    if (!update) return;
    const T_<PW> wh = cvt<PW>(RS->wused[k]);
    void* zn = (k + 1 == m) ? out : Za;
    for (uint64_t i = gtid; i < n; i += gstride) {
      const T_<PW> zi = k > 0 ? ld<PW>(Za, i) : AW::zero();
      st<PW>(zn, i, AW::add(AW::mul(wh, ld<PW>(P, i)), zi));
    }
  } else if (blockIdx.x == 0 && threadIdx.x == 0) {  // RM_BOOK
    if (update) {
      const double l = (double)(call / RS->cycle - 1ull);
      for (int q = 0; q < m; ++q) {
        if (RS->wupd[q]) {
          RS->omegas[q] = __ddiv_rn(__dadd_rn(__dmul_rn(l, RS->omegas[q]), RS->wused[q]), __dadd_rn(l, 1.0));
        } else {
          RS->calls[2] += 1ull;
        }
      }
      RS->calls[1] += 1ull;
    }
    RS->calls[0] = call + 1ull;
    cnt[CNT_INV + level] += 1ull;
    cnt[CNT_IT + level] += (unsigned long long)m;
    cnt[CNT_PRECOND] += (unsigned long long)m;
  }
}

}  // namespace f3rg
