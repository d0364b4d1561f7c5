// trsv.cuh -- the triangular sweeps of the block-Jacobi ILU(0)/IC(0) apply
// (reference BlockJacobiIlu0::apply, src/ilu.cpp:187-263), bit-exact.
//
// Every row's value is the reference's sequential expression
//     t_i = ( init_i - f_1 * t_{c1} - f_2 * t_{c2} - ... ) [/ d_i]
// each product and difference rounded once at C = promote(factor, r) (C = binary16
// for the fp16-F3R default: the reference's Half rounds every op). Only the ORDER
// in which rows are computed changes: the host schedule (precond.cpp) groups rows
// by dependency level into warp slices.
//
// Synchronisation, per row: a row's value and the sweep's epoch travel in ONE word
// (binary16: epoch<<16 | bits; binary32: epoch<<32 | bits), stored with
// st.relaxed.gpu and polled with ld.relaxed.gpu -- a reader sees either a stale
// word (older epoch) or the final value, so a dependency costs one L2 round trip
// once it is written, with no fences or counters on the critical path (binary64
// rows use a value array plus a release/acquire flag). Epochs advance per launch.
// Polling every dependency of every waiting row would flood the L2 slices, so a
// warp first sleeps on a cheap hint -- the number of levels completed so far,
// kept by per-level slice counters off the critical path -- until its slice's
// level is F3RG_SWEEP_AHEAD (4) levels from the frontier, and only then polls
// its rows' dependency words.
//
// Progress: warp w owns slices w, w + W, w + 2W, ... in schedule order and a slice
// only waits for earlier slices. The earliest unfinished slice therefore never
// waits, so the sweep cannot deadlock provided every CTA eventually becomes
// resident (the grid is capped at the occupancy capacity, launch_precond.cu).
#pragma once

#include "common.cuh"
#include "levels.cuh"
#include "precond.hpp"

namespace f3rg {

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// row cells of one sweep at compute precision C; base = n rows x 12 bytes
template <int C> struct Cells;
template <> struct Cells<P16> {
  uint32_t* w;
  using Word = uint32_t;
  __device__ static Cells make(void* base, uint64_t) { return Cells{static_cast<uint32_t*>(base)}; }
  __device__ __forceinline__ Word fetch(uint32_t i) const { return ld_relaxed_u32(w + i); }
  __device__ __forceinline__ static bool ready(Word x, unsigned ep) { return (x >> 16) == (ep & 0xffffu); }
  __device__ __forceinline__ static __half value(Word x) { return __ushort_as_half((unsigned short)(x & 0xffffu)); }
  __device__ __forceinline__ __half read(uint32_t i) const { return value(__ldg(w + i)); }
  __device__ __forceinline__ void publish(uint32_t i, __half v, unsigned ep) const {
    st_relaxed_u32(w + i, ((ep & 0xffffu) << 16) | (uint32_t)__half_as_ushort(v));
  }
};
template <> struct Cells<P32> {
  unsigned long long* w;
  using Word = unsigned long long;
  __device__ static Cells make(void* base, uint64_t) { return Cells{static_cast<unsigned long long*>(base)}; }
  __device__ __forceinline__ Word fetch(uint32_t i) const { return ld_relaxed_u64(w + i); }
  __device__ __forceinline__ static bool ready(Word x, unsigned ep) { return (unsigned)(x >> 32) == ep; }
  __device__ __forceinline__ static float value(Word x) { return __uint_as_float((unsigned)(x & 0xffffffffull)); }
  __device__ __forceinline__ float read(uint32_t i) const { return value(__ldg(w + i)); }
  __device__ __forceinline__ void publish(uint32_t i, float v, unsigned ep) const {
    st_relaxed_u64(w + i, ((unsigned long long)ep << 32) | (unsigned long long)__float_as_uint(v));
  }
};
template <> struct Cells<P64> {
  double* v;
  uint32_t* f;
  struct Word {
    uint32_t f;
    double v;
  };
  __device__ static Cells make(void* base, uint64_t n) {
    return Cells{static_cast<double*>(base), reinterpret_cast<uint32_t*>(static_cast<double*>(base) + n)};
  }
  __device__ __forceinline__ Word fetch(uint32_t i) const {
    Word x;
    x.f = ld_acquire_u32(f + i);  // orders the value load after the flag
    x.v = ld_relaxed_f64(v + i);
    return x;
  }
  __device__ __forceinline__ static bool ready(const Word& x, unsigned ep) { return x.f == ep; }
  __device__ __forceinline__ static double value(const Word& x) { return x.v; }
  __device__ __forceinline__ double read(uint32_t i) const { return __ldg(v + i); }
  __device__ __forceinline__ void publish(uint32_t i, double x, unsigned ep) const {
    st_relaxed_f64(v + i, x);
    st_release_u32(f + i, ep);
  }
};

// epoch a launch publishes after `e0`: never 0 modulo 2^16, so neither zeroed cells
// nor a 16-bit wrap can look current (consecutive epochs differ by 1 or 2)
__device__ __forceinline__ unsigned next_epoch(unsigned e0) {
  unsigned e = e0 + 1u;
  if ((e & 0xffffu) == 0u) e += 1u;
  return e;
}

#ifndef F3RG_SWEEP_CHUNK
#define F3RG_SWEEP_CHUNK 16
#endif
constexpr int kSweepChunk = F3RG_SWEEP_CHUNK;  // entries in flight per lane (a 27-point row: one round)

// Process this warp's slices. init(row) -> T_<C> starting value; epi(row, value)
// after the row is published.
// nl: this launch's ordinal (launches completed + 1), the multiplier of the
// per-level slice counts in level_done (which accumulate over launches). It is a
// separate counter from the epoch tag, which skips multiples of 2^16.
template <int TF, int C, class Init, class Epi>
__device__ __forceinline__ void sweep_slices(const SweepDev& S, const Cells<C>& cells, unsigned* level_done,
                                             unsigned* frontier, unsigned ep, unsigned nl, const Init& init,
                                             Epi& epi) {
  using A = Ar<C>;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t s = gw; s < S.nslices; s += nw) {
    const uint32_t slot = s * 32u + lane;
    const uint32_t row = __ldg(S.rows + slot);
    const bool live = row != 0xffffffffu;
    const uint32_t cnt = live ? __ldg(S.cnt + slot) : 0u;
    const uint64_t base = (uint64_t)__ldg(S.soff + s) * 32u + lane;
    const uint32_t L = __ldg(S.lvl + s);
    // factor entries of the first round: independent of the wait, issued before it
    uint32_t col[kSweepChunk];
    T_<TF> f[kSweepChunk];
#pragma unroll
    for (int c = 0; c < kSweepChunk; ++c) {
      if ((uint32_t)c < cnt) {
        col[c] = __ldg(S.col + base + (uint64_t)c * 32u);
        f[c] = ldg<TF>(S.val, base + (uint64_t)c * 32u);
      }
    }
    T_<C> acc = live ? init(row) : A::zero();
    // far from the frontier: sleep instead of polling
    for (;;) {
      const unsigned fr = *(volatile unsigned*)frontier;
      if (fr + S.ahead >= L) break;
      __nanosleep(S.sleep_ns * (L - S.ahead - fr));
    }
    for (uint32_t e0 = 0; e0 < cnt; e0 += kSweepChunk) {
      if (e0 > 0) {
#pragma unroll
        for (int c = 0; c < kSweepChunk; ++c) {
          if (e0 + c < cnt) {
            col[c] = __ldg(S.col + base + (uint64_t)(e0 + c) * 32u);
            f[c] = ldg<TF>(S.val, base + (uint64_t)(e0 + c) * 32u);
          }
        }
      }
      typename Cells<C>::Word w[kSweepChunk];
#pragma unroll
      for (int c = 0; c < kSweepChunk; ++c)
        if (e0 + c < cnt) w[c] = cells.fetch(col[c]);
      // poll the stale dependencies until all are current. poll = 0: every stale
      // one each round (one round trip per round); poll = 1: spin on the last stale
      // one only (the most recently levelled in schedule order), then re-check
      for (;;) {
        int last = -1;
#pragma unroll
        for (int c = 0; c < kSweepChunk; ++c)
          if (e0 + c < cnt && !Cells<C>::ready(w[c], ep)) last = c;
        if (last < 0) break;
        if (S.poll == 1) {
#pragma unroll
          for (int c = 0; c < kSweepChunk; ++c)
            if (c == last) {
              do {
                w[c] = cells.fetch(col[c]);
              } while (!Cells<C>::ready(w[c], ep));
            }
        }
#pragma unroll
        for (int c = 0; c < kSweepChunk; ++c)
          if (e0 + c < cnt && !Cells<C>::ready(w[c], ep)) w[c] = cells.fetch(col[c]);
      }
#pragma unroll
      for (int c = 0; c < kSweepChunk; ++c)
        if (e0 + c < cnt) acc = A::sub(acc, A::mul(cvt<C>(f[c]), Cells<C>::value(w[c])));
    }
    if (live) {
      if (S.dg) acc = A::div(acc, cvt<C>(ldg<TF>(S.dg, slot)));
      cells.publish(row, acc, ep);
      epi(row, acc);
    }
    // frontier hint (off the critical path): the slice that completes level L
    // advances it
    __syncwarp();
    if (lane == 0) {
      const unsigned target = nl * __ldg(S.lvl_ns + L);  // mod 2^32, like the counter
      if (atomicAdd(level_done + L, 1u) + 1u == target) atomicMax(frontier, L + 1u);
    }
  }
}

// the last CTA of a sweep launch advances the direction's epoch and rewinds the
// frontier hint for the next launch
__device__ __forceinline__ void sweep_done(SweepCtl* ctl, unsigned ep, unsigned nl) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(&ctl->done, 1u) == gridDim.x - 1) {
      ctl->done = 0u;
      ctl->frontier = 0u;
      ctl->epoch = ep;
      ctl->launches = nl;
    }
  }
}

// fused Richardson update of the backward sweep (richardson.cpp:36,49 on a plain
// call): z_{k+1} = fl(fl(w_k * p) + z_k), z_0 = 0 (fill, :18)
struct RichEpi {
  const RichState* RS;  // null: no fused update
  int k;
  const void* zin;  // z_k (null: zero)
  void* zout;
};

// forward sweep: init = r_i (at PIN) widened to C
template <int TF, int PIN>
__global__ void __launch_bounds__(256) k_sweep_fwd(SweepDev S, const void* in, void* cells, unsigned* level_done,
                                                   SweepCtl* ctl, Gate gate) {
  pdl_wait();
  if (gate.closed()) return;
  constexpr int C = pmax(TF, PIN);
  const unsigned ep = next_epoch(*(volatile unsigned*)&ctl->epoch);
  const unsigned nl = *(volatile unsigned*)&ctl->launches + 1u;
  const Cells<C> cl = Cells<C>::make(cells, S.n);
  auto init = [&](uint32_t row) { return cvt<C>(ldg<PIN>(in, row)); };
  struct {
    __device__ __forceinline__ void operator()(uint32_t, T_<C>) const {}
  } epi;
  sweep_slices<TF, C>(S, cl, level_done, &ctl->frontier, ep, nl, init, epi);
  sweep_done(ctl, ep, nl);
}

// backward sweep: init = the forward value of the row; out z_i = value rounded to
// POUT; with RichEpi on a plain call also the fused z update
template <int TF, int C, int POUT>
__global__ void __launch_bounds__(256) k_sweep_bwd(SweepDev S, const void* fcells, void* cells, void* out,
                                                   unsigned* level_done, SweepCtl* ctl, Gate gate, RichEpi re) {
  pdl_wait();
  if (gate.closed()) return;
  const unsigned ep = next_epoch(*(volatile unsigned*)&ctl->epoch);
  const unsigned nl = *(volatile unsigned*)&ctl->launches + 1u;
  const Cells<C> fw = Cells<C>::make(const_cast<void*>(fcells), S.n);
  const Cells<C> cl = Cells<C>::make(cells, S.n);
  bool fuse = false;
  T_<POUT> wk = Ar<POUT>::zero();
  if (re.RS) {
    const unsigned long long call = re.RS->calls[0];
    const bool update = re.RS->cycle != 0ull && (call % re.RS->cycle) == 0ull;
    fuse = !update;
    wk = cvt<POUT>(re.RS->omegas[re.k]);
  }
  auto init = [&](uint32_t row) { return fw.read(row); };
  auto epi = [&](uint32_t row, T_<C> v) {
    const T_<POUT> p = cvt<POUT>(v);
    st<POUT>(out, row, p);
    if (fuse) {
      using AO = Ar<POUT>;
      const T_<POUT> zi = re.zin ? ld<POUT>(re.zin, row) : AO::zero();
      st<POUT>(re.zout, row, AO::add(AO::mul(wk, p), zi));
    }
  };
  sweep_slices<TF, C>(S, cl, level_done, &ctl->frontier, ep, nl, init, epi);
  sweep_done(ctl, ep, nl);
}

}  // namespace f3rg
