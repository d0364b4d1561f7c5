// spmv.cuh -- CSR SpMV for sm_100a: row-tiles streamed into shared memory by
// the Tensor Memory Accelerator's 1-D bulk copies (cp.async.bulk + mbarrier,
// double-buffered, one issuing thread), one thread per row accumulating in the
// row's stored column order.
//
// Reference semantics (src/csr.cpp:23-37): y_i = sum_k val[k] * x[col[k]] with the
// accumulator at C = promote(TA, TX) starting at +0, each product and each sum
// rounded to C, sequential in stored order; result rounded to TY. Keeping one
// thread per row reproduces that order exactly, so every SpMV flavour is
// bit-identical to the reference; the bulk copies make the val/col streams fully
// coalesced (the naive one-thread-per-row load pattern would be L1-wavefront bound
// on B200).
//
// Tiles: contiguous row ranges with <= NT rows and <= TNNZ nonzeros (built on the
// host, tiles.cpp). A row longer than TNNZ gets a tile of its own and is summed
// straight from global memory by one thread (same order, slow, never hit by the
// benchmark matrices).
#pragma once

#include "common.cuh"
#include "state.hpp"

namespace f3rg {


template <int PA>
struct TileCfg {
#ifndef F3RG_TILE_SCALE
#define F3RG_TILE_SCALE 8
#endif
#ifndef F3RG_STAGES
#define F3RG_STAGES 2
#endif
  static constexpr int NT = 256;                                      // threads = max rows per tile
  static constexpr int SA = (int)sizeof(T_<PA>);
  // ~48 KB of (val, col) per stage at scale 8 (TNNZ multiples of 1024)
  static constexpr int TNNZ = (PA == P16 ? 1024 : PA == P32 ? 768 : 512) * F3RG_TILE_SCALE;
  static constexpr int VAL = 16 / SA;                                 // elements per 16 B
  static constexpr int STAGES = F3RG_STAGES;
  static constexpr int VAL_BYTES = ((TNNZ + 2 * VAL) * SA + 15) / 16 * 16;
  static constexpr int COL_BYTES = (TNNZ + 8) * 4;
  static constexpr int RP_BYTES = (NT + 12) * 4;
  static constexpr int STAGE_BYTES = VAL_BYTES + COL_BYTES + RP_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 64;
};

// N consecutive entries of one row: issue the N gathers, then accumulate in order.
template <int C, int N, class TA, class Gather>
__device__ __forceinline__ void row_chunk(T_<C>& acc, const TA* pv, const uint32_t* pc, const Gather& g) {
  typename Gather::Raw xs[N];
#pragma unroll
  for (int u = 0; u < N; ++u) xs[u] = g.load(pc[u]);
#pragma unroll
  for (int u = 0; u < N; ++u) acc = Ar<C>::add(acc, Ar<C>::mul(cvt<C>(pv[u]), g.value(xs[u])));
}

// Streams all tiles owned by this CTA (tile t = blockIdx.x + i*gridDim.x) through
// shared memory and calls epi.row(row, acc) for every row with acc at
// C = promote(PA, gather precision).
template <int PA, int C, class Gather, class Epi>
__device__ __forceinline__ void spmv_tiles(const CsrDev& A, const TilesDev& T, Gather& g, Epi& e, uint8_t* smem) {
  using Cfg = TileCfg<PA>;
  using TA = T_<PA>;
  constexpr int NT = Cfg::NT, ST = Cfg::STAGES, VAL = Cfg::VAL;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ST * Cfg::STAGE_BYTES);
  const TA* vals = static_cast<const TA*>(A.val[PA]);
  const uint32_t G = gridDim.x, tid = threadIdx.x;

  if (tid == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
  }
  __syncthreads();

  auto stage_ptr = [&](int s) { return smem + s * Cfg::STAGE_BYTES; };
  auto issue = [&](uint32_t t, int s) {
    const uint32_t r0 = T.r0[t], r1 = T.r0[t + 1], k0 = T.k0[t], k1 = T.k0[t + 1];
    uint64_t* bar = &bars[s];
    fence_proxy_async();
    if (k1 - k0 > (uint32_t)Cfg::TNNZ) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
      return;
    }
    const uint32_t k0v = k0 & ~(uint32_t)(VAL - 1), k1v = (k1 + VAL - 1) & ~(uint32_t)(VAL - 1);
    const uint32_t k0c = k0 & ~3u, k1c = (k1 + 3) & ~3u;
    const uint32_t r0a = r0 & ~3u, r1a = (r1 + 1 + 3) & ~3u;
    const uint32_t vb = (k1v - k0v) * Cfg::SA, cb = (k1c - k0c) * 4u, rb = (r1a - r0a) * 4u;
    mbar_arrive_expect_tx(bar, vb + cb + rb);
    uint8_t* sp = stage_ptr(s);
    if (vb) bulk_g2s(sp, vals + k0v, vb, bar);
    if (cb) bulk_g2s(sp + Cfg::VAL_BYTES, A.ci + k0c, cb, bar);
    bulk_g2s(sp + Cfg::VAL_BYTES + Cfg::COL_BYTES, A.rp + r0a, rb, bar);
  };

  if (tid == 0) {
    for (int s = 0; s < ST; ++s) {
      const uint32_t t = blockIdx.x + (uint32_t)s * G;
      if (t < T.ntiles) issue(t, s);
    }
  }
  // gathers are issued CHUNK at a time (independent loads in flight per thread)
  // before the sequential, order-preserving accumulation consumes them
#ifndef F3RG_CHUNK
#define F3RG_CHUNK 8
#endif
  constexpr int CHUNK = F3RG_CHUNK;
  uint32_t it = 0;
  for (uint32_t t = blockIdx.x; t < T.ntiles; t += G, ++it) {
    const int s = (int)(it % ST);
    const uint32_t par = (it / ST) & 1u;
    const uint32_t r0 = T.r0[t], r1 = T.r0[t + 1], k0 = T.k0[t], k1 = T.k0[t + 1];
    const bool longrow = k1 - k0 > (uint32_t)Cfg::TNNZ;
    const uint32_t row = r0 + tid;
    // row-local epilogue operands do not depend on the tile: start them now so
    // their latency hides behind the tile transfer and the row sum
    if (longrow ? tid == 0 : row < r1) e.prefetch(longrow ? r0 : row);
    mbar_wait(&bars[s], par);
    if (!longrow) {
      const uint8_t* sp = stage_ptr(s);
      const TA* sv = reinterpret_cast<const TA*>(sp);
      const uint32_t* sc = reinterpret_cast<const uint32_t*>(sp + Cfg::VAL_BYTES);
      const uint32_t* sr = reinterpret_cast<const uint32_t*>(sp + Cfg::VAL_BYTES + Cfg::COL_BYTES);
      const uint32_t k0v = k0 & ~(uint32_t)(VAL - 1), k0c = k0 & ~3u, r0a = r0 & ~3u;
      if (row < r1) {
        const uint32_t kb = sr[row - r0a], ke = sr[row + 1 - r0a];
        T_<C> acc = Ar<C>::zero();
        const TA* pv = sv + (kb - k0v);
        const uint32_t* pc = sc + (kb - k0c);
        const uint32_t len = ke - kb;
        // unpredicated chunks of 8 then 4 (raw loads first: all in flight, few live
        // registers), then a predicated tail of <= 3
        uint32_t q = 0;
        for (; q + CHUNK <= len; q += CHUNK) row_chunk<C, CHUNK>(acc, pv + q, pc + q, g);
        for (; q + 4 <= len; q += 4) row_chunk<C, 4>(acc, pv + q, pc + q, g);
        {
          typename Gather::Raw xs[3];
#pragma unroll
          for (int u = 0; u < 3; ++u)
            if (q + u < len) xs[u] = g.load(pc[q + u]);
#pragma unroll
          for (int u = 0; u < 3; ++u)
            if (q + u < len) acc = Ar<C>::add(acc, Ar<C>::mul(cvt<C>(pv[q + u]), g.value(xs[u])));
        }
        e.row(row, acc);
      }
    } else if (tid == 0) {
      T_<C> acc = Ar<C>::zero();
      for (uint32_t k = k0; k < k1; ++k)
        acc = Ar<C>::add(acc, Ar<C>::mul(cvt<C>(vals[k]), g.value(g.load(A.ci[k]))));
      e.row(r0, acc);
    }
    __syncthreads();
    if (tid == 0) {
      const uint32_t tn = t + (uint32_t)ST * G;
      if (tn < T.ntiles) issue(tn, s);
    }
  }
  // all issued tiles were consumed; retire the barriers so a later pass in the
  // same kernel can re-initialise them
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < ST; ++s) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&bars[s])) : "memory");
  (void)NT;
}

// ---- gathers ----------------------------------------------------------------------
// Two phases so a chunk of loads can be in flight with few live registers:
// load(c) issues the raw global load, value(raw) turns it into the operand at C.
// x[c] stored at PX, widened to C
template <int PX, int C>
struct GatherPlain {
  using Raw = T_<PX>;
  const void* x;
  __device__ __forceinline__ Raw load(uint32_t c) const { return ldg<PX>(x, c); }
  __device__ __forceinline__ T_<C> value(Raw r) const { return cvt<C>(r); }
};

// same, for a vector written earlier in the same (cooperative) kernel
template <int PX, int C>
struct GatherCG {
  using Raw = T_<PX>;
  const void* x;
  __device__ __forceinline__ Raw load(uint32_t c) const { return ldcg<PX>(x, c); }
  __device__ __forceinline__ T_<C> value(Raw r) const { return cvt<C>(r); }
};

// ---- epilogues --------------------------------------------------------------------
// Epilogue contract: prefetch(i) is called for the thread's row before the tile
// lands (issue independent loads there), row(i, acc) after its sum is complete.
template <int C, int PY>
struct EpiStore {
  void* y;
  __device__ __forceinline__ void prefetch(uint32_t) {}
  __device__ __forceinline__ void row(uint32_t i, T_<C> acc) { st<PY>(y, i, cvt<PY>(acc)); }
};

}  // namespace f3rg
