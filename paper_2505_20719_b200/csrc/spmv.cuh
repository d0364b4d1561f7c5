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
// Column stream, IDX = 0: u32 indices (4 B/nnz). IDX = 1 ("D16"): u16 in-row
// deltas + one u32 first column per row (2 B/nnz + 4 B/row), decoded by a running
// sum during the (already sequential) row walk -- same columns, same order, a
// third fewer bytes for an fp16 matrix. IDX = 2 ("P16", fp16 matrices only): the
// D16 delta and the fp16 value of an entry packed in one 32-bit word, so the row
// walk does one shared-memory load per entry instead of two (same bytes as D16).
//
// Tiles: contiguous row ranges with <= NT rows and <= TNNZ nonzeros (built on the
// host, spec.cpp build_tiles). Matrices with irregular row lengths are streamed
// from a row-sorted copy (rows ordered by length inside windows of sigma rows, as
// SELL-C-sigma does, so a tile's rows finish together); T.perm maps a tile row back
// to its matrix row for the epilogue. Each row's sum is unchanged. A row longer than TNNZ gets a tile of its own and is
// summed straight from global memory by one thread (same order, slow, never hit by
// the benchmark matrices).
#pragma once

#include <type_traits>

#include "common.cuh"
#include "state.hpp"
#include "wsell.cuh"
#include "wsell_pk.cuh"

#ifndef F3RG_TILE_MINB  // tile kernels: min CTAs per SM (register budget)
#define F3RG_TILE_MINB 3
#endif
#ifndef F3RG_D16_STAGES  // pipeline depth of fp16 D16 tiles
#define F3RG_D16_STAGES 2
#endif
#ifndef F3RG_CHUNK
#define F3RG_CHUNK 16
#endif
#ifndef F3RG_TNNZ16  // entries per fp16 tile (256 rows of a 27-point stencil)
#define F3RG_TNNZ16 7168
#endif
#ifndef F3RG_TNNZ32
#define F3RG_TNNZ32 6912
#endif
#ifndef F3RG_TNNZ64
#define F3RG_TNNZ64 4096
#endif
// short-row shape (IDX bit 2; matrices with <= 12 entries per row on
// average, the 7-point operators of configs 1/3/4): one gather chunk per row,
// fewer registers and smaller tiles so four CTAs share an SM
// (tools/variant_sweep.py m4_c8: config 4 1231 -> 836 ms, config 3 156 -> 132 ms)
#ifndef F3RG_SHORT_MINB
#define F3RG_SHORT_MINB 4
#endif
#ifndef F3RG_SHORT_CHUNK
#define F3RG_SHORT_CHUNK 8
#endif
#ifndef F3RG_SHORT_TNNZ16
#define F3RG_SHORT_TNNZ16 4352
#endif
#ifndef F3RG_SHORT_TNNZ32
#define F3RG_SHORT_TNNZ32 3200
#endif
#ifndef F3RG_SHORT_TNNZ64
#define F3RG_SHORT_TNNZ64 2048
#endif
// gather-bound shape (IDX bit 3; matrices whose rows needed sorting, config 5):
// the regular shape with half-size tiles, so the SM's 256 KB leaves more room to
// the L1 that serves the scattered x gathers (tools/spmv_probe.py on config 5,
// profiles/r01d_config5_tile_sweep.jsonl: fp64 SpMV 9157 -> 4161 us, fp16 1945 -> 1858 us
// at half size; fp32 5797 -> 2733 us at quarter size, its best)
#ifndef F3RG_GATHER_TNNZ16
#define F3RG_GATHER_TNNZ16 3584
#endif
#ifndef F3RG_GATHER_TNNZ32
#define F3RG_GATHER_TNNZ32 1728
#endif
#ifndef F3RG_GATHER_TNNZ64
#define F3RG_GATHER_TNNZ64 2048
#endif
#ifndef F3RG_P16_CHUNK  // P16 rows keep the chunk's values in registers too
#define F3RG_P16_CHUNK 9
#endif

namespace f3rg {

// IDX of the tiled kernels: bits 0-1 = column stream (0 u32, 1 D16, 2 P16),
// bit 2 = short-row shape, bit 3 = gather-bound shape, bit 4 = the windowed SELL
// engine (wsell.cuh: one 1024-thread CTA per SM, its own layout)
constexpr int idx_col(int idx) { return idx & 3; }
constexpr bool idx_short(int idx) { return (idx & 4) != 0; }
constexpr bool idx_gather(int idx) { return (idx & 8) != 0; }
constexpr bool idx_wsell(int idx) { return (idx & 16) != 0; }
constexpr int tile_minb(int idx) { return idx_wsell(idx) ? 1 : idx_short(idx) ? F3RG_SHORT_MINB : F3RG_TILE_MINB; }
constexpr int tile_threads(int idx) { return idx_wsell(idx) ? kWsThreads : 256; }
// block_sum scratch of a tile kernel: 8 values per warp
constexpr int tile_scratch(int idx) { return tile_threads(idx) / 32 * 8; }

template <int PA, int IDX_ = 0>
struct TileCfg {
  static constexpr int IDX = idx_col(IDX_);
  static constexpr bool SHORT = idx_short(IDX_);
  static constexpr bool GATHER = idx_gather(IDX_);
  static constexpr int NT = 256;  // threads = max rows per tile
  static constexpr int SA = (int)sizeof(T_<PA>);
  // Three CTAs per SM (F3RG_TILE_MINB; 2 stages of <= ~31 KB for fp16 D16/P16
  // tiles). The tile table is shared by all column formats, so TNNZ depends on PA
  // only: fp16 / fp32 tiles hold 256 rows of a 27-point stencil, fp64 ones 151.
  // Stage count and chunk size are from tools/variant_sweep.py on config 2.
  static constexpr int TNNZ =
      SHORT    ? (PA == P16 ? F3RG_SHORT_TNNZ16 : PA == P32 ? F3RG_SHORT_TNNZ32 : F3RG_SHORT_TNNZ64)
      : GATHER ? (PA == P16 ? F3RG_GATHER_TNNZ16 : PA == P32 ? F3RG_GATHER_TNNZ32 : F3RG_GATHER_TNNZ64)
               : (PA == P16 ? F3RG_TNNZ16 : PA == P32 ? F3RG_TNNZ32 : F3RG_TNNZ64);
  static constexpr int VAL = 16 / SA;  // value elements per 16 B
  static constexpr int CS = IDX == 1 ? 2 : 4;
  static constexpr int CAL = 16 / CS;  // column elements per 16 B
  static constexpr int STAGES = (PA == P16 && IDX >= 1) ? F3RG_D16_STAGES : 2;
  static constexpr int VAL_BYTES = IDX == 2 ? 0 : ((TNNZ + 2 * VAL) * SA + 15) / 16 * 16;
  static constexpr int COL_BYTES = ((TNNZ + 2 * CAL) * CS + 15) / 16 * 16;
  static constexpr int RP_BYTES = (NT + 12) * 4;
  static constexpr int FIRST_BYTES = IDX >= 1 ? (NT + 12) * 4 : 0;
  static constexpr int STAGE_BYTES = VAL_BYTES + COL_BYTES + RP_BYTES + FIRST_BYTES;
  static constexpr int SMEM_BYTES = idx_wsell(IDX_) ? kWsSmem : STAGES * STAGE_BYTES + 64;
};

// Streams all tiles owned by this CTA (tile t = blockIdx.x + i*gridDim.x) through
// shared memory and calls epi.row(row, acc) for every row with acc at
// C = promote(PA, gather precision).
// CH: gather chunk (0 = default: F3RG_CHUNK, or F3RG_P16_CHUNK for the P16 stream)
template <int PA, int C, int IDX_, int CH = 0, class Gather, class Epi>
__device__ __forceinline__ void spmv_row_tiles(const CsrDev& A, const TilesDev& T, Gather& g, Epi& e, uint8_t* smem) {
  g.set_policy(l2_policy(T.l2hint ? 2 : 0));  // the gathered vector
  using Cfg = TileCfg<PA, IDX_>;
  const uint64_t spol = l2_policy(T.l2hint ? 1 : 0);  // the matrix streams
  constexpr int IDX = Cfg::IDX;
  using TA = T_<PA>;
  using TC = typename std::conditional<IDX == 1, uint16_t, uint32_t>::type;
  constexpr int ST = Cfg::STAGES, VAL = Cfg::VAL, CAL = Cfg::CAL;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ST * Cfg::STAGE_BYTES);
  const TA* vals = static_cast<const TA*>(A.val[PA]);
  static_assert(IDX != 2 || PA == P16, "the packed P16 stream holds fp16 values");
  const TC* cols;
  if constexpr (IDX == 1) cols = A.dcol;
  else if constexpr (IDX == 2) cols = A.pk;
  else cols = A.ci;
  const uint32_t G = gridDim.x, tid = threadIdx.x;

  if (tid == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
  }
  __syncthreads();

  auto stage_ptr = [&](int s) { return smem + s * Cfg::STAGE_BYTES; };
  auto phys = [&](uint32_t t) { return T.reverse ? T.ntiles - 1u - t : t; };
  auto issue = [&](uint32_t tl, int s) {
    const uint32_t t = phys(tl);
    const uint32_t r0 = T.r0[t], r1 = T.r0[t + 1], k0 = T.k0[t], k1 = T.k0[t + 1];
    uint64_t* bar = &bars[s];
    fence_proxy_async();
    if (k1 - k0 > (uint32_t)Cfg::TNNZ) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
      return;
    }
    const uint32_t k0v = k0 & ~(uint32_t)(VAL - 1), k1v = (k1 + VAL - 1) & ~(uint32_t)(VAL - 1);
    const uint32_t k0c = k0 & ~(uint32_t)(CAL - 1), k1c = (k1 + CAL - 1) & ~(uint32_t)(CAL - 1);
    const uint32_t r0a = r0 & ~3u, r1a = (r1 + 1 + 3) & ~3u;
    const uint32_t vb = IDX == 2 ? 0u : (k1v - k0v) * Cfg::SA, cb = (k1c - k0c) * Cfg::CS,
                   rb = (r1a - r0a) * 4u;
    const uint32_t fb = IDX >= 1 ? (((r1 + 3) & ~3u) - r0a) * 4u : 0u;
    mbar_arrive_expect_tx(bar, vb + cb + rb + fb);
    uint8_t* sp = stage_ptr(s);
    if (vb) bulk_g2s_hint(sp, vals + k0v, vb, bar, spol);
    if (cb) bulk_g2s_hint(sp + Cfg::VAL_BYTES, cols + k0c, cb, bar, spol);
    bulk_g2s_hint(sp + Cfg::VAL_BYTES + Cfg::COL_BYTES, A.rp + r0a, rb, bar, spol);
    if (IDX && fb) bulk_g2s_hint(sp + Cfg::VAL_BYTES + Cfg::COL_BYTES + Cfg::RP_BYTES, A.first + r0a, fb, bar, spol);
  };

  if (tid == 0) {
    for (int s = 0; s < ST; ++s) {
      const uint32_t t = blockIdx.x + (uint32_t)s * G;
      if (t < T.ntiles) issue(t, s);
    }
  }
  // up to CHUNK gathers of a row are issued before the first is consumed (one
  // latency round per CHUNK entries); groups of 8 are unpredicated, only the last
  // partial group is predicated
  constexpr int CHUNK = CH ? CH : Cfg::SHORT ? F3RG_SHORT_CHUNK : IDX == 2 ? F3RG_P16_CHUNK : F3RG_CHUNK;
  // groups of GS unpredicated loads (8, or the whole chunk when it is not a multiple
  // of 8: a 27-point row is exactly 3 chunks of 9)
  constexpr int GS = CHUNK % 8 == 0 ? 8 : CHUNK, NG = CHUNK / GS;
  uint32_t it = 0;
  for (uint32_t t = blockIdx.x; t < T.ntiles; t += G, ++it) {
    const int s = (int)(it % ST);
    const uint32_t par = (it / ST) & 1u;
    const uint32_t tp = phys(t);
    const uint32_t r0 = T.r0[tp], r1 = T.r0[tp + 1], k0 = T.k0[tp], k1 = T.k0[tp + 1];
    const bool longrow = k1 - k0 > (uint32_t)Cfg::TNNZ;
    const uint32_t row = r0 + tid;
    // the epilogue's row: the matrix row itself, or perm[row] for sorted-row tiles
    const uint32_t erow = longrow ? (T.perm ? __ldg(T.perm + r0) : r0)
                                  : (T.perm && row < r1 ? __ldg(T.perm + row) : row);
    // row-local epilogue operands do not depend on the tile: start them now so
    // their latency hides behind the tile transfer and the row sum
    if (longrow ? tid == 0 : row < r1) e.prefetch(erow);
    mbar_wait(&bars[s], par);
    if (!longrow) {
      const uint8_t* sp = stage_ptr(s);
      const TA* sv = reinterpret_cast<const TA*>(sp);
      const TC* sc = reinterpret_cast<const TC*>(sp + Cfg::VAL_BYTES);
      const uint32_t* sr = reinterpret_cast<const uint32_t*>(sp + Cfg::VAL_BYTES + Cfg::COL_BYTES);
      const uint32_t k0v = k0 & ~(uint32_t)(VAL - 1), k0c = k0 & ~(uint32_t)(CAL - 1), r0a = r0 & ~3u;
      if (row < r1) {
        const uint32_t kb = sr[row - r0a], ke = sr[row + 1 - r0a];
        T_<C> acc = Ar<C>::zero();
        const TA* pv = sv + (kb - k0v);
        const TC* pc = sc + (kb - k0c);
        const uint32_t len = ke - kb;
        uint32_t col = 0;  // D16 / P16: running column
        if constexpr (IDX >= 1)
          col = reinterpret_cast<const uint32_t*>(sp + Cfg::VAL_BYTES + Cfg::COL_BYTES + Cfg::RP_BYTES)[row - r0a];
        // column of entry q (and, P16, its value out of the same word)
        auto fetch = [&](uint32_t q, TA& a) -> uint32_t {
          if constexpr (IDX == 2) {
            const uint32_t w = pc[q];
            if (q > 0) col += (w >> 16) + 1u;
            a = bits_as<TA>((unsigned short)(w & 0xffffu));
            return col;
          } else if constexpr (IDX == 1) {
            if (q > 0) col += pc[q] + 1u;
            return col;
          } else {
            return pc[q];
          }
        };
        for (uint32_t q = 0; q < len; q += CHUNK) {
          const uint32_t cnt = len - q < (uint32_t)CHUNK ? len - q : (uint32_t)CHUNK;
          typename Gather::Raw xs[CHUNK];
          TA av[CHUNK];  // P16 values (unused otherwise)
#pragma unroll
          for (int b = 0; b < NG; ++b) {
            if ((uint32_t)(GS * b + GS) <= cnt) {
#pragma unroll
              for (int u = 0; u < GS; ++u) xs[GS * b + u] = g.load(fetch(q + GS * b + u, av[GS * b + u]));
            } else {
#pragma unroll
              for (int u = 0; u < GS; ++u)
                if ((uint32_t)(GS * b + u) < cnt) xs[GS * b + u] = g.load(fetch(q + GS * b + u, av[GS * b + u]));
            }
          }
          auto aval = [&](int i) -> TA {
            if constexpr (IDX == 2) return av[i];
            else return pv[q + i];
          };
#pragma unroll
          for (int b = 0; b < NG; ++b) {
            if ((uint32_t)(GS * b + GS) <= cnt) {
#pragma unroll
              for (int u = 0; u < GS; ++u)
                acc = Ar<C>::add(acc, Ar<C>::mul(cvt<C>(aval(GS * b + u)), g.value(xs[GS * b + u])));
            } else {
#pragma unroll
              for (int u = 0; u < GS; ++u)
                if ((uint32_t)(GS * b + u) < cnt)
                  acc = Ar<C>::add(acc, Ar<C>::mul(cvt<C>(aval(GS * b + u)), g.value(xs[GS * b + u])));
            }
          }
        }
        e.row(erow, acc);
      }
    } else if (tid == 0) {
      T_<C> acc = Ar<C>::zero();
      uint32_t col = 0;
      if constexpr (IDX >= 1) col = A.first[r0];
      for (uint32_t k = k0; k < k1; ++k) {
        uint32_t c;
        TA a;
        if constexpr (IDX == 2) {
          const uint32_t w = A.pk[k];
          if (k > k0) col += (w >> 16) + 1u;
          c = col;
          a = bits_as<TA>((unsigned short)(w & 0xffffu));
        } else if constexpr (IDX == 1) {
          if (k > k0) col += A.dcol[k] + 1u;
          c = col;
          a = vals[k];
        } else {
          c = A.ci[k];
          a = vals[k];
        }
        acc = Ar<C>::add(acc, Ar<C>::mul(cvt<C>(a), g.value(g.load(c))));
      }
      e.row(erow, acc);
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
  pdl_trigger();
}

// The SpMV engine of a tile kernel: the row tiles above, or the windowed SELL
// engine (IDX bit 4, gather-bound matrices) -- same per-row sums either way.
template <int PA, int C, int IDX_, int CH = 0, class Gather, class Epi>
__device__ __forceinline__ void spmv_tiles(const CsrDev& A, const TilesDev& T, Gather& g, Epi& e, uint8_t* smem) {
  if constexpr (idx_wsell(IDX_)) {
    // fp16 matrix and a 2-byte ring (Richardson on z1, the L3 spmv_dots, the fp16 SpMV): the packed stream
    // ... and any matrix with a 4-byte ring (the L2 and L1 spmv_dots, fp16 A times fp32 x): code + value streams
    constexpr int RSZ = (int)sizeof(typename WsRing<Gather>::R);
    if constexpr ((PA == P16 && RSZ == 2) || RSZ == 4) wsell_pass_pk<PA, C>(A, T, g, e, smem);
    else wsell_pass<PA, C>(A, T, g, e, smem);
  } else {
    spmv_row_tiles<PA, C, IDX_, CH>(A, T, g, e, smem);
  }
}

// ---- gathers ----------------------------------------------------------------------
// Two phases so a chunk of loads can be in flight with few live registers:
// load(c) issues the raw global load, value(raw) turns it into the operand at C.
// x[c] stored at PX, widened to C
template <int PX, int C>
struct GatherPlain {
  using Raw = T_<PX>;
  const void* x;
  uint64_t pol = 0;  // L2 policy, set by the SpMV engine (set_policy)
  __device__ __forceinline__ void set_policy(uint64_t p) { pol = p; }
  __device__ __forceinline__ Raw load(uint32_t c) const { return ldg_hint<PX>(x, c, pol); }
  __device__ __forceinline__ T_<C> value(Raw r) const { return cvt<C>(r); }
};

// same, for a vector written earlier in the same (cooperative) kernel
template <int PX, int C>
struct GatherCG {
  using Raw = T_<PX>;
  const void* x;
  uint64_t pol = 0;  // L2 policy, set by the SpMV engine (set_policy)
  __device__ __forceinline__ void set_policy(uint64_t p) { pol = p; }
  __device__ __forceinline__ Raw load(uint32_t c) const { return ldcg_hint<PX>(x, c, pol); }
  __device__ __forceinline__ T_<C> value(Raw r) const { return cvt<C>(r); }
};

// same, L1-cached: a vector written earlier in the same kernel before a grid barrier
template <int PX, int C>
struct GatherCA {
  using Raw = T_<PX>;
  const void* x;
  uint64_t pol = 0;  // L2 policy, set by the SpMV engine (set_policy)
  __device__ __forceinline__ void set_policy(uint64_t p) { pol = p; }
  __device__ __forceinline__ Raw load(uint32_t c) const { return ldca_hint<PX>(x, c, pol); }
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
