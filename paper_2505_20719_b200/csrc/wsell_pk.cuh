// wsell_pk.cuh -- the windowed SELL pass over the PACKED stream (wsell_pk_layout.hpp):
// fp16 matrix, 2-byte ring elements (plain Richardson on materialised z1, the L3
// spmv_dots, the fp16 SpMV). Same engine as wsell.cuh -- one 1024-thread CTA per SM,
// the band of x in a shared-memory ring slid window by window, sorted 32-row slices
// claimed longest-first, row sums parked in shared memory for a coalesced epilogue --
// with 4 bytes per slot instead of 6: one 32-bit word holds the slot's 16-bit code and
// its fp16 value, and a far entry is an escape pair of two slots of its own row
// ([kPkEsc + column >> 16, +0], [column & 0xffff, value]), so there is no side list,
// no second stream and no dependent load. Each row is still summed by one thread in
// stored column order at C = promote(f16, TX); the padding and escape slots add +-0
// to an accumulator that is never -0, so the results are bit-identical to wsell.cuh,
// to the row tiles and to the reference (src/csr.cpp:23-37).
//
// The same pass serves every 4-byte ring (class 1, state.hpp pk_*: the L2 and L1 spmv_dots,
// and the fp16 matrix times an fp32 vector) with the codes and the values as two streams of
// 2 and 2 / 4 / 8 bytes per slot.
//
// Kernel windows lie on a global grid of kPkTW rows; a CTA owns whole sort windows and
// may start and end inside a window. Ring invariant for the window at rows
// [B, B + TW): the ring (kPkRing slots, slot = row mod kPkRing, the last one reserved
// for zero) holds x[B - W, B + 2 TW + W).
#pragma once

#include "wsell.cuh"

namespace f3rg {

constexpr int kPkSmem0 = kPkRing * 2 + kWsYBytes + 64, kPkSmem1 = pk_ring(1) * 4 + kWsYBytes + 64;
static_assert(kPkSmem0 <= kWsSmem && kPkSmem1 <= kWsSmem, "the packed passes run inside the windowed engine's shared memory");

template <int PA, int C, class G, class Epi>
__device__ __forceinline__ void wsell_pass_pk(const CsrDev& A, const TilesDev& T, G& g, Epi& e, uint8_t* smem) {
  using RT = WsRing<G>;
  using R = typename RT::R;
  using Raw = typename G::Raw;
  constexpr int RS = (int)sizeof(R);
  static_assert(RS == 2 || RS == 4, "packed layouts exist for 2- and 4-byte ring elements");
  constexpr int CL = RS == 2 ? 0 : 1;
  constexpr bool PACKED = CL == 0;  // one word per slot (code | fp16 value << 16); else a code and a value stream
  static_assert(!PACKED || PA == P16, "the packed word carries an fp16 value");
  constexpr int CS = (int)sizeof(T_<C>);
  constexpr int TW = pk_tw(CL), W = pk_w(CL);
  constexpr uint32_t RN = (uint32_t)pk_ring(CL), PADC = pk_pad(CL), ESC = pk_esc(CL);
  constexpr int kPkRingBytes = (int)RN * RS;
  constexpr int KW = TW / kWsSort;
  constexpr int PF = TW / kWsThreads;
  constexpr int U = PA == P64 ? 1 : F3RG_WS_U;
  constexpr bool YDBL = 2 * TW * CS <= kWsYBytes;
  static_assert(TW % kWsSort == 0 && PF >= 1 && TW * CS <= kWsYBytes, "window geometry");

  R* ring = reinterpret_cast<R*>(smem);
  T_<C>* ybuf = reinterpret_cast<T_<C>*>(smem + kPkRingBytes);
  unsigned* claim = reinterpret_cast<unsigned*>(smem + kPkRingBytes + kWsYBytes);
  WsPolicy<G>::set(g, l2_policy(T.l2hint ? 2 : 0));    // ring fills and far gathers: keep x in L2
  const uint64_t spol = l2_policy(T.l2hint ? 1 : 0);  // the matrix stream
  const int64_t n = (int64_t)A.n;
  const uint32_t tid = threadIdx.x, lane = tid & 31u;
  const uint32_t* __restrict__ cwin = PACKED ? T.pk_cwin : T.pk1_cwin;
  const uint32_t* __restrict__ soffp = PACKED ? T.pk_soff : T.pk1_soff;
  const uint32_t* __restrict__ rowp = PACKED ? T.pk_row : T.pk1_row;
  const uint32_t sw0 = cwin[blockIdx.x], sw1 = cwin[blockIdx.x + 1];
  const uint4* __restrict__ words = reinterpret_cast<const uint4*>(T.pk_words);    // PACKED
  const uint2* __restrict__ codes = reinterpret_cast<const uint2*>(T.pk1_code);    // else: 4 codes per lane and chunk
  (void)words;
  (void)codes;
  const int64_t row0 = (int64_t)sw0 * kWsSort;                                             // this CTA's rows
  const int64_t row1 = (int64_t)sw1 * kWsSort < n ? (int64_t)sw1 * kWsSort : n;

  __syncthreads();  // a previous pass in the same kernel is done with the shared memory
  if (tid < 2) claim[tid] = 0u;
  if (tid < (uint32_t)RS) smem[(size_t)PADC * RS + tid] = 0;  // the zero slot
  const int64_t Bfirst = row0 / TW * TW;
  if (sw0 < sw1) {  // ring for the first window: x[B - W, B + 2TW + W)
    int64_t i0 = Bfirst - W;
    if (i0 < 0) i0 = 0;
    int64_t i1 = Bfirst + 2 * TW + W;
    if (i1 > n) i1 = n;
    for (int64_t i = i0 + tid; i < i1; i += kWsThreads) {
      const uint32_t s = (uint32_t)i % RN;
      if (s < PADC) ring[s] = RT::put(g, g.load((uint32_t)i));
    }
  }
  __syncthreads();

  uint32_t it = 0;
  for (int64_t B = Bfirst; sw0 < sw1 && B < row1; B += TW, ++it) {
    // the CTA's sort windows inside this kernel window
    const uint32_t swa = (uint32_t)(B / kWsSort) > sw0 ? (uint32_t)(B / kWsSort) : sw0;
    const uint32_t swb = (uint32_t)((B + TW) / kWsSort) < sw1 ? (uint32_t)((B + TW) / kWsSort) : sw1;
    const uint32_t kw = swb - swa;
    (void)KW;
    // the ring block two windows ahead, into registers now, into the ring after the barrier
    const int64_t pb = B + 2 * TW + W;
    Raw pf[PF];
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int64_t i = pb + (int64_t)q * kWsThreads + tid;
      if (i < n) pf[q] = g.load((uint32_t)i);
    }
    T_<C>* yb = ybuf + (YDBL ? (it & 1u) * TW : 0u);
    const uint32_t nsl = kw * (uint32_t)kWsSlices;
    unsigned* cl = &claim[it & 1u];
    for (;;) {
      uint32_t j = 0;
      if (lane == 0) j = atomicAdd(cl, 1u);
      j = __shfl_sync(0xffffffffu, j, 0);
      if (j >= nsl) break;
      // claim order: slice rank j / kw of sort window j % kw -- descending length
      const uint32_t s = (swa + j % kw) * (uint32_t)kWsSlices + j / kw;
      const uint32_t e0 = __ldg(soffp + s), e1 = __ldg(soffp + s + 1);
      const uint32_t row = __ldg(rowp + (size_t)s * 32 + lane);
      const uint32_t nq = (e1 - e0) >> 7;  // chunks: 32 lanes x 4 slots
      const uint64_t qb = (uint64_t)(e0 >> 2) + lane;  // this lane's quad of chunk 0
      T_<C> acc = Ar<C>::zero();
      // one lane's quad of a chunk: 4 codes and 4 values (PACKED: one uint4 of words)
      struct Quad {
        uint4 w;          // PACKED: code | value << 16
        uint2 c;          // else: codes
        WsVals<PA> v;     // else: values
      };
      auto load_quad = [&](uint32_t q, Quad& x) {
        if constexpr (PACKED) {
          x.w = q < nq ? ws_ld16(words + qb + (uint64_t)q * 32, spol) : make_uint4(PADC, PADC, PADC, PADC);
        } else {
          if (q < nq) {
            x.c = ws_ld8(codes + qb + (uint64_t)q * 32, spol);
            x.v.load(T.pk1_val, qb + (uint64_t)q * 32, spol);
          } else {
            x.c = make_uint2(PADC | (PADC << 16), PADC | (PADC << 16));
            x.v.zero();
          }
        }
      };
      auto code_at = [&](const Quad& x, int k) -> uint32_t {
        if constexpr (PACKED) return quad_at(x.w, k) & 0xffffu;
        else return (k & 1) ? ((k < 2 ? x.c.x : x.c.y) >> 16) : ((k < 2 ? x.c.x : x.c.y) & 0xffffu);
      };
      auto val_at = [&](const Quad& x, int k) {
        if constexpr (PACKED) return __ushort_as_half((unsigned short)(quad_at(x.w, k) >> 16));
        else return x.v.at(k);
      };
      Quad cc[U], cn[U];
#pragma unroll
      for (int u = 0; u < U; ++u) load_quad((uint32_t)u, cc[u]);
      for (uint32_t q0 = 0; q0 < nq; q0 += U) {
#pragma unroll
        for (int u = 0; u < U; ++u) load_quad(q0 + U + u, cn[u]);  // next step's stream, in flight during this one
        R xr[4 * U];
        Raw xf[4 * U];
        bool farf[4 * U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          bool low = false;     // this slot is the low half of a far column
          uint32_t hi = 0;      // (escape code - ESC) << 16 of the slot before
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t code = code_at(cc[u], k);
            const uint32_t idx = code < PADC ? code : PADC;  // escape and low-half slots read zero
            farf[4 * u + k] = low;
            xr[4 * u + k] = ring[idx];
            xf[4 * u + k] = low ? g.load(hi | code) : Raw{};
            const bool esc = !low && code >= ESC;
            hi = (code - ESC) << 16;
            low = esc;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const T_<C> xv = !farf[4 * u + k] ? RT::get(g, xr[4 * u + k]) : RT::get(g, RT::put(g, xf[4 * u + k]));
            acc = Ar<C>::add(acc, Ar<C>::mul(cvt<C>(val_at(cc[u], k)), xv));
          }
#pragma unroll
        for (int u = 0; u < U; ++u) cc[u] = cn[u];
      }
      if (row != kWsPad) yb[(uint32_t)((int64_t)row - B)] = acc;
    }
    __syncthreads();  // every row sum of the window is in yb; the band's bottom block is free
    if (tid == 0) claim[it & 1u] = 0u;  // reused two windows on, after the next barrier
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int64_t i = pb + (int64_t)q * kWsThreads + tid;
      const uint32_t s = (uint32_t)i % RN;
      if (i < n && s < PADC) ring[s] = RT::put(g, pf[q]);
    }
    const int64_t ra = B > row0 ? B : row0, rb = B + TW < row1 ? B + TW : row1;
    for (int64_t i = ra + tid; i < rb; i += kWsThreads) {
      e.prefetch((uint32_t)i);
      e.row((uint32_t)i, yb[(uint32_t)(i - B)]);
    }
    if constexpr (!YDBL) __syncthreads();  // the one row-sum buffer is free again
  }
  pdl_trigger();
}

}  // namespace f3rg
