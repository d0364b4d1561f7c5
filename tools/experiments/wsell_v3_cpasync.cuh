// wsell.cuh -- windowed SELL-32 SpMV engine for gather-bound matrices (config 5:
// n = 2e7 unstructured rows whose columns scatter around the diagonal with a
// 5,000-row standard deviation, plus 5 % uniform long-range entries).
//
// Why: with one thread per row and the gathered vector read through L1 (the tile
// engine, spmv.cuh), every entry of such a matrix is its own 128-byte line request;
// the L1 tag stage serves about one line per clock per SM, which is exactly the
// 2 ms the config-5 fp16 pass took (4.1 M lines per SM at 1.965 GHz). Here the
// gathered vector lives in shared memory instead: each persistent CTA (one per SM,
// kWsWarps warps) owns a contiguous run of rows and keeps the band of x those rows
// can touch in a ring, slid forward window by window with plain loads issued one
// window ahead. The first version of this engine tested every entry against the
// band on the device and spent 47 instructions per entry (issue-bound, ncu
// profiles/r02q_*); now everything per entry is decided on the host
// (wsell_layout.hpp):
//  * an entry is a 16-bit SLOT into one shared-memory array of ring elements: the
//    ring itself (slot = column mod RN), the executing warp's far-value scratch (the
//    long-range 5 %: the warp gathers a segment's far values from L2 one segment
//    ahead and parks them there), or the slot that holds zero (padding). The gather
//    is one LDS whatever the entry is, and the column stream is 2 bytes per entry;
//  * the slices (32 rows sorted by length, chunk-major) of every kernel window are
//    assigned to the warps on the host, longest first, and each warp walks ONE flat
//    list of step records (1-2 chunks of 32 lanes x 4 entries each) whose flags say
//    where a slice starts and ends, where a far segment starts and where the kernel
//    window ends. The stream loads run two steps ahead of the arithmetic, across
//    slices and windows.
// Each row is still summed by one thread in stored column order at
// C = promote(TA, TX), each product and sum rounded to C (src/csr.cpp:23-37), so
// results are bit-identical to the tile engine and to the reference.
//
// Per kernel window of TW rows: the warps write each row's sum into a shared-memory
// buffer at the row's position, then, after one CTA barrier, the epilogue runs over
// the window's rows in natural order (coalesced row-local operands). Ring invariant
// for the window at rows [B, B+TW): the ring holds x[B-W, B+2TW+W) (RN = 2TW + 2W
// elements): the gathers' band [B-W, B+TW+W) plus the top block of the next
// window's band; the block after that is loaded into registers at the window's
// start and stored after its barrier into the slots the window just freed.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "state.hpp"

namespace f3rg {

constexpr int kWsThreads = kWsWarps * 32;
constexpr int kWsSort = (int)kWsSortRows;  // rows per sort window (layout unit)
#ifndef F3RG_WS_STAGES  // stream stages per warp at most (what fits is used)
#define F3RG_WS_STAGES 4
#endif
// dynamic shared memory of a pass: everything the SM has, minus the kernels' static
// scratch (<= 2 KB)
constexpr int kWsSmem = 232448 - 2048;
constexpr int ws_slot_bytes(int cl) { return (ws_slots(cl) * (2 << cl) + 127) / 128 * 128; }
// per-warp staging: per stage the step's slots (2 chunks x 256 B), values, row indices
// (128 B) and the far columns of the next segment (kWsFarSlots x 4 B); two record batches
constexpr int kWsRecBytes = 2 * 32 * 8;
constexpr int ws_stage_bytes(int sa) { return 512 + 2 * 128 * sa + 128 + kWsFarSlots * 4; }
// geometry of a pass with ring class cl, value size sa and accumulator size cs: two
// row-sum buffers when at least one stage still fits beside them, else one (and a
// second barrier per window); as many stages as fit, at most F3RG_WS_STAGES
constexpr int ws_perwarp(int cl, int cs, bool ydbl) {
  return (kWsSmem - ws_slot_bytes(cl) - (ydbl ? 2 : 1) * ws_tw(cl) * cs) / kWsWarps / 128 * 128;
}
constexpr int ws_stages_fit(int cl, int sa, int cs, bool ydbl) {
  return (ws_perwarp(cl, cs, ydbl) - kWsRecBytes) / ws_stage_bytes(sa);
}
constexpr bool ws_ydbl(int cl, int sa, int cs) { return ws_stages_fit(cl, sa, cs, true) >= 1; }
constexpr int ws_stages(int cl, int sa, int cs) {
  return ws_stages_fit(cl, sa, cs, ws_ydbl(cl, sa, cs)) > F3RG_WS_STAGES ? F3RG_WS_STAGES
                                                                          : ws_stages_fit(cl, sa, cs, ws_ydbl(cl, sa, cs));
}

// What the ring stores for a gather: its raw load, or (gathers with a per-element
// transform, e.g. Richardson's z1 = w0 * v) the transformed value, so the transform
// runs once per ring element instead of once per gathered entry.
template <class G, class = void>
struct WsRing {
  using R = typename G::Raw;
  __device__ __forceinline__ static R put(const G&, typename G::Raw r) { return r; }
  __device__ __forceinline__ static auto get(const G& g, R r) { return g.value(r); }
};
template <class G>
struct WsRing<G, std::void_t<typename G::RingT>> {
  using R = typename G::RingT;
  __device__ __forceinline__ static R put(const G& g, typename G::Raw r) { return g.ring_put(r); }
  __device__ __forceinline__ static auto get(const G& g, R r) { return g.ring_get(r); }
};

// L2 policy of the engine's vector loads (ring fills, far gathers): the gather's own
// set_policy, or set_ring_policy where the tile engine's gathers take none
template <class G, class = void>
struct WsPolicy {
  __device__ __forceinline__ static void set(G& g, uint64_t p) { g.set_policy(p); }
};
template <class G>
struct WsPolicy<G, std::void_t<decltype(std::declval<G&>().set_ring_policy(0ull))>> {
  __device__ __forceinline__ static void set(G& g, uint64_t p) { g.set_ring_policy(p); }
};

template <int K, int N, class F>
__device__ __forceinline__ void ws_static_for(F&& f) {
  if constexpr (K < N) {
    f(std::integral_constant<int, K>{});
    ws_static_for<K + 1, N>(f);
  }
}

// asynchronous global -> shared copies (LDGSTS): they hold no register and no
// scoreboard, and complete in commit-group order, so a warp can keep several steps of
// its stream in flight -- ptxas puts all of a loop's global loads on ONE scoreboard,
// which serialises any register-prefetch pipeline (profiles/r02s_*)
template <int BYTES>
__device__ __forceinline__ void ws_cp(uint32_t dst, const void* src, uint64_t pol) {
  static_assert(BYTES == 4 || BYTES == 8 || BYTES == 16, "cp.async size");
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], %2, %3;" ::"r"(dst), "l"(src), "n"(BYTES), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void ws_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void ws_cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// one lane's 4 values of a chunk, out of the staged copy
template <int PA>
struct WsVals;
template <>
struct WsVals<P16> {
  uint2 q;
  __device__ __forceinline__ void load(const uint8_t* chunk, uint32_t lane) {
    q = reinterpret_cast<const uint2*>(chunk)[lane];
  }
  __device__ __forceinline__ __half at(int e) const {
    const uint32_t w = e < 2 ? q.x : q.y;
    return __ushort_as_half((unsigned short)((e & 1) ? (w >> 16) : (w & 0xffffu)));
  }
};
template <>
struct WsVals<P32> {
  uint4 q;
  __device__ __forceinline__ void load(const uint8_t* chunk, uint32_t lane) {
    q = reinterpret_cast<const uint4*>(chunk)[lane];
  }
  __device__ __forceinline__ float at(int e) const {
    return __uint_as_float(e == 0 ? q.x : e == 1 ? q.y : e == 2 ? q.z : q.w);
  }
};
template <>
struct WsVals<P64> {
  uint4 a, b;
  __device__ __forceinline__ void load(const uint8_t* chunk, uint32_t lane) {
    a = reinterpret_cast<const uint4*>(chunk)[2 * lane];
    b = reinterpret_cast<const uint4*>(chunk)[2 * lane + 1];
  }
  __device__ __forceinline__ double at(int e) const {
    const uint4& h = e < 2 ? a : b;
    return (e & 1) ? __hiloint2double((int)h.w, (int)h.z) : __hiloint2double((int)h.y, (int)h.x);
  }
};

// Streams this CTA's windows; calls e.prefetch(i); e.row(i, acc) for every row i in
// natural order, acc at C. Launch: gridDim.x == T.ws_G, blockDim.x == kWsThreads,
// kWsSmem bytes of dynamic shared memory. Square matrices on one rank only (x has
// n elements).
template <int PA, int C, class G, class Epi>
__device__ __forceinline__ void wsell_pass(const CsrDev& A, const TilesDev& T, G& g, Epi& e, uint8_t* smem) {
  using RT = WsRing<G>;
  using R = typename RT::R;
  using Raw = typename G::Raw;
  constexpr int RS = (int)sizeof(R);
  static_assert(RS == 2 || RS == 4 || RS == 8, "ring element size");
  constexpr int CL = RS == 2 ? 0 : RS == 4 ? 1 : 2;  // ring class
  constexpr uint32_t RN = (uint32_t)ws_rn(CL);
  constexpr int TW = ws_tw(CL), W = ws_w(CL);
  constexpr int CS = (int)sizeof(T_<C>), SA = (int)sizeof(T_<PA>);
  constexpr bool YDBL = ws_ydbl(CL, SA, CS);  // two row-sum buffers, or one and a second barrier per window
  constexpr int S = ws_stages(CL, SA, CS);    // stream stages in flight per warp
  static_assert(S >= 1, "no room for a stream stage");
  constexpr int PERWARP = ws_perwarp(CL, CS, YDBL), STAGEB = ws_stage_bytes(SA);
  constexpr int VQ = 4 * SA;                  // bytes of one lane's value quad
  constexpr int OFF_VAL = 512, OFF_ROW = 512 + 64 * VQ, OFF_FAR = OFF_ROW + 128;
  constexpr int PF = (TW + kWsThreads - 1) / kWsThreads;  // ring elements each thread carries one window ahead
  constexpr int FK = kWsFarSlots / 32;  // far values per lane and segment
  static_assert(TW % kWsSort == 0 && W > 0 && PF >= 1, "window geometry");

  R* ringR = reinterpret_cast<R*>(smem);
  T_<C>* ybuf = reinterpret_cast<T_<C>*>(smem + ws_slot_bytes(CL));
  WsPolicy<G>::set(g, l2_policy(T.l2hint ? 2 : 0));    // ring fills and far gathers: keep x in L2
  const uint64_t spol = l2_policy(T.l2hint ? 1 : 0);  // the matrix stream
  const int64_t n = (int64_t)A.n;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t sw0 = T.ws_cwin[blockIdx.x], sw1 = T.ws_cwin[blockIdx.x + 1];
  const uint4 hdr = __ldg(T.ws_hdr[CL] + (size_t)blockIdx.x * kWsWarps + warp);
  const uint2* __restrict__ recp = T.ws_rec[CL] + hdr.x;
  const uint32_t nrec = hdr.y;
  const uint32_t* __restrict__ farp = T.ws_far[CL];
  const uint2* __restrict__ slotq = reinterpret_cast<const uint2*>(T.ws_slot[CL]);
  const uint8_t* __restrict__ vals = static_cast<const uint8_t*>(T.ws_val);
  R* scr = ringR + ws_far0(CL) + warp * kWsFarSlots;
  uint8_t* wst = smem + ws_slot_bytes(CL) + (YDBL ? 2 : 1) * TW * CS + warp * PERWARP;  // this warp's staging
  uint8_t* recb = wst + S * STAGEB;                                                      // its two record batches
  const uint32_t wst_s = smem_u32(wst), recb_s = smem_u32(recb);

  __syncthreads();  // a previous pass in the same kernel is done with the shared memory
  if (tid < (uint32_t)RS) smem[(size_t)ws_zero(CL) * RS + tid] = 0;  // the zero slot
  int64_t B = (int64_t)sw0 * kWsSort;  // first row of the current kernel window
  if (sw0 < sw1) {  // ring for the first window: x[B-W, B+2TW+W)
    int64_t i0 = B - W;
    if (i0 < 0) i0 = 0;
    int64_t i1 = B + 2 * TW + W;
    if (i1 > n) i1 = n;
    for (int64_t i = i0 + tid; i < i1; i += kWsThreads) ringR[(uint32_t)i % RN] = RT::put(g, g.load((uint32_t)i));
  }
  const int64_t cta_end = (int64_t)sw1 * kWsSort < n ? (int64_t)sw1 * kWsSort : n;

  // record batches 0 and 1 (lane l copies record l of the batch; read back by broadcast)
  if (lane < nrec) ws_cp<8>(recb_s + lane * 8u, recp + lane, spol);
  if (32u + lane < nrec) ws_cp<8>(recb_s + 256u + lane * 8u, recp + 32u + lane, spol);
  ws_cp_commit();

  // far pipeline: a segment's values are gathered (register loads) while the segment
  // before it runs, from the columns that arrived with that segment's first step.
  // Prime it with segment 0.
  uint32_t nf_cur = hdr.w, nf_nxt = 0u;
  uint32_t foff = hdr.z + ((hdr.w + 3u) & ~3u);  // far columns of the next segment to stage
  Raw farv[FK];
  {
    uint32_t farc[FK];
#pragma unroll
    for (int k = 0; k < FK; ++k)
      if (k * 32 + lane < nf_cur) farc[k] = __ldg(farp + hdr.z + k * 32 + lane);
#pragma unroll
    for (int k = 0; k < FK; ++k)
      if (k * 32 + lane < nf_cur) farv[k] = g.load(farc[k]);
  }

  // the ring block two windows ahead: into registers now, into the ring after the barrier
  Raw pf[PF];
  auto ring_prefetch = [&]() {
    const int64_t pb = B + 2 * TW + W;
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int64_t i = pb + (int64_t)q * kWsThreads + tid;
      if (q * kWsThreads + (int)tid < TW && i < n) pf[q] = g.load((uint32_t)i);
    }
  };
  if (sw0 < sw1) ring_prefetch();
  ws_cp_wait<0>();
  __syncthreads();  // ring, zero slot and the first records are in place

  uint32_t it = 0;
  T_<C>* yb = ybuf;
  T_<C> acc = Ar<C>::zero();
  auto window_end = [&]() {
    __syncthreads();  // every row sum of the window is in yb; the band's bottom block is free
    const int64_t pb = B + 2 * TW + W;
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int64_t i = pb + (int64_t)q * kWsThreads + tid;
      if (q * kWsThreads + (int)tid < TW && i < n) ringR[(uint32_t)i % RN] = RT::put(g, pf[q]);
    }
    const int64_t rend = B + TW < cta_end ? B + TW : cta_end;
    for (int64_t i = B + tid; i < rend; i += kWsThreads) {
      e.prefetch((uint32_t)i);
      e.row((uint32_t)i, yb[(uint32_t)(i - B)]);
    }
    if constexpr (!YDBL) __syncthreads();
    B += TW;
    ++it;
    if constexpr (YDBL) yb = ybuf + (it & 1u) * TW;
    ring_prefetch();
  };

  // per stage: the step's flags and second record word (registers; the loop below is
  // unrolled over the stages)
  uint32_t sf[S], sy[S];
  // issue step i's copies into stage st (one commit group per call, empty past the end)
  auto fetch = [&](uint32_t i, auto ST) {
    constexpr int st = decltype(ST)::value;
    sf[st] = 0u;
    if (i < nrec) {
      const uint32_t b = i & 31u, bat = i >> 5;
      if (b == 0u) {  // batch bat is in place (waited for by an earlier step); stage the one after it
        __syncwarp();
        if (bat > 0u && i + 32u + lane < nrec)
          ws_cp<8>(recb_s + ((bat + 1u) & 1u) * 256u + lane * 8u, recp + i + 32u + lane, spol);
      }
      const uint2 r = *reinterpret_cast<const uint2*>(recb + (bat & 1u) * 256u + b * 8u);
      const uint32_t f = r.x >> 24;
      sf[st] = f;
      sy[st] = r.y;
      const uint64_t q = (uint64_t)(r.x & 0xffffffu) * 32u + lane;
      const uint32_t sb = wst_s + (uint32_t)st * STAGEB;
      if (f & kWsQ1) {
        ws_cp<8>(sb + lane * 8u, slotq + q, spol);
        if constexpr (VQ == 8) ws_cp<8>(sb + OFF_VAL + lane * 8u, vals + q * 8u, spol);
        else if constexpr (VQ == 16) ws_cp<16>(sb + OFF_VAL + lane * 16u, vals + q * 16u, spol);
        else {
          ws_cp<16>(sb + OFF_VAL + lane * 32u, vals + q * 32u, spol);
          ws_cp<16>(sb + OFF_VAL + lane * 32u + 16u, vals + q * 32u + 16u, spol);
        }
      }
      if (f & kWsQ2) {
        ws_cp<8>(sb + 256u + lane * 8u, slotq + q + 32u, spol);
        if constexpr (VQ == 8) ws_cp<8>(sb + OFF_VAL + 32 * VQ + lane * 8u, vals + (q + 32u) * 8u, spol);
        else if constexpr (VQ == 16) ws_cp<16>(sb + OFF_VAL + 32 * VQ + lane * 16u, vals + (q + 32u) * 16u, spol);
        else {
          ws_cp<16>(sb + OFF_VAL + 32 * VQ + lane * 32u, vals + (q + 32u) * 32u, spol);
          ws_cp<16>(sb + OFF_VAL + 32 * VQ + lane * 32u + 16u, vals + (q + 32u) * 32u + 16u, spol);
        }
      }
      if (f & kWsLast) ws_cp<4>(sb + OFF_ROW + lane * 4u, T.ws_row + (size_t)(r.y & 0xffffffu) * 32u + lane, spol);
      if (f & kWsSeg) {  // the far columns of the segment after the one this step opens
        if (lane < (uint32_t)kWsFarSlots / 4u) ws_cp<16>(sb + OFF_FAR + lane * 16u, farp + foff + lane * 4u, spol);
        foff += ((r.y >> 24) + 3u) & ~3u;
      }
    }
    ws_cp_commit();
  };
  auto term = [&](const WsVals<PA>& v, int k, R x) {
    acc = Ar<C>::add(acc, Ar<C>::mul(cvt<C>(v.at(k)), RT::get(g, x)));
  };
  auto consume = [&](auto ST) {
    constexpr int st = decltype(ST)::value;
    ws_cp_wait<S - 1>();  // this step's group (and every older one) has landed
    __syncwarp();
    const uint32_t f = sf[st];
    const uint8_t* sb = wst + st * STAGEB;
    if (f & kWsSeg) {
      __syncwarp();  // every lane is done reading the previous segment's values
#pragma unroll
      for (int k = 0; k < FK; ++k)
        if (k * 32 + lane < nf_cur) scr[k * 32 + lane] = RT::put(g, farv[k]);
      __syncwarp();
      nf_nxt = sy[st] >> 24;
#pragma unroll
      for (int k = 0; k < FK; ++k)
        if (k * 32 + lane < nf_nxt) farv[k] = g.load(reinterpret_cast<const uint32_t*>(sb + OFF_FAR)[k * 32 + lane]);
      nf_cur = nf_nxt;
    }
    if (f & kWsFirst) acc = Ar<C>::zero();
    if ((f & (kWsQ1 | kWsQ2)) == (kWsQ1 | kWsQ2)) {
      const uint2 s0 = reinterpret_cast<const uint2*>(sb)[lane], s1 = reinterpret_cast<const uint2*>(sb + 256)[lane];
      WsVals<PA> v0, v1;
      v0.load(sb + OFF_VAL, lane);
      v1.load(sb + OFF_VAL + 32 * VQ, lane);
      const R x0 = ringR[s0.x & 0xffffu], x1 = ringR[s0.x >> 16], x2 = ringR[s0.y & 0xffffu], x3 = ringR[s0.y >> 16],
              x4 = ringR[s1.x & 0xffffu], x5 = ringR[s1.x >> 16], x6 = ringR[s1.y & 0xffffu], x7 = ringR[s1.y >> 16];
      term(v0, 0, x0);
      term(v0, 1, x1);
      term(v0, 2, x2);
      term(v0, 3, x3);
      term(v1, 0, x4);
      term(v1, 1, x5);
      term(v1, 2, x6);
      term(v1, 3, x7);
    } else if (f & kWsQ1) {
      const uint2 s0 = reinterpret_cast<const uint2*>(sb)[lane];
      WsVals<PA> v0;
      v0.load(sb + OFF_VAL, lane);
      const R x0 = ringR[s0.x & 0xffffu], x1 = ringR[s0.x >> 16], x2 = ringR[s0.y & 0xffffu], x3 = ringR[s0.y >> 16];
      term(v0, 0, x0);
      term(v0, 1, x1);
      term(v0, 2, x2);
      term(v0, 3, x3);
    }
    if (f & kWsLast) {
      const uint32_t row = reinterpret_cast<const uint32_t*>(sb + OFF_ROW)[lane];
      if (row != kWsPadIdx) yb[(uint32_t)((int64_t)row - B)] = acc;
    }
    if (f & kWsWend) window_end();
  };

  ws_static_for<0, S>([&](auto D) { fetch((uint32_t)decltype(D)::value, D); });
  for (uint32_t i = 0; i < nrec; i += S) {
    ws_static_for<0, S>([&](auto D) {
      constexpr int d = decltype(D)::value;
      if (i + d < nrec) {
        consume(D);
        fetch(i + d + S, D);
      }
    });
  }
  ws_cp_wait<0>();
  pdl_trigger();
}

}  // namespace f3rg
