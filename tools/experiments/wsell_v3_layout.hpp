// wsell_layout.hpp -- host-side builder of the windowed SELL layout the device
// engine in wsell.cuh streams (gather-bound matrices, config 5). Header-only so the
// tuning microbenchmark (tools/wsell_microbench.cu) builds exactly what engine.cpp
// uploads.
//
// Rows: inside sort windows of kWsSortRows consecutive rows the rows are ordered by
// length (descending, stable) and cut into slices of 32 rows; a slice stores its
// entries chunk-major -- chunk q holds entries 4q..4q+3 of every lane's row, 32 lanes
// x 4 entries = 128 slots, lane l's quad at [q*128 + l*4] -- and is as wide as its
// longest row rounded up to 4. Each row's entries keep their stored column order, so
// the one-thread-per-row sum is the reference's (src/csr.cpp:23-37).
//
// Per ring class (state.hpp: 2-/4-/8-byte ring elements) the CTA's rows are cut into
// kernel windows of TW rows and every stored entry becomes a 16-bit slot:
//   * column inside the window's band [B - W, B + TW + W): slot = column mod RN, the
//     position the ring keeps x[column] at, whatever the window;
//   * any other column ("far", config 5's 5 % uniform long-range entries): the entry's
//     position in its far segment, inside the scratch of the warp that will run it;
//     the segment's columns go to the far list, which the warp gathers one segment
//     ahead of its use;
//   * padding: the slot that always holds zero (the padded value is +0 too; a row
//     accumulator is never -0, so adding the +-0 product leaves it unchanged).
// The warps' work is fixed here as well: in every kernel window the slices go to the
// kWsWarps warps longest-processing-time-first, and each warp's slices, over all the
// windows of its CTA, are flattened into one list of step records (one or two chunks
// per step) flagged with what happens around the step (slice start / end, far-segment
// start, window end). The device loop has no per-entry decisions left.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "state.hpp"

namespace f3rg {

struct WsClassHost {
  std::vector<uint16_t> slot;  // one per stored entry (+ pad)
  std::vector<uint2> rec;      // step records, (CTA, warp)-major
  std::vector<uint32_t> far;   // far columns, segment after segment (each padded to a multiple of 4 entries)
  std::vector<uint4> hdr;      // per (CTA, warp): {first record, records, first far column, far entries of segment 0}
};

struct WsLayoutHost {
  uint64_t E = 0;              // stored entries (padding included)
  uint32_t G = 0;              // CTAs the windows are split over
  std::vector<uint32_t> soff;  // slices + 1: entry offset of each slice (multiples of 128)
  std::vector<uint32_t> row;   // slices * 32: matrix row of each slice lane (kWsPadIdx: none)
  std::vector<uint32_t> src;   // E: CSR entry of each stored entry (kWsPadIdx: padding)
  std::vector<uint32_t> cwin;  // G + 1: sort windows of each CTA
  WsClassHost cls[3];
};

namespace ws_detail {

struct WarpList {
  std::vector<uint2> rec;
  std::vector<uint32_t> far;
  std::vector<uint32_t> segrec;  // record that opens each segment
  std::vector<uint32_t> segcnt;  // far entries of each segment
  uint32_t segfar = 0;           // far entries in the open segment
  void close_segment() {         // pad the open segment's columns to a multiple of 4 (16-byte copies)
    if (segrec.empty()) return;
    segcnt.push_back(segfar);
    while (far.size() % 4) far.push_back(0u);
  }
};

}  // namespace ws_detail

// rp/ci: the matrix's CSR (n rows, square); G: CTAs (one per SM)
inline void ws_build_layout(uint64_t n, const uint32_t* rp, const uint32_t* ci, uint32_t G, WsLayoutHost& L) {
  using namespace ws_detail;
  constexpr uint64_t SW = kWsSortRows, NS = kWsSortRows / 32;
  const uint64_t nwin = (n + SW - 1) / SW, nsl = nwin * NS;
  auto len = [&](uint32_t i) { return rp[i + 1] - rp[i]; };
  L.G = G;
  L.row.assign(nwin * SW, kWsPadIdx);
  std::vector<uint32_t> width(nsl, 0);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t w = 0; w < (int64_t)nwin; ++w) {
    uint32_t* o = &L.row[(uint64_t)w * SW];
    const uint64_t r0 = (uint64_t)w * SW, r1 = std::min<uint64_t>(n, r0 + SW);
    for (uint64_t i = r0; i < r1; ++i) o[i - r0] = (uint32_t)i;
    std::stable_sort(o, o + (r1 - r0), [&](uint32_t a, uint32_t b) { return len(a) > len(b); });
    for (uint64_t j = 0; j < NS; ++j) {
      uint32_t k = 0;
      for (uint64_t l = 0; l < 32; ++l) {
        const uint32_t r = o[j * 32 + l];
        if (r != kWsPadIdx) k = std::max(k, len(r));
      }
      width[(uint64_t)w * NS + j] = (k + 3u) & ~3u;
    }
  }
  L.soff.assign(nsl + 1, 0);
  uint64_t acc = 0;
  for (uint64_t s = 0; s < nsl; ++s) {
    L.soff[s] = (uint32_t)acc;
    acc += (uint64_t)width[s] * 32u;
    // entry offsets are 32-bit, chunk indices (entry / 128) 24-bit in the step records
    if (acc >= (1ull << 31) || nsl >= (1ull << 24)) throw std::length_error("windowed SELL layout exceeds 2^31 entries");
  }
  L.soff[nsl] = (uint32_t)acc;
  L.E = acc;
  L.src.assign(L.E + 16, kWsPadIdx);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t s = 0; s < (int64_t)nsl; ++s)
    for (uint32_t l = 0; l < 32; ++l) {
      const uint32_t r = L.row[(uint64_t)s * 32 + l];
      if (r == kWsPadIdx) continue;
      const uint32_t ln = len(r);
      for (uint32_t k = 0; k < ln; ++k) L.src[L.soff[s] + (k >> 2) * 128u + l * 4u + (k & 3u)] = rp[r] + k;
    }
  // CTA split: whole sort windows, balanced by stored entries
  L.cwin.assign(G + 1, 0);
  {
    uint64_t w = 0;
    for (uint32_t c = 1; c < G; ++c) {
      const uint64_t target = (L.E * c + G - 1) / G;
      while (w < nwin && L.soff[w * NS] < target) ++w;
      L.cwin[c] = (uint32_t)w;
    }
    L.cwin[G] = (uint32_t)nwin;
  }

  for (int cl = 0; cl < 3; ++cl) {
    WsClassHost& K = L.cls[cl];
    const int64_t RN = ws_rn(cl), TW = ws_tw(cl), W = ws_w(cl);
    const uint32_t KW = (uint32_t)(TW / (int64_t)SW);
    const uint32_t FAR0 = (uint32_t)ws_far0(cl), ZERO = (uint32_t)ws_zero(cl);
    K.slot.assign(L.E + 16, (uint16_t)ZERO);
    std::vector<WarpList> lists((size_t)G * kWsWarps);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t g = 0; g < (int64_t)G; ++g) {
      WarpList* wl = &lists[(size_t)g * kWsWarps];
      std::vector<uint32_t> ids;
      std::vector<uint32_t> mine[kWsWarps];
      uint32_t col[2][128];
      uint8_t kind[2][128];  // 0 padding, 1 ring, 2 far
      for (uint32_t sw = L.cwin[g]; sw < L.cwin[g + 1]; sw += KW) {
        const uint32_t kw = std::min<uint32_t>(KW, L.cwin[g + 1] - sw);
        const int64_t B = (int64_t)sw * (int64_t)SW;
        const int64_t lo = std::max<int64_t>(0, B - W), hi = std::min<int64_t>((int64_t)n, B + TW + W);
        ids.clear();
        for (uint32_t s = sw * (uint32_t)NS; s < (sw + kw) * (uint32_t)NS; ++s) ids.push_back(s);
        auto nch = [&](uint32_t s) { return (L.soff[s + 1] - L.soff[s]) >> 7; };
        std::stable_sort(ids.begin(), ids.end(), [&](uint32_t a, uint32_t b) { return nch(a) > nch(b); });
        uint64_t load[kWsWarps] = {};
        for (int w = 0; w < kWsWarps; ++w) mine[w].clear();
        for (uint32_t s : ids) {  // longest processing time first
          int best = 0;
          for (int w = 1; w < kWsWarps; ++w)
            if (load[w] < load[best]) best = w;
          mine[best].push_back(s);
          load[best] += nch(s) + 1u;
        }
        for (int w = 0; w < kWsWarps; ++w) {
          WarpList& Q = wl[w];
          const size_t rec0 = Q.rec.size();
          // classify one chunk: columns and kinds of its 128 entries; returns the far count
          auto classify = [&](uint32_t e0, int t) {
            uint32_t nf = 0;
            for (uint32_t q = 0; q < 128; ++q) {
              const uint32_t k = L.src[e0 + q];
              if (k == kWsPadIdx) {
                kind[t][q] = 0;
                continue;
              }
              const uint32_t c = ci[k];
              col[t][q] = c;
              const bool in = (int64_t)c >= lo && (int64_t)c < hi;
              kind[t][q] = in ? 1 : 2;
              nf += in ? 0u : 1u;
            }
            return nf;
          };
          auto place = [&](uint32_t e0, int t) {
            for (uint32_t q = 0; q < 128; ++q) {
              if (kind[t][q] == 1) {
                K.slot[e0 + q] = (uint16_t)(col[t][q] % (uint32_t)RN);
              } else if (kind[t][q] == 2) {
                K.slot[e0 + q] = (uint16_t)(FAR0 + (uint32_t)w * kWsFarSlots + Q.segfar++);
                Q.far.push_back(col[t][q]);
              }
            }
          };
          for (uint32_t s : mine[w]) {
            const uint32_t nc = nch(s), e0 = L.soff[s];
            if (nc == 0) {  // only empty rows: their sums are +0
              Q.rec.push_back(uint2{(kWsFirst | kWsLast) << 24, s});
              continue;
            }
            uint32_t c = 0;
            while (c < nc) {
              uint32_t flags = kWsQ1 | (c == 0 ? kWsFirst : 0u);
              const uint32_t cstart = c;
              const uint32_t f1 = classify(e0 + c * 128u, 0);
              if (Q.segrec.empty() || Q.segfar + f1 > (uint32_t)kWsFarSlots) {
                Q.close_segment();
                Q.segrec.push_back((uint32_t)Q.rec.size());  // this step's record, pushed below
                Q.segfar = 0;
                flags |= kWsSeg;
              }
              place(e0 + c * 128u, 0);
              ++c;
              if (c < nc) {
                const uint32_t f2 = classify(e0 + c * 128u, 1);
                if (Q.segfar + f2 <= (uint32_t)kWsFarSlots) {
                  place(e0 + c * 128u, 1);
                  flags |= kWsQ2;
                  ++c;
                }
              }
              if (c >= nc) flags |= kWsLast;
              Q.rec.push_back(uint2{((e0 >> 7) + cstart) | (flags << 24), s});
            }
          }
          if (Q.rec.size() == rec0) Q.rec.push_back(uint2{kWsWend << 24, 0u});  // nothing to do in this window
          else Q.rec.back().x |= kWsWend << 24;
        }
      }
    }
    // concatenate the (CTA, warp) lists
    const size_t NL = lists.size();
    std::vector<uint64_t> ro(NL + 1, 0), fo(NL + 1, 0);
    for (size_t i = 0; i < NL; ++i) {
      WarpList& Q = lists[i];
      Q.close_segment();
      // a segment-opening record carries the size of the segment after it
      for (size_t q = 0; q < Q.segrec.size(); ++q)
        Q.rec[Q.segrec[q]].y |= (q + 1 < Q.segcnt.size() ? Q.segcnt[q + 1] : 0u) << 24;
      ro[i + 1] = ro[i] + Q.rec.size();
      fo[i + 1] = fo[i] + Q.far.size();
    }
    if (fo[NL] >= (1ull << 32) || ro[NL] >= (1ull << 32)) throw std::length_error("windowed SELL schedule too large");
    K.rec.assign(ro[NL] + 64, uint2{0u, 0u});
    K.far.assign(fo[NL] + 256, 0u);
    K.hdr.resize(NL);
#pragma omp parallel for schedule(dynamic, 32)
    for (int64_t i = 0; i < (int64_t)NL; ++i) {
      const WarpList& Q = lists[i];
      std::copy(Q.rec.begin(), Q.rec.end(), K.rec.begin() + ro[i]);
      std::copy(Q.far.begin(), Q.far.end(), K.far.begin() + fo[i]);
      K.hdr[i] = uint4{(uint32_t)ro[i], (uint32_t)Q.rec.size(), (uint32_t)fo[i], Q.segcnt.empty() ? 0u : Q.segcnt[0]};
    }
  }
}

}  // namespace f3rg
