// wsell_pk_layout.hpp -- host-side builder of the PACKED windowed SELL layout: the
// stream the fp16-matrix passes with a 2-byte ring (plain Richardson, the L3
// spmv_dots, the fp16 SpMV -- 3/4 of a config-5 solve) read instead of the
// 4-byte column word + 2-byte value of the general layout (engine.cpp build_wsell).
//
// One 32-bit word per SLOT: a 16-bit code in the low half, the entry's fp16 value in
// the high half (state.hpp kPk*):
//   * an entry whose column lies in its window's band and maps to a usable ring slot:
//     code = the slot (column mod kPkRing);
//   * any other ("far") entry takes TWO consecutive slots of its row, never split over
//     two quads: [kPkEsc + (column >> 16), +0] then [column & 0xffff, value];
//   * padding: [kPkPad, +0], the reserved ring slot that holds zero. The escape slot is
//     a padding slot to the arithmetic as well (value +0 times the zero slot).
// Rows keep their entries in stored column order, so the one-thread-per-row sum is the
// reference's (src/csr.cpp:23-37); the +-0 products of padding and escape slots leave
// the accumulator unchanged (it is never -0).
//
// Kernel windows lie on a GLOBAL grid of kPkTW rows (window base = row / kPkTW * kPkTW),
// so an entry's band does not depend on how the sort windows are split over the CTAs:
// a CTA owns whole sort windows and may start and end inside a kernel window.
// As in the general layout the rows of a sort window (kWsSortRows) are ordered by their
// (extended) length, descending and stable, cut into slices of 32 rows, stored
// chunk-major (chunk q = slots 4q..4q+3 of every lane's row), and a slice is as wide as
// its longest row rounded up to 4.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "state.hpp"

namespace f3rg {

struct PkLayoutHost {
  uint64_t E = 0;              // stored slots (padding and escape slots included)
  uint32_t G = 0;              // CTAs
  uint64_t far = 0;            // far entries (each took one extra slot)
  std::vector<uint32_t> soff;  // slices + 1: slot offset of each slice (multiples of 128)
  std::vector<uint32_t> row;   // slices * 32: matrix row of each slice lane (kWsPadIdx: none)
  std::vector<uint32_t> src;   // E: CSR entry whose value the slot carries (kWsPadIdx: +0)
  std::vector<uint16_t> code;  // E
  std::vector<uint32_t> cwin;  // G + 1: sort windows of each CTA
};

// rp/ci: the matrix's CSR (n rows, square, n < 2^30); G: CTAs (one per SM)
// cl: ring class of the geometry (state.hpp pk_ring / pk_tw / pk_w): 0 the packed fp16 stream's, 1 the 4-byte rings'
inline void pk_build_layout(uint64_t n, const uint32_t* rp, const uint32_t* ci, uint32_t G, PkLayoutHost& L, int cl = 0) {
  constexpr uint64_t SW = kWsSortRows, NS = kWsSortRows / 32;
  const int64_t TW = pk_tw(cl), W = pk_w(cl), RN = pk_ring(cl);
  const uint32_t kPkLimit = pk_pad(cl), kPkPad = pk_pad(cl), kPkEsc = pk_esc(cl);  // this class's codes
  if (n >= (1ull << 30)) throw std::length_error("packed windowed layout needs n < 2^30");
  const uint64_t nwin = (n + SW - 1) / SW, nsl = nwin * NS;
  L.G = G;
  // walks row r's entries and calls slot(pos, code, src) for every slot it takes; returns the slot count
  auto walk = [&](uint32_t r, auto&& slot, uint32_t* nfar = nullptr) {
    const int64_t B = (int64_t)(r / (uint64_t)TW) * TW;
    const int64_t lo = std::max<int64_t>(0, B - W), hi = std::min<int64_t>((int64_t)n, B + TW + W);
    uint32_t pos = 0;
    for (uint32_t k = rp[r]; k < rp[r + 1]; ++k) {
      const uint32_t c = ci[k];
      const uint32_t s = (uint32_t)((int64_t)c % RN);
      if ((int64_t)c >= lo && (int64_t)c < hi && s < kPkLimit) {
        slot(pos++, (uint16_t)s, k);
      } else {
        if ((pos & 3u) == 3u) slot(pos++, (uint16_t)kPkPad, kWsPadIdx);  // keep the pair inside one quad
        slot(pos++, (uint16_t)(kPkEsc + (c >> 16)), kWsPadIdx);
        slot(pos++, (uint16_t)(c & 0xffffu), k);
        if (nfar) ++*nfar;
      }
    }
    return pos;
  };
  std::vector<uint32_t> xlen(n);
  uint64_t far = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : far)
  for (int64_t r = 0; r < (int64_t)n; ++r) {
    uint32_t esc = 0;
    xlen[r] = walk((uint32_t)r, [](uint32_t, uint16_t, uint32_t) {}, &esc);
    far += esc;
  }
  L.far = far;
  L.row.assign(nwin * SW, kWsPadIdx);
  std::vector<uint32_t> width(nsl, 0);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t w = 0; w < (int64_t)nwin; ++w) {
    uint32_t* o = &L.row[(uint64_t)w * SW];
    const uint64_t r0 = (uint64_t)w * SW, r1 = std::min<uint64_t>(n, r0 + SW);
    for (uint64_t i = r0; i < r1; ++i) o[i - r0] = (uint32_t)i;
    std::stable_sort(o, o + (r1 - r0), [&](uint32_t a, uint32_t b) { return xlen[a] > xlen[b]; });
    for (uint64_t j = 0; j < NS; ++j) {
      uint32_t k = 0;
      for (uint64_t l = 0; l < 32; ++l) {
        const uint32_t r = o[j * 32 + l];
        if (r != kWsPadIdx) k = std::max(k, xlen[r]);
      }
      width[(uint64_t)w * NS + j] = (k + 3u) & ~3u;
    }
  }
  L.soff.assign(nsl + 1, 0);
  uint64_t acc = 0;
  for (uint64_t s = 0; s < nsl; ++s) {
    L.soff[s] = (uint32_t)acc;
    acc += (uint64_t)width[s] * 32u;
    if (acc >= (1ull << 32) - 256) throw std::length_error("packed windowed layout exceeds 2^32 slots");
  }
  L.soff[nsl] = (uint32_t)acc;
  L.E = acc;
  L.src.assign(L.E + 16, kWsPadIdx);
  L.code.assign(L.E + 16, (uint16_t)kPkPad);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t s = 0; s < (int64_t)nsl; ++s)
    for (uint32_t l = 0; l < 32; ++l) {
      const uint32_t r = L.row[(uint64_t)s * 32 + l];
      if (r == kWsPadIdx) continue;
      const uint64_t base = (uint64_t)L.soff[s] + l * 4u;
      walk(r, [&](uint32_t pos, uint16_t code, uint32_t k) {
        const uint64_t e = base + (uint64_t)(pos >> 2) * 128u + (pos & 3u);
        L.code[e] = code;
        L.src[e] = k;
      });
    }
  // CTA split: whole sort windows, balanced by stored slots
  L.cwin.assign(G + 1, 0);
  uint64_t w = 0;
  for (uint32_t c = 1; c < G; ++c) {
    const uint64_t target = (L.E * c + G - 1) / G;
    while (w < nwin && L.soff[w * NS] < target) ++w;
    L.cwin[c] = (uint32_t)w;
  }
  L.cwin[G] = (uint32_t)nwin;
}

}  // namespace f3rg
