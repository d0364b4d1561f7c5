// launch_setup.cu -- problem setup on the device: the symmetric
// diagonal scaling of reference src/scaling.cpp:11-38,
//   d_i = 1 / sqrt(|a_ii|),  a~_ij = (a_ij * d_i) * d_j,  b~_i = b_i * d_i,
// element-wise with the same IEEE operations in the same order (correctly rounded
// sqrt and division on both sides), so the scaled system is bit-identical.
#include "dispatch.cuh"

namespace f3rg {

// d from the diagonal entries (dpos[i] = position of a_ii); a zero diagonal records
// the smallest offending row in *bad (initialised to ~0 by the caller)
__global__ void __launch_bounds__(256) k_scale_d(const double* vals, const uint32_t* dpos, double* d, uint64_t n,
                                                 unsigned long long* bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double aii = vals[dpos[i]];
    if (aii == 0.0) atomicMin(bad, (unsigned long long)i);
    d[i] = __ddiv_rn(1.0, __dsqrt_rn(fabs(aii)));
  }
}

// a~_ij = (a_ij * d_i) * d_j, one thread per row (rows walk their entries in order)
__global__ void __launch_bounds__(256) k_scale_vals(const uint32_t* rp, const uint32_t* ci, double* vals,
                                                    const double* d, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double di = d[i];
    for (uint32_t k = rp[i]; k < rp[i + 1]; ++k) vals[k] = __dmul_rn(__dmul_rn(vals[k], di), d[ci[k]]);
  }
}

__global__ void __launch_bounds__(256) k_scale_rhs(const double* b, const double* d, double* out, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = __dmul_rn(b[i], d[i]);
}

cudaError_t launch_diag_scale(Launch l, const uint32_t* rp, const uint32_t* ci, double* vals, const uint32_t* dpos,
                              double* d, uint64_t n, unsigned long long* bad) {
  const int g = l.grid ? l.grid : stream_grid();
  k_scale_d<<<g, kThreads, 0, l.stream>>>(vals, dpos, d, n, bad);
  k_scale_vals<<<g, kThreads, 0, l.stream>>>(rp, ci, vals, d, n);
  return cudaGetLastError();
}

cudaError_t launch_scale_rhs(Launch l, const double* b, const double* d, double* out, uint64_t n) {
  const int g = l.grid ? l.grid : stream_grid();
  k_scale_rhs<<<g, kThreads, 0, l.stream>>>(b, d, out, n);
  return cudaGetLastError();
}

// Row permutation of a CSR value array (sorted-row tiles, engine.cpp
// DeviceMatrix::init): new row q is old row perm[q], dst[rp_new[q] + t] =
// src[rp_old[perm[q]] + t]; one warp per row, E-byte elements copied bit for bit.
template <class E>
__global__ void __launch_bounds__(256) k_permute_rows(const uint32_t* rp_old, const uint32_t* rp_new,
                                                      const uint32_t* perm, const E* src, E* dst, uint64_t n) {
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  const unsigned lane = threadIdx.x & 31u;
  for (uint64_t q = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; q < n; q += warps) {
    const uint32_t o = rp_old[perm[q]], b = rp_new[q], len = rp_new[q + 1] - b;
    for (uint32_t t = lane; t < len; t += 32) dst[b + t] = src[o + t];
  }
}

cudaError_t launch_permute_rows(Launch l, int esize, const uint32_t* rp_old, const uint32_t* rp_new,
                                const uint32_t* perm, const void* src, void* dst, uint64_t n) {
  const int g = l.grid ? l.grid : stream_grid();
  switch (esize) {
    case 2: k_permute_rows<<<g, kThreads, 0, l.stream>>>(rp_old, rp_new, perm, static_cast<const uint16_t*>(src),
                                                          static_cast<uint16_t*>(dst), n); break;
    case 4: k_permute_rows<<<g, kThreads, 0, l.stream>>>(rp_old, rp_new, perm, static_cast<const uint32_t*>(src),
                                                          static_cast<uint32_t*>(dst), n); break;
    case 8: k_permute_rows<<<g, kThreads, 0, l.stream>>>(rp_old, rp_new, perm,
                                                          static_cast<const unsigned long long*>(src),
                                                          static_cast<unsigned long long*>(dst), n); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// Windowed SELL layout (wsell.cuh, engine.cpp build_wsell): entry e of the layout is
// CSR entry src[e] (kWsPad: a padding slot). Columns get kWsPad, values +0 there
// (never read: the engine skips padded columns); everything else is copied bit for bit.
template <class E>
__global__ void __launch_bounds__(256) k_ws_scatter(const uint32_t* src, const E* in, E* out, uint64_t cnt, E pad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += stride) {
    const uint32_t k = src[e];
    out[e] = k == 0xffffffffu ? pad : in[k];
  }
}

cudaError_t launch_ws_scatter(Launch l, int esize, const uint32_t* src, const void* in, void* out, uint64_t cnt,
                              bool pad_ones) {
  const int g = l.grid ? l.grid : stream_grid();
  switch (esize) {
    case 2: k_ws_scatter<<<g, kThreads, 0, l.stream>>>(src, static_cast<const uint16_t*>(in),
                                                        static_cast<uint16_t*>(out), cnt, (uint16_t)0); break;
    case 4: k_ws_scatter<<<g, kThreads, 0, l.stream>>>(src, static_cast<const uint32_t*>(in),
                                                        static_cast<uint32_t*>(out), cnt,
                                                        pad_ones ? 0xffffffffu : 0u); break;
    case 8: k_ws_scatter<<<g, kThreads, 0, l.stream>>>(src, static_cast<const unsigned long long*>(in),
                                                        static_cast<unsigned long long*>(out), cnt, 0ull); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// Encoded column stream of the windowed engine for one ring class (wsell.cuh): one
// warp per 32-row slice. The slice's kernel window follows from its sort window and
// the CTA that owns it (cwin: G + 1 sort-window boundaries): the CTA's windows start
// at its first sort window and hold KW sort windows each. An entry whose column lies
// in the window's band [B - W, B + TW + W) (clipped to [0, n)) becomes the byte
// offset of its ring slot, (column mod RN) * RS; padding becomes zoff; any other
// entry keeps its column with kWsFarBit set.
__global__ void __launch_bounds__(256) k_ws_encode(const uint32_t* __restrict__ src, const uint32_t* __restrict__ ci,
                                                   const uint32_t* __restrict__ soff, const uint32_t* __restrict__ cwin,
                                                   uint32_t G, uint64_t nsl, uint64_t n, int cl, uint32_t zoff,
                                                   uint32_t* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t RN = ws_rn(cl), TW = ws_tw(cl), W = ws_w(cl);
  const uint32_t KW = (uint32_t)(TW / (int64_t)kWsSortRows), RS = 2u << cl;
  for (uint64_t s = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < nsl; s += nwarps) {
    const uint32_t sw = (uint32_t)(s / (kWsSortRows / 32));
    uint32_t lo_g = 0, hi_g = G;  // the CTA g with cwin[g] <= sw < cwin[g + 1]
    while (hi_g - lo_g > 1) {
      const uint32_t mid = (lo_g + hi_g) >> 1;
      if (cwin[mid] <= sw) lo_g = mid;
      else hi_g = mid;
    }
    const uint32_t sw0 = cwin[lo_g];
    const int64_t B = (int64_t)(sw0 + (sw - sw0) / KW * KW) * (int64_t)kWsSortRows;
    const int64_t lo = B - W < 0 ? 0 : B - W, hi = B + TW + W > (int64_t)n ? (int64_t)n : B + TW + W;
    for (uint32_t e = soff[s] + lane; e < soff[s + 1]; e += 32u) {
      const uint32_t k = src[e];
      uint32_t v = zoff;
      if (k != kWsPadIdx) {
        const uint32_t c = ci[k];
        v = ((int64_t)c >= lo && (int64_t)c < hi) ? (uint32_t)((int64_t)c & (RN - 1)) * RS : (kWsFarBit | c);
      }
      out[e] = v;
    }
  }
}

cudaError_t launch_ws_encode(Launch l, const uint32_t* src, const uint32_t* ci, const uint32_t* soff,
                             const uint32_t* cwin, uint32_t G, uint64_t nsl, uint64_t n, int cl, uint32_t* out) {
  const int g = l.grid ? l.grid : stream_grid();
  k_ws_encode<<<g, kThreads, 0, l.stream>>>(src, ci, soff, cwin, G, nsl, n, cl, kWsZeroOffset, out);
  return cudaGetLastError();
}

// Packed windowed layout (wsell_pk_layout.hpp): word = slot code | fp16 value bits << 16; a slot
// without an entry of its own (padding, the escape half of a far pair) carries +0
__global__ void __launch_bounds__(256) k_pk_pack(const uint32_t* __restrict__ src, const uint16_t* __restrict__ code,
                                                 const uint16_t* __restrict__ val16, uint32_t* __restrict__ out,
                                                 uint64_t cnt) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += stride) {
    const uint32_t k = src[e];
    out[e] = (uint32_t)code[e] | (k == kWsPadIdx ? 0u : (uint32_t)val16[k] << 16);
  }
}

cudaError_t launch_pk_pack(Launch l, const uint32_t* src, const uint16_t* code, const void* val16, uint32_t* out,
                           uint64_t cnt) {
  const int g = l.grid ? l.grid : stream_grid();
  k_pk_pack<<<g, kThreads, 0, l.stream>>>(src, code, static_cast<const uint16_t*>(val16), out, cnt);
  return cudaGetLastError();
}

}  // namespace f3rg
