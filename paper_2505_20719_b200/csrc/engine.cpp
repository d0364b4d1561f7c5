// engine.cpp -- host driver of the device level chain.
//
// Mirrors ComposedSolver (reference src/nesting.cpp:176-352) with every level
// below the outermost one executed as device work captured ONCE into a CUDA graph
// (one graph = one full invocation of level 2, i.e. the preconditioning action of
// one outer Arnoldi step, ~130 kernel nodes for fp16-F3R). The host synchronises
// once per outer step, for the reference's only data-dependent stop
// (|g_{j+1}| < tol*||b||, src/fgmres.cpp:127). Inner levels run their full
// budgets with no tolerance test (src/nesting.cpp:99); their rare early stops
// (happy breakdown / NaN) are honoured on the device through per-level "dead"
// flags that gate every later kernel of that invocation.
#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "launch.hpp"
#include "wsell_pk_layout.hpp"

namespace f3rg {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void DevBuf::alloc(size_t bytes) {
  release();
  if (bytes == 0) bytes = 16;
  F3RG_CUDA(cudaMalloc(&p_, bytes));
  n_ = bytes;
}
void DevBuf::release() {
  if (p_) cudaFree(p_);
  p_ = nullptr;
  n_ = 0;
}

static size_t psize(int p) { return p == 0 ? 2 : p == 1 ? 4 : 8; }

// ---- DeviceMatrix -------------------------------------------------------------------
void validate_csr(uint64_t n, const uint32_t* rp, const uint32_t* ci, uint64_t ncols) {
  const uint64_t lim = uint64_t{1} << 31;
  if (ncols == 0) ncols = n;
  if (n >= lim || ncols >= lim) throw Error(ERR_DIMENSION, "matrix exceeds 32-bit index range");
  if (!rp) throw Error(ERR_DIMENSION, "row_ptr length must be n+1");
  const uint64_t nnz = rp[n];
  if (nnz >= lim) throw Error(ERR_DIMENSION, "matrix exceeds 32-bit index range");
  if (rp[0] != 0) throw Error(ERR_DIMENSION, "row_ptr endpoints invalid");
  for (uint64_t i = 0; i < n; ++i) {
    if (rp[i] > rp[i + 1]) throw Error(ERR_DIMENSION, "row_ptr must be non-decreasing");
    for (uint32_t k = rp[i]; k < rp[i + 1]; ++k) {
      if (ci[k] >= ncols) throw Error(ERR_DIMENSION, "column index out of bounds in row " + std::to_string(i));
      if (k > rp[i] && ci[k] <= ci[k - 1])
        throw Error(ERR_DIMENSION, "columns must be strictly increasing in row " + std::to_string(i));
    }
  }
}

DeviceMatrix::DeviceMatrix(uint64_t n, const uint32_t* row_ptr, const uint32_t* col_idx, const double* values,
                           uint64_t ncols)
    : n_(n), nnz_(row_ptr ? row_ptr[n] : 0) {
  init(row_ptr, col_idx, values, ncols, nullptr);
}

DeviceMatrix::DeviceMatrix(uint64_t n, const uint32_t* row_ptr, const uint32_t* col_idx, const double* values,
                           Scale scale)
    : n_(n), nnz_(row_ptr ? row_ptr[n] : 0) {
  init(row_ptr, col_idx, values, 0, &scale);
}

void DeviceMatrix::init(const uint32_t* row_ptr, const uint32_t* col_idx, const double* values, uint64_t ncols,
                        const Scale* scale) {
  validate_csr(n_, row_ptr, col_idx, ncols);
  // diagonal positions for the device scaling (the reference's diagonal_index
  // lookup and its missing-diagonal error, src/scaling.cpp:14-16)
  std::vector<uint32_t> dpos;
  if (scale) {
    dpos.resize(n_ + 1);
    for (uint64_t i = 0; i < n_; ++i) {
      const uint32_t* b = col_idx + row_ptr[i];
      const uint32_t* e = col_idx + row_ptr[i + 1];
      const uint32_t* it = std::lower_bound(b, e, (uint32_t)i);
      if (it == e || *it != i)
        throw Error(ERR_FACTORIZATION, "diagonal scaling: missing diagonal entry in row " + std::to_string(i));
      dpos[i] = (uint32_t)(it - col_idx);
      if (values[dpos[i]] == 0.0)
        throw Error(ERR_FACTORIZATION, "diagonal scaling: zero diagonal entry in row " + std::to_string(i));
    }
  }
  // padded so the 16-byte-granular bulk copies never read past an allocation
  rp_.alloc((n_ + 1) * 4 + 32);
  ci_.alloc(nnz_ * 4 + 32);
  F3RG_CUDA(cudaMemset(rp_.get(), 0, rp_.bytes()));
  F3RG_CUDA(cudaMemset(ci_.get(), 0, ci_.bytes()));
  F3RG_CUDA(cudaMemcpy(rp_.get(), row_ptr, (n_ + 1) * 4, cudaMemcpyHostToDevice));
  if (nnz_) F3RG_CUDA(cudaMemcpy(ci_.get(), col_idx, nnz_ * 4, cudaMemcpyHostToDevice));
  for (int p = 0; p < 3; ++p) {
    val_[p].alloc(nnz_ * psize(p) + 32);
    F3RG_CUDA(cudaMemset(val_[p].get(), 0, val_[p].bytes()));
  }
  if (nnz_) F3RG_CUDA(cudaMemcpy(val_[2].get(), values, nnz_ * 8, cudaMemcpyHostToDevice));
  if (scale && n_) {
    DevBuf dp(n_ * 4 + 16), d(n_ * 8 + 16), bad(16);
    F3RG_CUDA(cudaMemcpy(dp.get(), dpos.data(), n_ * 4, cudaMemcpyHostToDevice));
    F3RG_CUDA(cudaMemset(bad.get(), 0xff, 8));
    F3RG_CUDA(launch_diag_scale(Launch{}, rp_.get<uint32_t>(), ci_.get<uint32_t>(), val_[2].get<double>(),
                                dp.get<uint32_t>(), d.get<double>(), n_, bad.get<unsigned long long>()));
    if (scale->d_dev) F3RG_CUDA(cudaMemcpy(scale->d_dev, d.get(), n_ * 8, cudaMemcpyDeviceToDevice));
  }
  // replicas: element-wise RNE demotion on the device (cvt.rn.f32.f64 / cvt.rn.f16.f64)
  F3RG_CUDA(launch_copy(2, 1, Launch{}, val_[2].get(), val_[1].get(), nnz_));
  F3RG_CUDA(launch_copy(2, 0, Launch{}, val_[2].get(), val_[0].get(), nnz_));
  // D16 column stream when every in-row gap fits 16 bits (F3RG_COLUMNS=u32 forces
  // the plain u32 stream, for A/B tests)
  const char* colfmt = std::getenv("F3RG_COLUMNS");
  bool d16 = !(colfmt && std::string(colfmt) == "u32") && nnz_ > 0;
  const bool p16 = !(colfmt && (std::string(colfmt) == "u32" || std::string(colfmt) == "d16"));
  for (uint64_t i = 0; d16 && i < n_; ++i)
    for (uint32_t k = row_ptr[i] + 1; k < row_ptr[i + 1]; ++k)
      if (col_idx[k] - col_idx[k - 1] > 65536u) {  // stored as gap - 1 (columns strictly increase)
        d16 = false;
        break;
      }
  // D16 / P16 streams of one row order (rp/ci on the host, the fp16 values on the device)
  auto delta_streams = [&](const uint32_t* rp, const uint32_t* ci, const DevBuf& v16, DevBuf& dcol, DevBuf& first,
                           DevBuf& pk) {
    std::vector<uint16_t> dc(nnz_ + 16, 0);
    std::vector<uint32_t> fc(n_ + 16, 0);
    for (uint64_t i = 0; i < n_; ++i) {
      if (rp[i] < rp[i + 1]) fc[i] = ci[rp[i]];
      for (uint32_t k = rp[i] + 1; k < rp[i + 1]; ++k) dc[k] = (uint16_t)(ci[k] - ci[k - 1] - 1u);
    }
    dcol.alloc(dc.size() * 2);
    first.alloc(fc.size() * 4);
    F3RG_CUDA(cudaMemcpy(dcol.get(), dc.data(), dc.size() * 2, cudaMemcpyHostToDevice));
    F3RG_CUDA(cudaMemcpy(first.get(), fc.data(), fc.size() * 4, cudaMemcpyHostToDevice));
    if (p16) {  // F3RG_COLUMNS=d16 keeps the separate fp16 value + delta streams
      pk.alloc(nnz_ * 4 + 32);
      F3RG_CUDA(cudaMemset(pk.get(), 0, pk.bytes()));
      F3RG_CUDA(launch_pack16(Launch{}, v16.get(), dcol.get<uint16_t>(), pk.get<uint32_t>(), nnz_));
    }
  };
  if (d16) delta_streams(row_ptr, col_idx, val_[0], dcol_, first_, pk_);
  // tile shape: short-row tiles (one gather chunk per row, four CTAs per SM) for
  // matrices averaging <= 12 entries per row -- the 7-point operators; the
  // 27-point and unstructured ones keep the regular shape (F3RG_SHAPE=0/1 forces)
  const char* shp = std::getenv("F3RG_SHAPE");
  const bool forced_shape = shp && *shp;
  shape_ = forced_shape ? std::min(2, std::max(0, std::atoi(shp))) : (n_ > 0 && nnz_ <= 12 * n_);
  std::vector<uint32_t> r0, k0;
  // Sorted-row tiles for irregular row lengths: a tile takes as long as its longest
  // row (one thread per row, sequential sums), so when the fp16 tiles' thread-slot
  // load sum(max row length x rows) exceeds 1.5x nnz (config 5: 3.6x) the tile
  // engine streams a copy whose rows are ordered by length (descending, stable)
  // inside windows of sigma = 8192 rows (config 5: 1.13x). F3RG_SORT_ROWS=0/1 forces.
  bool sort_rows = false;
  if (n_ > 0 && nnz_ > 0) {
    const char* so = std::getenv("F3RG_SORT_ROWS");
    if (so && *so) {
      sort_rows = std::atoi(so) != 0;
    } else {
      build_tiles(n_, row_ptr, tile_max_rows(), tile_max_nnz(0 /* fp16 */, shape_), r0, k0);
      double load = 0;
      for (size_t t = 0; t + 1 < r0.size(); ++t) {
        uint32_t mx = 0;
        for (uint32_t i = r0[t]; i < r0[t + 1]; ++i) mx = std::max(mx, row_ptr[i + 1] - row_ptr[i]);
        load += (double)mx * (r0[t + 1] - r0[t]);
      }
      sort_rows = load > 1.5 * (double)nnz_;
    }
  }
  // irregular rows are gather-bound rows (config 5): half-size tiles leave L1 room
  if (sort_rows && !forced_shape && shape_ == 0) shape_ = 2;
  // ... and go to the windowed SELL engine (wsell.cuh) when the matrix is square and
  // on one rank (the engine's band of x is indexed by row); F3RG_WSELL=0/1 forces
  {
    const char* wse = std::getenv("F3RG_WSELL");
    const bool square = ncols == 0 || ncols == n_;
    const bool want = wse && *wse ? wse[0] != '0' : (sort_rows && !forced_shape);
    if (want && square && n_ > 0 && nnz_ > 0 && n_ < (1ull << 30)) {
      build_wsell(row_ptr);
      build_wsell_pk(row_ptr, col_idx);
      shape_ = 3;
      sort_rows = false;
    }
  }
  const uint32_t* trp = row_ptr;  // row pointers the tiles are cut from
  std::vector<uint32_t> srp;
  if (sort_rows) {
    const char* sg = std::getenv("F3RG_SORT_SIGMA");
    const uint64_t sigma = sg && *sg ? std::max<long long>(1, std::atoll(sg)) : 8192;
    std::vector<uint32_t> perm(n_);
    for (uint64_t i = 0; i < n_; ++i) perm[i] = (uint32_t)i;
    auto len = [&](uint32_t i) { return row_ptr[i + 1] - row_ptr[i]; };
    for (uint64_t w = 0; w < n_; w += sigma)
      std::stable_sort(perm.begin() + w, perm.begin() + std::min(n_, w + sigma),
                       [&](uint32_t a, uint32_t b) { return len(a) > len(b); });
    srp.assign(n_ + 1, 0);
    std::vector<uint32_t> sci(nnz_ + 16, 0);
    for (uint64_t q = 0; q < n_; ++q) {
      const uint32_t i = perm[q];
      srp[q + 1] = srp[q] + len(i);
      std::copy(col_idx + row_ptr[i], col_idx + row_ptr[i + 1], sci.begin() + srp[q]);
    }
    perm_.alloc(n_ * 4 + 16);
    srp_.alloc((n_ + 1) * 4 + 32);
    sci_.alloc(nnz_ * 4 + 32);
    F3RG_CUDA(cudaMemset(srp_.get(), 0, srp_.bytes()));
    F3RG_CUDA(cudaMemset(sci_.get(), 0, sci_.bytes()));
    F3RG_CUDA(cudaMemcpy(perm_.get(), perm.data(), n_ * 4, cudaMemcpyHostToDevice));
    F3RG_CUDA(cudaMemcpy(srp_.get(), srp.data(), (n_ + 1) * 4, cudaMemcpyHostToDevice));
    F3RG_CUDA(cudaMemcpy(sci_.get(), sci.data(), nnz_ * 4, cudaMemcpyHostToDevice));
    for (int p = 0; p < 3; ++p) {  // the (scaled, demoted) values, moved on the device bit for bit
      sval_[p].alloc(nnz_ * psize(p) + 32);
      F3RG_CUDA(cudaMemset(sval_[p].get(), 0, sval_[p].bytes()));
      F3RG_CUDA(launch_permute_rows(Launch{}, (int)psize(p), rp_.get<uint32_t>(), srp_.get<uint32_t>(),
                                    perm_.get<uint32_t>(), val_[p].get(), sval_[p].get(), n_));
    }
    if (d16) delta_streams(srp.data(), sci.data(), sval_[0], sdcol_, sfirst_, spk_);
    trp = srp.data();
  }
  for (int p = 0; p < 3; ++p) {
    build_tiles(n_, trp, tile_max_rows(), tile_max_nnz(p, shape_), r0, k0);
    ntiles_[p] = (uint32_t)(r0.size() - 1);
    tr0_[p].alloc(r0.size() * 4);
    tk0_[p].alloc(k0.size() * 4);
    F3RG_CUDA(cudaMemcpy(tr0_[p].get(), r0.data(), r0.size() * 4, cudaMemcpyHostToDevice));
    F3RG_CUDA(cudaMemcpy(tk0_[p].get(), k0.data(), k0.size() * 4, cudaMemcpyHostToDevice));
  }
  // L2 eviction priorities (common.cuh l2_policy) once a pass streams more than half
  // the 126 MB L2: then the gathered vector, not the matrix, is what the L2 can keep
  // (config 1's 11 MB fp16 replica stays L2-resident across passes without them).
  // F3RG_L2HINT=0/1 forces.
  const char* h = std::getenv("F3RG_L2HINT");
  l2hint_ = h && *h ? (h[0] == '0' ? 0u : 1u) : (stream_bytes(0) > 64e6 ? 1u : 0u);
  F3RG_CUDA(cudaDeviceSynchronize());
}

// Windowed SELL layout (wsell.cuh): rows sorted by length inside windows of
// kWsSortRows, 64 slices of 32 rows per window, each slice chunk-major and as wide
// as its longest row rounded up to 4; the windows are split over one CTA per SM by
// stored entries. The columns and the three value replicas are moved into the
// layout on the device, bit for bit.
void DeviceMatrix::build_wsell(const uint32_t* rp) {
  constexpr uint64_t SW = kWsSortRows, NS = kWsSortRows / 32;
  const uint64_t nwin = (n_ + SW - 1) / SW, nsl = nwin * NS;
  auto len = [&](uint32_t i) { return rp[i + 1] - rp[i]; };
  std::vector<uint32_t> order(nwin * SW, kWsPadIdx), width(nsl, 0);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t w = 0; w < (int64_t)nwin; ++w) {
    uint32_t* o = &order[(uint64_t)w * SW];
    const uint64_t r0 = (uint64_t)w * SW, r1 = std::min<uint64_t>(n_, r0 + SW);
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
  std::vector<uint32_t> soff(nsl + 1, 0);
  uint64_t acc = 0;
  for (uint64_t s = 0; s < nsl; ++s) {
    soff[s] = (uint32_t)acc;
    acc += (uint64_t)width[s] * 32u;
    if (acc >= 0xffffffffull) throw Error(ERR_UNSUPPORTED, "windowed SELL layout exceeds 2^32 entries");
  }
  soff[nsl] = (uint32_t)acc;
  ws_E_ = acc;
  std::vector<uint32_t> src(ws_E_ + 16, kWsPadIdx);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t s = 0; s < (int64_t)nsl; ++s)
    for (uint32_t l = 0; l < 32; ++l) {
      const uint32_t r = order[(uint64_t)s * 32 + l];
      if (r == kWsPadIdx) continue;
      const uint32_t L = len(r);
      for (uint32_t k = 0; k < L; ++k) src[soff[s] + (k >> 2) * 128u + l * 4u + (k & 3u)] = rp[r] + k;
    }
  // CTA split: sort windows, balanced by stored entries
  ws_G_ = (uint32_t)sm_count();
  std::vector<uint32_t> cwin(ws_G_ + 1, 0);
  uint64_t w = 0;
  for (uint32_t c = 1; c < ws_G_; ++c) {
    const uint64_t target = (ws_E_ * c + ws_G_ - 1) / ws_G_;
    while (w < nwin && soff[w * NS] < target) ++w;
    cwin[c] = (uint32_t)w;
  }
  cwin[ws_G_] = (uint32_t)nwin;
  auto up = [&](DevBuf& b, const std::vector<uint32_t>& v) {
    b.alloc(v.size() * 4 + 16);
    F3RG_CUDA(cudaMemcpy(b.get(), v.data(), v.size() * 4, cudaMemcpyHostToDevice));
  };
  up(ws_soff_, soff);
  up(ws_row_, order);
  up(ws_cwin_, cwin);
  DevBuf dsrc;
  up(dsrc, src);
  for (int c = 0; c < 3; ++c) {  // the column stream, encoded per ring class (wsell.cuh)
    ws_enc_[c].alloc(ws_E_ * 4 + 64);
    F3RG_CUDA(cudaMemset(ws_enc_[c].get(), 0, ws_E_ * 4 + 64));
    F3RG_CUDA(launch_ws_encode(Launch{}, dsrc.get<uint32_t>(), ci_.get<uint32_t>(), ws_soff_.get<uint32_t>(),
                               ws_cwin_.get<uint32_t>(), ws_G_, nsl, n_, c, ws_enc_[c].get<uint32_t>()));
  }
  for (int p = 0; p < 3; ++p) {
    ws_val_[p].alloc(ws_E_ * psize(p) + 64);
    F3RG_CUDA(launch_ws_scatter(Launch{}, (int)psize(p), dsrc.get<uint32_t>(), val_[p].get(), ws_val_[p].get(),
                                ws_E_, false));
  }
  F3RG_CUDA(cudaDeviceSynchronize());
}

// Packed windowed layout (wsell_pk.cuh): built on the host (wsell_pk_layout.hpp), the fp16
// values packed in on the device from the fp16 replica, bit for bit.
void DeviceMatrix::build_wsell_pk(const uint32_t* rp, const uint32_t* ci) {
  PkLayoutHost L;
  try {
    pk_build_layout(n_, rp, ci, (uint32_t)sm_count(), L);
  } catch (const std::length_error& e) {
    throw Error(ERR_UNSUPPORTED, e.what());
  }
  pk_E_ = L.E;
  pk_far_ = L.far;
  auto up = [&](DevBuf& b, const void* v, size_t bytes) {
    b.alloc(bytes + 64);
    F3RG_CUDA(cudaMemset(b.get(), 0, bytes + 64));
    if (bytes) F3RG_CUDA(cudaMemcpy(b.get(), v, bytes, cudaMemcpyHostToDevice));
  };
  up(pk_soff_, L.soff.data(), L.soff.size() * 4);
  up(pk_row_, L.row.data(), L.row.size() * 4);
  up(pk_cwin_, L.cwin.data(), L.cwin.size() * 4);
  DevBuf dsrc, dcode;
  up(dsrc, L.src.data(), L.src.size() * 4);
  up(dcode, L.code.data(), L.code.size() * 2);
  pk_words_.alloc(pk_E_ * 4 + 256);
  F3RG_CUDA(cudaMemset(pk_words_.get(), 0, pk_E_ * 4 + 256));
  F3RG_CUDA(launch_pk_pack(Launch{}, dsrc.get<uint32_t>(), dcode.get<uint16_t>(), val_[0].get(),
                           pk_words_.get<uint32_t>(), pk_E_));
  F3RG_CUDA(cudaDeviceSynchronize());
  // class 1 (4-byte rings: the L2 and L1 spmv_dots, an fp16 matrix times an fp32 vector): the code
  // stream as built, every replica's values scattered into the same slots on the device
  // (padding / escape slots: +0)
  PkLayoutHost L1;
  try {
    pk_build_layout(n_, rp, ci, (uint32_t)sm_count(), L1, 1);
  } catch (const std::length_error& e) {
    throw Error(ERR_UNSUPPORTED, e.what());
  }
  pk1_E_ = L1.E;
  up(pk1_soff_, L1.soff.data(), L1.soff.size() * 4);
  up(pk1_row_, L1.row.data(), L1.row.size() * 4);
  up(pk1_cwin_, L1.cwin.data(), L1.cwin.size() * 4);
  up(pk1_code_, L1.code.data(), L1.code.size() * 2);
  DevBuf dsrc1;
  up(dsrc1, L1.src.data(), L1.src.size() * 4);
  for (int p = 0; p < 3; ++p) {
    pk1_val_[p].alloc(pk1_E_ * psize(p) + 256);
    F3RG_CUDA(launch_ws_scatter(Launch{}, (int)psize(p), dsrc1.get<uint32_t>(), val_[p].get(), pk1_val_[p].get(),
                                pk1_E_, false));
  }
  F3RG_CUDA(cudaDeviceSynchronize());
}

double DeviceMatrix::stream_bytes(int pa) const {
  const double n = (double)n_, nnz = (double)nnz_;
  if (pk_E_ && pa == 0) {  // fp16 replica on the packed windowed layout: one 4-byte word per slot + slice tables
    const double nsl = (double)((n_ + kWsSortRows - 1) / kWsSortRows) * (kWsSortRows / 32);
    return (double)pk_E_ * 4.0 + nsl * 32.0 * 4.0 + (nsl + 1.0) * 4.0;
  }
  if (pk1_E_ && pa == 1) {  // fp32 replica on the class-1 code + value streams
    const double nsl = (double)((n_ + kWsSortRows - 1) / kWsSortRows) * (kWsSortRows / 32);
    return (double)pk1_E_ * 6.0 + nsl * 32.0 * 4.0 + (nsl + 1.0) * 4.0;
  }
  if (ws_E_) {  // windowed SELL: chunk-major columns + values (padding included), slice rows and offsets
    const double E = (double)ws_E_, nsl = (double)((n_ + kWsSortRows - 1) / kWsSortRows) * (kWsSortRows / 32);
    return E * (psize(pa) + 4.0) + nsl * 32.0 * 4.0 + (nsl + 1.0) * 4.0;
  }
  return nnz * psize(pa) + (d16() ? 2.0 * nnz + 4.0 * n : 4.0 * nnz) + 4.0 * (n + 1);
}

CsrDev DeviceMatrix::csr_plain() const {
  CsrDev c;
  c.n = n_;
  c.nnz = nnz_;
  c.rp = rp_.get<const uint32_t>();
  c.ci = ci_.get<const uint32_t>();
  for (int p = 0; p < 3; ++p) c.val[p] = val_[p].get();
  c.dcol = dcol_.get<const uint16_t>();
  c.first = first_.get<const uint32_t>();
  c.pk = pk_.get<const uint32_t>();
  return c;
}

CsrDev DeviceMatrix::csr() const {
  if (!perm_.get()) return csr_plain();
  CsrDev c;
  c.n = n_;
  c.nnz = nnz_;
  c.rp = srp_.get<const uint32_t>();
  c.ci = sci_.get<const uint32_t>();
  for (int p = 0; p < 3; ++p) c.val[p] = sval_[p].get();
  c.dcol = sdcol_.get<const uint16_t>();
  c.first = sfirst_.get<const uint32_t>();
  c.pk = spk_.get<const uint32_t>();
  return c;
}

TilesDev DeviceMatrix::tiles(int p) const {
  TilesDev t;
  t.r0 = tr0_[p].get<const uint32_t>();
  t.k0 = tk0_[p].get<const uint32_t>();
  t.ntiles = ntiles_[p];
  t.shape = (uint32_t)shape_;
  t.perm = perm_.get<const uint32_t>();
  t.l2hint = l2hint_;
  if (ws_E_) {
    t.ws_soff = ws_soff_.get<const uint32_t>();
    t.ws_row = ws_row_.get<const uint32_t>();
    for (int c = 0; c < 3; ++c) t.ws_enc[c] = ws_enc_[c].get<const uint32_t>();
    t.ws_val = ws_val_[p].get();
    t.ws_cwin = ws_cwin_.get<const uint32_t>();
    t.ws_G = ws_G_;
    if (pk_E_ && p == 0) {
      t.pk_soff = pk_soff_.get<const uint32_t>();
      t.pk_row = pk_row_.get<const uint32_t>();
      t.pk_words = pk_words_.get<const uint32_t>();
      t.pk_cwin = pk_cwin_.get<const uint32_t>();
    }
    if (pk1_E_) {
      t.pk1_soff = pk1_soff_.get<const uint32_t>();
      t.pk1_row = pk1_row_.get<const uint32_t>();
      t.pk1_cwin = pk1_cwin_.get<const uint32_t>();
      t.pk1_code = pk1_code_.get<const uint16_t>();
      t.pk1_val = pk1_val_[p].get();
    }
  }
  return t;
}

// ---- Solver ---------------------------------------------------------------------------
struct Solver::Level {
  LevelSpec spec;
  int W = 2;   // basis / rhs precision (level 0: fp64, the precision of b)
  int PA = 2;  // matrix replica
  int PZ = 2;  // storage precision of the preconditioned vectors Z (child output, exact)
  int child = 2;  // 0 FGMRES, 1 Richardson, 2 primary preconditioner
  // FGMRES
  DevBuf V, Z, state, H, cs, sn, g, y, scale;
  LevelState* dstate = nullptr;
  LevelState host;
  // Richardson
  DevBuf rs, omegas, wused, wupd, calls, R, Za, Zb, P;
  RichState* drs = nullptr;
  size_t vbytes(uint64_t n) const { return n * psize(W); }
  size_t zbytes(uint64_t n) const { return n * psize(PZ); }
};

struct Solver::ProfRec {
  std::string name;
  double bytes;
  cudaEvent_t e0, e1;
};

Solver::Solver(const Spec& spec, std::shared_ptr<DeviceMatrix> a, int precond_kind, Exchange* ex,
               std::shared_ptr<const DevicePrecond> m)
    : spec_(spec), a_(std::move(a)), ex_(ex), M_(std::move(m)) {
  if (spec_.levels.empty()) throw Error(ERR_SOLVER, "composed solver needs at least one level");
  for (const auto& L : spec_.levels)
    if (L.m < 1) throw Error(ERR_SOLVER, "every level needs m >= 1");
  for (size_t d = 1; d < spec_.levels.size(); ++d) {
    const auto& up = spec_.levels[d - 1];
    const auto& dn = spec_.levels[d];
    if (dn.pa > up.pa || dn.pv > up.pv)
      throw Error(ERR_SOLVER, "precision increases from level " + std::to_string(d) + " to level " +
                                  std::to_string(d + 1) + " (pass allow_precision_increase to permit)");
  }
  if (spec_.levels.size() > 15) throw Error(ERR_SOLVER, "at most 15 nesting levels are supported");
  if (precond_kind != PK_IDENTITY && !has_m())
    throw Error(ERR_UNSUPPORTED, "an ILU(0)/IC(0) primary preconditioner needs its factorisation (f3rg_ilu_factorize)");
  if (M_ && M_->rows() != a_->rows()) throw Error(ERR_DIMENSION, "preconditioner size does not match the matrix");
  if (has_m() && ex_)
    throw Error(ERR_UNSUPPORTED, "row-block partition: a block-Jacobi ILU(0)/IC(0) primary preconditioner is not "
                                 "implemented (its blocks need not align with the ranks)");
  for (size_t d = 0; d + 1 < spec_.levels.size(); ++d)
    if (spec_.levels[d].kind == LK_RICHARDSON)
      throw Error(ERR_UNSUPPORTED, "a Richardson level with an inner solver below it is not implemented on the device");
  for (const auto& L : spec_.levels) {
    if (L.kind == LK_FGMRES && L.m > 1000) throw Error(ERR_UNSUPPORTED, "FGMRES cycle length above 1000");
    // the per-level reset image holds 1000 weights (reset_state)
    if (L.kind == LK_RICHARDSON && L.m > 1000) throw Error(ERR_UNSUPPORTED, "Richardson step count above 1000");
  }
  id_ = spec_.to_string();
  if (const char* e = std::getenv("F3RG_NO_REVERSE")) reverse_off_ = e[0] == '1';
  n_ = a_->rows();
  ld_ = n_;
  if (ex_) {
    const PartPlan& p = ex_->plan();
    if (p.n_own() != n_) throw Error(ERR_DIMENSION, "partition: matrix rows differ from the rank's plan");
    off_ = p.off();
    ld_ = p.ld();
    if (spec_.levels[0].kind != LK_FGMRES)
      throw Error(ERR_UNSUPPORTED, "row-block partition: the outermost level must be FGMRES");
    for (const auto& L : spec_.levels)
      if (L.kind == LK_RICHARDSON && L.m > 2)
        throw Error(ERR_UNSUPPORTED, "row-block partition: Richardson levels with m > 2 are not implemented");
  }
  if (ex_ && seq_reductions())
    throw Error(ERR_UNSUPPORTED, "sequential reductions are a single-rank validation mode");
  build_levels();
  // the in-process transport synchronises ranks on the host between kernels, so it
  // launches eagerly; NCCL exchanges are stream work and go into the graph
  if (lv_.size() >= 2 && lv_[0]->spec.kind == LK_FGMRES && lv_[1]->spec.kind == LK_FGMRES) {
    if (!ex_) {
      inner_exec_ = capture_invocation();
      has_inner_graph_ = true;
    } else if (ex_->capturable()) {
      has_inner_graph_ = true;  // variants captured on first use (invocation_graph)
    }
  }
}

Solver::~Solver() {
  if (inner_exec_) cudaGraphExecDestroy(inner_exec_);
  for (auto& kv : part_exec_) cudaGraphExecDestroy(kv.second);
  if (own_stream_ && !(ex_ && ex_->stream())) cudaStreamDestroy(own_stream_);
  if (info_host_) cudaFreeHost(info_host_);
  if (io_host_) cudaFreeHost(io_host_);
  if (stage_host_) cudaFreeHost(stage_host_);
  if (reset_host_) cudaFreeHost(reset_host_);
  for (auto& p : prof_) {
    cudaEventDestroy(p->e0);
    cudaEventDestroy(p->e1);
  }
}

void Solver::build_levels() {
  const int D = (int)spec_.levels.size();
  if (ex_ && ex_->stream()) own_stream_ = ex_->stream();
  else F3RG_CUDA(cudaStreamCreateWithFlags(&own_stream_, cudaStreamNonBlocking));
  dead_.alloc(16 * sizeof(int));
  cnt_.alloc(CNT_N * sizeof(unsigned long long));
  partials_.alloc((size_t)max_partial_blocks() * 16 * sizeof(double));
  dpartials_.alloc((size_t)max_partial_blocks() * 16 * sizeof(double));  // projection partials (k_spmv_dots)
  counter_.alloc(64);
  bar_.alloc(64);
  info_.alloc(sizeof(StepInfo));
  norm_.alloc(64);
  F3RG_CUDA(cudaMemset(dead_.get(), 0, dead_.bytes()));
  F3RG_CUDA(cudaMemset(cnt_.get(), 0, cnt_.bytes()));
  F3RG_CUDA(cudaMemset(counter_.get(), 0, counter_.bytes()));
  F3RG_CUDA(cudaMemset(bar_.get(), 0, bar_.bytes()));
  F3RG_CUDA(cudaHostAlloc((void**)&info_host_, sizeof(StepInfo), cudaHostAllocDefault));
  F3RG_CUDA(cudaHostAlloc((void**)&stage_host_, 64 * sizeof(double), cudaHostAllocDefault));

  for (int d = 0; d < D; ++d) {
    auto L = std::make_unique<Level>();
    L->spec = spec_.levels[d];
    L->PA = L->spec.pa;
    L->W = d == 0 ? (L->spec.kind == LK_FGMRES ? 2 : L->spec.pv) : L->spec.pv;
    lv_.push_back(std::move(L));
  }
  for (int d = 0; d < D; ++d) {
    Level& L = *lv_[d];
    if (d + 1 < D) {
      L.child = lv_[d + 1]->spec.kind == LK_FGMRES ? 0 : 1;
      L.PZ = lv_[d + 1]->W;  // child output precision (exactly representable)
    } else {
      L.child = 2;
      L.PZ = L.W;
    }
    if (L.spec.kind == LK_FGMRES) {
      const int m = L.spec.m;
      // basis vectors at stride ld_ (ext layout when partitioned: the owned rows at
      // off_, halo entries around them)
      L.V.alloc((size_t)(m + 1) * L.vbytes(ld_) + 16);
      L.Z.alloc((size_t)m * L.zbytes(ld_) + 16);
      if (ex_) {
        F3RG_CUDA(cudaMemset(L.V.get(), 0, L.V.bytes()));
        F3RG_CUDA(cudaMemset(L.Z.get(), 0, L.Z.bytes()));
      }
      L.H.alloc((size_t)(m + 1) * m * 8);
      L.cs.alloc((size_t)m * 8);
      L.sn.alloc((size_t)m * 8);
      L.g.alloc((size_t)(m + 1) * 8);
      L.y.alloc((size_t)m * 8);
      L.scale.alloc((size_t)(m + 1) * 8);
      F3RG_CUDA(cudaMemset(L.H.get(), 0, L.H.bytes()));
      F3RG_CUDA(cudaMemset(L.scale.get(), 0, L.scale.bytes()));
      std::memset(&L.host, 0, sizeof L.host);
      L.host.m = m;
      L.host.div_step = -1;
      L.host.H = L.H.get<double>();
      L.host.cs = L.cs.get<double>();
      L.host.sn = L.sn.get<double>();
      L.host.g = L.g.get<double>();
      L.host.y = L.y.get<double>();
      L.host.scale = L.scale.get<double>();
      L.state.alloc(sizeof(LevelState));
      F3RG_CUDA(cudaMemcpy(L.state.get(), &L.host, sizeof(LevelState), cudaMemcpyHostToDevice));
      L.dstate = L.state.get<LevelState>();
    } else {
      const int m = L.spec.m;
      L.omegas.alloc((size_t)m * 8);
      L.wused.alloc((size_t)m * 8);
      L.wupd.alloc((size_t)m * 4);
      L.calls.alloc(4 * 8);
      L.R.alloc(L.vbytes(ld_) + 16);
      L.Za.alloc(L.vbytes(ld_) + 16);
      if (ex_) {
        F3RG_CUDA(cudaMemset(L.R.get(), 0, L.R.bytes()));
        F3RG_CUDA(cudaMemset(L.Za.get(), 0, L.Za.bytes()));
      }
      // Zb: step ping-pong for m > 2; s = A p of update calls under sequential reductions
      L.Zb.alloc(L.vbytes(n_) + 16);
      if (has_m()) L.P.alloc(L.vbytes(n_) + 16);
      RichState h;
      h.m = m;
      h.cycle = L.spec.cycle;
      h.omegas = L.omegas.get<double>();
      h.wused = L.wused.get<double>();
      h.wupd = L.wupd.get<int>();
      h.calls = L.calls.get<unsigned long long>();
      h.R = L.R.get();
      h.Za = L.Za.get();
      h.Zb = L.Zb.get();
      L.rs.alloc(sizeof(RichState));
      F3RG_CUDA(cudaMemcpy(L.rs.get(), &h, sizeof h, cudaMemcpyHostToDevice));
      L.drs = L.rs.get<RichState>();
    }
  }
  // pinned images of every Richardson level's initial state (reset_state,
  // reset_richardson): 1000 weights + the 4 call counters per level
  F3RG_CUDA(cudaHostAlloc((void**)&reset_host_, (size_t)D * 1024 * sizeof(double), cudaHostAllocDefault));
  for (int d = 0; d < D; ++d) {
    const LevelSpec& S = spec_.levels[d];
    double* img = reset_host_ + (size_t)d * 1024;
    for (int k = 0; k < S.m && k < 1000; ++k) img[k] = S.has_omega ? S.omega : 1.0;
    unsigned long long calls[4] = {1ull, 0ull, 0ull, 0ull};
    std::memcpy(img + 1000, calls, sizeof calls);
  }
  reset_state(own_stream_);
  F3RG_CUDA(cudaStreamSynchronize(own_stream_));
  if (has_m()) {
    // the sweeps' workspace (row values, level counters) and the staging vector
    work_ = M_->make_work();
    work_->prepare(M_->compute_prec(lv_[D - 1]->W), own_stream_);  // before the graph capture
    mbuf_.alloc(n_ * 8 + 16);
    F3RG_CUDA(cudaStreamSynchronize(own_stream_));
  }
  Level& top = *lv_[0];
  xbuf_.alloc(ld_ * psize(top.spec.pv) + 16);
  rbuf_.alloc(n_ * 8 + 16);
  zbuf_.alloc(n_ * 8 + 16);
  if (top.spec.kind == LK_FGMRES) {
    io_.alloc(sizeof(IoSlot));
    F3RG_CUDA(cudaHostAlloc((void**)&io_host_, sizeof(IoSlot) * (size_t)top.spec.m, cudaHostAllocDefault));
  }
}

// stream-ordered copies from the pinned reset image (the solver's streams are
// non-blocking: a legacy-stream cudaMemcpy would not be ordered with them)
void Solver::reset_richardson(int l, cudaStream_t s) {
  Level& L = *lv_[l];
  const double* img = reset_host_ + (size_t)l * 1024;
  F3RG_CUDA(cudaMemcpyAsync(L.omegas.get(), img, (size_t)L.spec.m * 8, cudaMemcpyHostToDevice, s));
  F3RG_CUDA(cudaMemcpyAsync(L.calls.get(), img + 1000, 4 * 8, cudaMemcpyHostToDevice, s));
}

// ---- profiling (eager mode only) ------------------------------------------------------
void Solver::prof_begin(cudaStream_t s) {
  if (!profiling_now_) return;
  auto r = std::make_unique<ProfRec>();
  cudaEventCreate(&r->e0);
  cudaEventCreate(&r->e1);
  cudaEventRecord(r->e0, s);
  prof_.push_back(std::move(r));
}
void Solver::prof_end(cudaStream_t s, const char* name, double bytes) {
  if (!profiling_now_) return;
  auto& r = prof_.back();
  r->name = name;
  r->bytes = bytes;
  cudaEventRecord(r->e1, s);
}

std::vector<Solver::KernelTime> Solver::profile_results() const {
  std::vector<KernelTime> out;
  for (const auto& r : prof_) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r->e0, r->e1);
    auto it = std::find_if(out.begin(), out.end(), [&](const KernelTime& k) { return k.name == r->name; });
    if (it == out.end()) {
      out.push_back({r->name, 0.0, 0, 0.0});
      it = out.end() - 1;
    }
    it->ms += ms;
    it->launches += 1;
    it->bytes += r->bytes;
  }
  return out;
}

#define PROF(name, bytes, call)        \
  do {                                 \
    prof_begin(s);                     \
    F3RG_CUDA(call);                   \
    prof_end(s, name, (double)(bytes)); \
  } while (0)

// bytes one pass over the matrix replica `pa` streams: values, the column stream
// actually in use (u32, or D16 = u16 deltas + u32 first column per row), row_ptr
double Solver::mbytes(int pa) const { return a_->stream_bytes(pa); }

static std::string kname(const char* base, int a, int b, int c) {
  return std::string(base) + "[" + precision_name(a) + "," + precision_name(b) + "," + precision_name(c) + "]";
}

// ---- device level chain ----------------------------------------------------------------
template <class F>
void Solver::reduce(cudaStream_t s, F&& launch) {
  if (!ex_) {
    launch(DistH{});
    return;
  }
  launch(DistH{1, ex_->size(), ex_->loc_buf(), nullptr});
  allgather(s);
  launch(DistH{2, ex_->size(), ex_->loc_buf(), ex_->all_buf()});
  ex_->done_reduce(s);
}

void Solver::enqueue_richardson(int l, int j, void* v_ext, const double* sj, void* z_own, cudaStream_t s) {
  Level& L = *lv_[l - 1];
  Level& R = *lv_[l];
  const uint64_t n = n_;
  int* dead = dead_.get<int>();
  auto* cnt = cnt_.get<unsigned long long>();
  SyncH sync{partials_.get<double>(), counter_.get<unsigned>()};
  const TilesDev T = a_->tiles(R.PA);
  const double bytes = mbytes(R.PA) + (double)n * (psize(L.W) + psize(R.W));
  if (has_m()) {
    enqueue_richardson_m(l, L.W, v_ext, sj, z_own, s);
    return;
  }
  if (!ex_) {
    PROF(kname("richardson", R.PA, R.W, L.W).c_str(), bytes,
         launch_richardson(R.PA, R.W, L.W, Launch{0, s}, a_->csr(), T, v_ext, sj, z_own, n, R.drs, GateH{dead, l}, l,
                           cnt, sync, bar_.get<unsigned>(), bar_.get<unsigned>() + 1, nullptr));
    (void)j;
    return;
  }
  // partitioned: halo of v, the plain sweep, then -- only where the call can be an
  // update call (plan_update_calls) -- the update phases with their exchanges (their
  // kernels still check call_count % c == 0 on the device and return on plain calls)
  halo(v_ext, L.W, s);
  PROF(kname("richardson", R.PA, R.W, L.W).c_str(), bytes,
       launch_richardson(R.PA, R.W, L.W, Launch{0, s}, a_->csr(), T, v_ext, sj, z_own, n, R.drs, GateH{dead, l}, l,
                         cnt, sync, bar_.get<unsigned>(), bar_.get<unsigned>() + 1, nullptr, off_, 1));
  const int m = R.spec.m;
  const bool maybe_update = ++rich_pos_ >= upd_from_;
  for (int k = 0; k < m && maybe_update; ++k) {
    if (k > 0) {
      halo(R.Za.get(), R.W, s);
      F3RG_CUDA(launch_rich_phase(R.PA, R.W, L.W, Launch{0, s}, a_->csr(), T, PH_RESID_H, k, v_ext, sj, off_, z_own, n,
                                  R.drs, R.R.get(), R.Za.get(), GateH{dead, l}, l, cnt, sync, DistH{}));
      halo(R.R.get(), R.W, s);
    }
    F3RG_CUDA(launch_rich_phase(R.PA, R.W, L.W, Launch{0, s}, a_->csr(), T, PH_DOTS_H, k, v_ext, sj, off_, z_own, n,
                                R.drs, R.R.get(), R.Za.get(), GateH{dead, l}, l, cnt, sync,
                                DistH{1, ex_->size(), ex_->loc_buf(), nullptr}));
    allgather(s);
    F3RG_CUDA(launch_rich_phase(R.PA, R.W, L.W, Launch{0, s}, a_->csr(), T, PH_UPDATE_H, k, v_ext, sj, off_, z_own, n,
                                R.drs, R.R.get(), R.Za.get(), GateH{dead, l}, l, cnt, sync,
                                DistH{2, ex_->size(), ex_->loc_buf(), ex_->all_buf()}));
    ex_->done_reduce(s);
  }
  F3RG_CUDA(launch_rich_phase(R.PA, R.W, L.W, Launch{0, s}, a_->csr(), T, PH_BOOK_H, 0, v_ext, sj, off_, z_own, n,
                              R.drs, R.R.get(), R.Za.get(), GateH{dead, l}, l, cnt, sync, DistH{}));
}

void Solver::enqueue_richardson_m(int l, int pv, const void* v, const double* sj, void* out, cudaStream_t s) {
  Level& R = *lv_[l];
  const uint64_t n = n_;
  int* dead = dead_.get<int>();
  auto* cnt = cnt_.get<unsigned long long>();
  SyncH sync{partials_.get<double>(), counter_.get<unsigned>()};
  const TilesDev T = a_->tiles(R.PA);
  const GateH gate{dead, l};
  const int m = R.spec.m;
  const double vb = (double)n * psize(R.W);
  auto phase = [&](int ph, int k) {
    return launch_richm_phase(R.PA, R.W, pv, Launch{0, s}, a_->csr(), T, ph, k, v, sj, out, n, R.drs, R.R.get(),
                              R.P.get(), R.Za.get(), gate, l, cnt, sync);
  };
  PROF("richm_start", (double)n * (psize(pv) + psize(R.W)), phase(RM_START_H, 0));
  for (int k = 0; k < m; ++k) {
    if (k > 0)
      PROF(kname("richm_resid", R.PA, R.W, pv).c_str(), mbytes(R.PA) + (double)n * psize(pv) + 2 * vb,
           phase(RM_RESID_H, k));
    RichEpiH re{R.drs, k, k > 0 ? R.Za.get() : nullptr, k + 1 == m ? out : R.Za.get()};
    prof_begin(s);
    M_->enqueue(*work_, R.R.get(), R.W, R.P.get(), R.W, s, dead, l, &re);
    prof_end(s, M_->config().symmetric ? "precond_ic0" : "precond_ilu0", 0.0);
    PROF(kname("richm_dots", R.PA, R.W, pv).c_str(), 0.0, phase(RM_DOTS_H, k));
    PROF("richm_update", 0.0, phase(RM_UPDATE_H, k));
  }
  PROF("richm_book", 0.0, phase(RM_BOOK_H, 0));
}

void Solver::enqueue_child_step(int l, int j, cudaStream_t s, bool top) {
  Level& L = *lv_[l];
  const uint64_t n = n_;
  // slot j of V / Z in the ext layout (ld_ stride); *_own: its owned rows
  char* vj = L.V.get<char>() + (size_t)j * L.vbytes(ld_);
  char* vj_own = vj + own(L.W);
  const double* sj = L.scale.get<double>() + j;
  char* zj = L.Z.get<char>() + (size_t)j * L.zbytes(ld_);
  char* zj_own = zj + own(L.PZ);
  void* V_own = L.V.get<char>() + own(L.W);
  int* dead = dead_.get<int>();
  auto* cnt = cnt_.get<unsigned long long>();
  SyncH sync{partials_.get<double>(), counter_.get<unsigned>()};
  if (L.child == 0) {
    if (top) {
      plan_update_calls(s);
      io_host_[j] = IoSlot{vj_own, sj, zj_own};
      F3RG_CUDA(cudaMemcpyAsync(io_.get(), &io_host_[j], sizeof(IoSlot), cudaMemcpyHostToDevice, s));
      if (has_inner_graph_ && !profiling_now_) {
        F3RG_CUDA(cudaGraphLaunch(invocation_graph(), s));
      } else {
        enqueue_fgmres(l + 1, nullptr, nullptr, nullptr, io_.get<IoSlot>(), s);
      }
    } else {
      enqueue_fgmres(l + 1, vj_own, sj, zj_own, nullptr, s);
    }
  } else if (L.child == 1) {
    if (top) plan_update_calls(s);
    enqueue_richardson(l + 1, j, vj, sj, zj_own, s);
  } else if (has_m()) {
    // z_j = M (s_j v_j): the normalised basis vector staged at W (counts the
    // PrimarySolver invocation), then the two sweeps (src/nesting.cpp:70-83)
    PROF(kname("copy_scaled", L.W, L.W, L.W).c_str(), 2.0 * n * psize(L.W),
         launch_copy_scaled(L.W, Launch{0, s}, vj_own, sj, mbuf_.get(), n, GateH{dead, l + 1}, cnt));
    prof_begin(s);
    M_->enqueue(*work_, mbuf_.get(), L.W, zj_own, L.PZ, s, dead, l + 1, nullptr);
    prof_end(s, M_->config().symmetric ? "precond_ic0" : "precond_ilu0", 0.0);
  } else {
    PROF(kname("copy_scaled", L.W, L.W, L.W).c_str(), 2.0 * n * psize(L.W),
         launch_copy_scaled(L.W, Launch{0, s}, vj_own, sj, zj_own, n, GateH{dead, l + 1}, cnt));
  }
  halo(zj, L.PZ, s);  // z_j is the SpMV input
  TilesDev T = a_->tiles(L.PA);
  // right after a Richardson pass over the same replica: walk the tiles backwards
  // so the pass starts on the tail end that is still in L2
  if (L.child == 1 && lv_[l + 1]->PA == L.PA && !reverse_off_) T.reverse = 1;
  const int nd = std::min(j + 1, 8);
  // Deferring the projection reduction to k_cgs (every CTA reduces the partials in
  // its prologue) measured no better than k_spmv_dots' own last-CTA tail (both
  // ~6 us on config 2, tools/tile_microbench.cu), so it stays off; the path is kept
  // for the fused-step kernel.
  const int defer = 0;
  int dgrid = 0;
  reduce(s, [&](DistH d) {
    PROF(kname("spmv_dots", L.PA, L.PZ, L.W).c_str(),
         d.mode == 2 ? 0.0 : mbytes(L.PA) + (double)n * (psize(L.PZ) + psize(L.W)) + (double)nd * n * psize(L.W),
         launch_spmv_dots(L.PA, L.PZ, L.W, Launch{0, s}, a_->csr(), T, zj, V_own, ld_, j, L.dstate,
                          GateH{dead, l + 1}, sync, dpartials_.get<double>(), defer, &dgrid, d));
  });
  for (int k0 = 8; k0 <= j; k0 += 8)
    reduce(s, [&](DistH d) {
      PROF(kname("multi_dot", L.W, L.W, L.W).c_str(),
           d.mode == 2 ? 0.0 : (double)n * psize(L.W) * (1 + std::min(8, j + 1 - k0)),
           launch_multi_dot(L.W, Launch{0, s}, V_own, n, j, k0, L.dstate, GateH{dead, l + 1}, sync, ld_, d));
    });
  reduce(s, [&](DistH d) {
    PROF(kname("cgs", L.W, L.W, L.W).c_str(), d.mode == 2 ? 0.0 : (double)n * psize(L.W) * (j + 3),
         launch_cgs(L.W, Launch{0, s}, V_own, n, j, L.dstate, dead, GateH{dead, l + 1}, l, top ? 1 : 0, top ? 1 : 0,
                    top ? info_.get<StepInfo>() : nullptr, sync, defer ? dpartials_.get<double>() : nullptr, dgrid,
                    ld_, d));
  });
}

void Solver::enqueue_fgmres(int l, void* src, const double* src_scale, void* dst, const IoSlot* io, cudaStream_t s) {
  Level& L = *lv_[l];
  Level& P = *lv_[l - 1];
  const uint64_t n = n_;
  int* dead = dead_.get<int>();
  auto* cnt = cnt_.get<unsigned long long>();
  SyncH sync{partials_.get<double>(), counter_.get<unsigned>()};
  reduce(s, [&](DistH d) {
    PROF(kname("level_start", P.W, L.W, L.W).c_str(), d.mode == 2 ? 0.0 : (double)n * (2 * psize(P.W) + psize(L.W)),
         launch_level_start(P.W, L.W, Launch{0, s}, src, src_scale, 0, L.V.get<char>() + own(L.W), n, L.dstate, dead,
                            GateH{dead, l}, l, cnt, sync, io, d));
  });
  for (int j = 0; j < L.spec.m; ++j) enqueue_child_step(l, j, s, false);
  PROF(kname("level_finish", L.PZ, L.W, L.W).c_str(), (double)n * (L.spec.m * psize(L.PZ) + psize(L.W)),
       launch_level_finish(L.PZ, L.W, L.W, Launch{0, s}, L.Z.get<char>() + own(L.PZ), n, L.dstate, dst, 1,
                           GateH{dead, l}, l, cnt, 1, io, ld_));
}

cudaGraphExec_t Solver::capture_invocation() {
  cudaStream_t cs = nullptr;
  F3RG_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaGraph_t graph = nullptr;
  F3RG_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
  try {
    enqueue_fgmres(1, nullptr, nullptr, nullptr, io_.get<IoSlot>(), cs);
  } catch (...) {
    cudaStreamEndCapture(cs, &graph);
    if (graph) cudaGraphDestroy(graph);
    cudaStreamDestroy(cs);
    throw;
  }
  F3RG_CUDA(cudaStreamEndCapture(cs, &graph));
  cudaGraphExec_t exec = nullptr;
  const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  cudaStreamDestroy(cs);
  F3RG_CUDA(e);
  return exec;
}

cudaGraphExec_t Solver::invocation_graph() {
  if (!ex_) return inner_exec_;
  auto it = part_exec_.find(upd_from_);
  if (it != part_exec_.end()) return it->second;
  // every rank reaches here with the same upd_from_ (replicated device state), so
  // the ranks capture matching collective sequences
  cudaGraphExec_t g = capture_invocation();
  part_exec_[upd_from_] = g;
  return g;
}

void Solver::plan_update_calls(cudaStream_t s) {
  rich_pos_ = 0;  // positions count the calls below this outer step
  int rl = -1;
  for (int d = 1; d < (int)lv_.size(); ++d)
    if (lv_[d]->spec.kind == LK_RICHARDSON) rl = d;
  if (!ex_ || rl < 0 || has_m()) {
    upd_from_ = 1;
    return;
  }
  const unsigned long long c = lv_[rl]->spec.cycle;
  if (c == 0) {  // never updates
    upd_from_ = 1 << 30;
    return;
  }
  auto* h = reinterpret_cast<unsigned long long*>(stage_host_ + 48);
  F3RG_CUDA(cudaMemcpyAsync(h, lv_[rl]->calls.get(), 8, cudaMemcpyDeviceToHost, s));
  F3RG_CUDA(cudaStreamSynchronize(s));
  // the invocation's calls are call_count C, C+1, ...; the first update is the first
  // multiple of c. Early stops inside the invocation only delay calls, never bring an
  // update earlier, so every position from there on keeps its update phases.
  const unsigned long long C = *h;
  upd_from_ = (int)((c - C % c) % c) + 1;
}

double Solver::read_double(const double* dev, cudaStream_t s) {
  F3RG_CUDA(cudaMemcpyAsync(stage_host_, dev, 8, cudaMemcpyDeviceToHost, s));
  F3RG_CUDA(cudaStreamSynchronize(s));
  return stage_host_[0];
}

double Solver::true_rel(const double* b, double bnorm, cudaStream_t s) {
  Level& top = *lv_[0];
  SyncH sync{partials_.get<double>(), counter_.get<unsigned>()};
  halo(xbuf_.get(), top.spec.pv, s);
  reduce(s, [&](DistH d) {
    PROF(kname("residual", 2, top.spec.pv, 2).c_str(), d.mode == 2 ? 0.0 : mbytes(2) + (double)n_ * (psize(top.spec.pv) + 16),
         launch_residual(2, top.spec.pv, 2, Launch{0, s}, a_->csr(), a_->tiles(2), xbuf_.get(), b, rbuf_.get(),
                         nullptr, norm_.get<double>(), sync, d));
  });
  return read_double(norm_.get<double>(), s) / bnorm;
}

Report Solver::run(const double* b, double* x_out, const RunOptions& opts, cudaStream_t stream) {
  const auto t0 = std::chrono::steady_clock::now();
  cudaStream_t s = stream ? stream : own_stream_;
  profiling_now_ = profile_;
  if (profiling_now_) {
    for (auto& p : prof_) {
      cudaEventDestroy(p->e0);
      cudaEventDestroy(p->e1);
    }
    prof_.clear();
  }
  Report rep;
  rep.solver_id = id_;
  n_halo_ = n_reduce_ = 0;
  const int D = (int)lv_.size();
  F3RG_CUDA(cudaMemsetAsync(cnt_.get(), 0, cnt_.bytes(), s));
  F3RG_CUDA(cudaMemsetAsync(dead_.get(), 0, dead_.bytes(), s));
  F3RG_CUDA(cudaMemsetAsync(xbuf_.get(), 0, xbuf_.bytes(), s));
  SyncH sync{partials_.get<double>(), counter_.get<unsigned>()};
  reduce(s, [&](DistH d) {
    PROF("norm2[b]", d.mode == 2 ? 0.0 : 8.0 * n_, launch_norm2(2, Launch{0, s}, b, n_, norm_.get<double>(), sync, d));
  });
  const double bnorm = read_double(norm_.get<double>(), s);
  if (bnorm == 0.0) {
    rep.converged = true;
    rep.residual_history.push_back(0.0);
  } else {
    rep.residual_history.push_back(1.0);
    rep = lv_[0]->spec.kind == LK_FGMRES ? run_fgmres_top(b, opts, s, bnorm, std::move(rep))
                                         : run_richardson_top(b, opts, s, bnorm, std::move(rep));
    rep.final_true_residual = true_rel(b, bnorm, s);
  }
  // counters (src/nesting.cpp:347-351)
  unsigned long long cnt[CNT_N];
  F3RG_CUDA(cudaMemcpyAsync(stage_host_, cnt_.get(), sizeof cnt, cudaMemcpyDeviceToHost, s));
  F3RG_CUDA(cudaStreamSynchronize(s));
  std::memcpy(cnt, stage_host_, sizeof cnt);
  rep.precond_invocations = cnt[CNT_PRECOND];
  rep.level_iterations.assign((size_t)D, 0ull);
  for (int d = 1; d < D; ++d) rep.level_iterations[d] = cnt[CNT_IT + d];
  rep.level_iterations[0] = lv_[0]->spec.kind == LK_FGMRES ? rep.outer_iterations : cnt[CNT_IT + 0];
  rep.omegas_final = innermost_omegas();
  if (x_out) F3RG_CUDA(launch_copy(lv_[0]->spec.pv, 2, Launch{0, s}, xbuf_.get<char>() + own(lv_[0]->spec.pv), x_out, n_));
  F3RG_CUDA(cudaStreamSynchronize(s));
  profiling_now_ = false;
  rep.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return rep;
}

Report Solver::run_fgmres_top(const double* b, const RunOptions& opts, cudaStream_t s, double bnorm, Report rep) {
  Level& top = *lv_[0];
  const int m1 = top.spec.m;
  const uint64_t n = n_;
  const double nnz = (double)a_->nnz();
  int* dead = dead_.get<int>();
  auto* cnt = cnt_.get<unsigned long long>();
  SyncH sync{partials_.get<double>(), counter_.get<unsigned>()};
  int executions = 0;
  const int max_exec = 1 + std::max(0, opts.max_outer_restarts);
  const bool restarted = opts.restart_budget > 0;  // fgmres_restarted (src/fgmres.cpp:163-222)
  for (;;) {
    // one precondition call per Arnoldi step of the outermost level
    const unsigned long long remaining =
        restarted ? opts.restart_budget - rep.outer_iterations : opts.max_outer_total - rep.outer_iterations;
    if (remaining == 0) {
      rep.flag = "capped";
      break;
    }
    const int len = (int)std::min<unsigned long long>((unsigned long long)m1, remaining);
    // ---- one cycle (src/fgmres.cpp:21-148) ----
    const bool first = executions == 0;
    if (first) {  // r = b
      reduce(s, [&](DistH d) {
        PROF("level_start[f64,f64,f64]", d.mode == 2 ? 0.0 : 16.0 * n,
             launch_level_start(2, 2, Launch{0, s}, const_cast<double*>(b), nullptr, 0, top.V.get<char>() + own(2), n,
                                top.dstate, dead, GateH{dead, 0}, 0, cnt, sync, nullptr, d));
      });
    } else {  // r = b - A x
      halo(xbuf_.get(), top.spec.pv, s);
      reduce(s, [&](DistH d) {
        PROF(kname("residual", top.PA, top.spec.pv, 2).c_str(),
             d.mode == 2 ? 0.0 : mbytes(top.PA) + (double)n * (psize(top.spec.pv) + 16),
             launch_residual(top.PA, top.spec.pv, 2, Launch{0, s}, a_->csr(), a_->tiles(top.PA), xbuf_.get(), b,
                             top.V.get<char>() + own(2), top.dstate, nullptr, sync, d));
      });
    }
    F3RG_CUDA(cudaMemsetAsync(dead, 0, sizeof(int), s));
    F3RG_CUDA(cudaMemcpyAsync(stage_host_, top.dstate, sizeof(LevelState), cudaMemcpyDeviceToHost, s));
    F3RG_CUDA(cudaStreamSynchronize(s));
    LevelState st;
    std::memcpy(&st, stage_host_, sizeof st);
    const double beta = st.beta;
    // cycle-level outcome
    int iterations = 0;
    bool diverged = false, happy = false;
    int div_step = -1;
    double residual_norm = beta;
    if (beta == 0.0 || !std::isfinite(beta)) {
      diverged = !std::isfinite(beta);
      div_step = diverged ? 0 : -1;
    } else {
      // x_is_zero: bnorm = beta; else norm2(converted(b, W)) = ||b|| at fp64
      F3RG_CUDA(launch_set_outer(Launch{0, s}, top.dstate, first ? beta : bnorm, opts.tol));
      for (int j = 0; j < len; ++j) {
        enqueue_child_step(0, j, s, true);
        F3RG_CUDA(cudaMemcpyAsync(info_host_, info_.get(), sizeof(StepInfo), cudaMemcpyDeviceToHost, s));
        F3RG_CUDA(cudaStreamSynchronize(s));
        const StepInfo inf = *info_host_;
        if (inf.diverged) {
          diverged = true;
          div_step = inf.div_step;
          break;
        }
        iterations = inf.k;
        residual_norm = inf.estimate;
        rep.residual_history.push_back(inf.estimate / bnorm);
        if (inf.happy) {
          happy = true;
          break;
        }
        if (inf.tol_hit) break;
      }
      (void)happy;
      // back-substitution + x += Z y
      PROF(kname("level_finish", top.PZ, top.W, top.spec.pv).c_str(),
           (double)n * (iterations * psize(top.PZ) + 2 * psize(top.spec.pv)),
           launch_level_finish(top.PZ, top.W, top.spec.pv, Launch{0, s}, top.Z.get<char>() + own(top.PZ), n, top.dstate,
                               xbuf_.get<char>() + own(top.spec.pv), 0, GateH{dead, 0}, 0, cnt, 0, nullptr, ld_));
    }
    rep.outer_iterations += (unsigned long long)iterations;
    if (diverged) {
      rep.flag = (restarted ? "divergence at step " : "divergence at outer step ") + std::to_string(div_step);
      break;
    }
    if (residual_norm < opts.tol * bnorm && true_rel(b, bnorm, s) < opts.tol) {
      rep.converged = true;
      break;
    }
    ++executions;
    if (restarted ? rep.outer_iterations >= opts.restart_budget : executions >= max_exec) {
      rep.flag = "capped";
      break;
    }
    if (opts.reset_richardson_on_restart)
      for (int d = 1; d < (int)lv_.size(); ++d)
        if (lv_[d]->spec.kind == LK_RICHARDSON) reset_richardson(d, s);
  }
  return rep;
}

Report Solver::run_richardson_top(const double* b, const RunOptions& opts, cudaStream_t s, double bnorm, Report rep) {
  Level& top = *lv_[0];
  const int pv = top.spec.pv;
  const uint64_t n = n_;
  const double nnz = (double)a_->nnz();
  int* dead = dead_.get<int>();
  auto* cnt = cnt_.get<unsigned long long>();
  SyncH sync{partials_.get<double>(), counter_.get<unsigned>()};
  F3RG_CUDA(launch_copy(2, pv, Launch{0, s}, b, rbuf_.get(), n));  // r = b
  for (;;) {
    if (rep.outer_iterations >= opts.max_outer_total) {
      rep.flag = "capped";
      break;
    }
    if (has_m()) {
      enqueue_richardson_m(0, pv, rbuf_.get(), nullptr, zbuf_.get(), s);
    } else {
      PROF(kname("richardson", top.PA, pv, pv).c_str(), mbytes(top.PA) + 2.0 * n * psize(pv),
           launch_richardson(top.PA, pv, pv, Launch{0, s}, a_->csr(), a_->tiles(top.PA), rbuf_.get(), nullptr,
                             zbuf_.get(), n, top.drs, GateH{dead, 0}, 0, cnt, sync, bar_.get<unsigned>(),
                             bar_.get<unsigned>() + 1, nullptr));
    }
    F3RG_CUDA(launch_axpy(pv, pv, Launch{0, s}, 1.0, zbuf_.get(), xbuf_.get(), n));
    rep.outer_iterations += 1;
    PROF(kname("residual", top.PA, pv, pv).c_str(), mbytes(top.PA) + (double)n * (2 * psize(pv) + 8),
         launch_residual(top.PA, pv, pv, Launch{0, s}, a_->csr(), a_->tiles(top.PA), xbuf_.get(), b, rbuf_.get(),
                         nullptr, norm_.get<double>(), sync));
    const double rel = read_double(norm_.get<double>(), s) / bnorm;
    rep.residual_history.push_back(rel);
    if (!std::isfinite(rel)) {
      rep.flag = "divergence";
      break;
    }
    if (rel < opts.tol && true_rel(b, bnorm, s) < opts.tol) {
      rep.converged = true;
      break;
    }
  }
  return rep;
}

void Solver::reset_state(cudaStream_t stream) {
  cudaStream_t s = stream ? stream : own_stream_;
  for (int d = 0; d < (int)lv_.size(); ++d)
    if (lv_[d]->spec.kind == LK_RICHARDSON) reset_richardson(d, s);
}

std::vector<double> Solver::innermost_omegas() {
  for (int d = (int)lv_.size() - 1; d >= 1; --d) {
    Level& L = *lv_[d];
    if (L.spec.kind == LK_RICHARDSON) {
      std::vector<double> w((size_t)L.spec.m);
      F3RG_CUDA(cudaDeviceSynchronize());
      F3RG_CUDA(cudaMemcpy(w.data(), L.omegas.get(), w.size() * 8, cudaMemcpyDeviceToHost));
      return w;
    }
  }
  return {};
}

std::vector<unsigned long long> Solver::level_invocations() {
  unsigned long long cnt[CNT_N];
  F3RG_CUDA(cudaDeviceSynchronize());
  F3RG_CUDA(cudaMemcpy(cnt, cnt_.get(), sizeof cnt, cudaMemcpyDeviceToHost));
  return std::vector<unsigned long long>(cnt + CNT_INV, cnt + CNT_INV + lv_.size());
}

}  // namespace f3rg

// ---- fp64 CG / BiCGStab (reference src/cg.cpp:22-171) ---------------------------------
namespace f3rg {

KrylovSolver::KrylovSolver(std::shared_ptr<DeviceMatrix> a, std::shared_ptr<const DevicePrecond> m)
    : a_(std::move(a)), n_(a_->rows()), M_(std::move(m)) {
  if (M_ && M_->rows() != n_) throw Error(ERR_DIMENSION, "preconditioner size does not match the matrix");
  F3RG_CUDA(cudaStreamCreateWithFlags(&own_, cudaStreamNonBlocking));
  for (DevBuf* b : {&x_, &r_, &p_, &q_, &s_, &t_, &rhat_, &tmp_}) b->alloc(n_ * 8 + 16);
  state_.alloc(sizeof(KState));
  partials_.alloc((size_t)max_partial_blocks() * 16 * sizeof(double));
  counter_.alloc(64);
  norm_.alloc(64);
  F3RG_CUDA(cudaMemset(counter_.get(), 0, counter_.bytes()));
  F3RG_CUDA(cudaHostAlloc((void**)&stage_host_, 4096, cudaHostAllocDefault));
  if (has_m()) {  // z = M r (CG), phat / shat (BiCGStab: phat in z_)
    z_.alloc(n_ * 8 + 16);
    shat_.alloc(n_ * 8 + 16);
    work_ = M_->make_work();
    work_->prepare(M_->compute_prec(2), own_);
    F3RG_CUDA(cudaStreamSynchronize(own_));
  }
}

KrylovSolver::~KrylovSolver() {
  if (stage_host_) cudaFreeHost(stage_host_);
  if (own_) cudaStreamDestroy(own_);
}

double KrylovSolver::true_rel(const double* b, double bnorm, cudaStream_t s) {
  // src/cg.cpp:10-17: spmv(a, x, ax); add_scaled(b, -1, ax, r); norm2(r) / bnorm
  SyncH sync{partials_.get<double>(), counter_.get<unsigned>()};
  F3RG_CUDA(launch_residual(2, 2, 2, Launch{0, s}, a_->csr(), a_->tiles(2), x_.get(), b, tmp_.get(), nullptr,
                            norm_.get<double>(), sync));
  F3RG_CUDA(cudaMemcpyAsync(stage_host_, norm_.get(), 8, cudaMemcpyDeviceToHost, s));
  F3RG_CUDA(cudaStreamSynchronize(s));
  return stage_host_[0] / bnorm;
}

Report KrylovSolver::solve(int which, const double* b, double* x_out, double tol, unsigned long long max_precond,
                           cudaStream_t stream) {
  if (which != 0 && which != 1) throw Error(ERR_SOLVER, "krylov solve: which must be 0 (cg) or 1 (bicgstab)");
  const auto t0 = std::chrono::steady_clock::now();
  cudaStream_t s = stream ? stream : own_;
  const uint64_t n = n_;
  Report rep;
  rep.solver_id = which == 0 ? "cg" : "bicgstab";
  SyncH sync{partials_.get<double>(), counter_.get<unsigned>()};
  auto read = [&](const void* dev, size_t bytes) {
    F3RG_CUDA(cudaMemcpyAsync(stage_host_, dev, bytes, cudaMemcpyDeviceToHost, s));
    F3RG_CUDA(cudaStreamSynchronize(s));
  };
  F3RG_CUDA(launch_norm2(2, Launch{0, s}, b, n, norm_.get<double>(), sync));
  read(norm_.get(), 8);
  const double bnorm = stage_host_[0];
  rep.residual_history.push_back(bnorm == 0.0 ? 0.0 : 1.0);
  if (bnorm == 0.0) {
    rep.converged = true;
    if (x_out) F3RG_CUDA(cudaMemsetAsync(x_out, 0, n * 8, s));
    F3RG_CUDA(cudaStreamSynchronize(s));
    return rep;
  }
  const unsigned long long cap = max_precond + 2;
  if (hist_.bytes() < cap * 8) hist_.alloc(cap * 8);
  F3RG_CUDA(cudaMemsetAsync(x_.get(), 0, n * 8, s));
  F3RG_CUDA(cudaMemcpyAsync(r_.get(), b, n * 8, cudaMemcpyDeviceToDevice, s));  // x0 = 0: r = b
  KState h{};
  h.bnorm = bnorm;
  h.tol = tol;
  h.rho = h.alpha = h.omega = 1.0;
  h.max_precond = max_precond;
  h.hist_cap = cap;
  h.hist = hist_.get<double>();
  if (which == 0) {  // z = M r, p = z, rz = (r, z) (src/cg.cpp:41-44)
    const void* z0 = r_.get();
    if (has_m()) {
      M_->enqueue(*work_, r_.get(), 2, z_.get(), 2, s, nullptr, 0, nullptr);
      z0 = z_.get();
    }
    F3RG_CUDA(cudaMemcpyAsync(p_.get(), z0, n * 8, cudaMemcpyDeviceToDevice, s));
    F3RG_CUDA(launch_dot(2, 2, 2, Launch{0, s}, r_.get(), z0, n, norm_.get<double>(), sync));
    read(norm_.get(), 8);
    h.rz = stage_host_[0];
    h.precond = 1;
  } else {  // rhat = r; p = v = 0
    F3RG_CUDA(cudaMemcpyAsync(rhat_.get(), r_.get(), n * 8, cudaMemcpyDeviceToDevice, s));
    F3RG_CUDA(cudaMemsetAsync(p_.get(), 0, n * 8, s));
    F3RG_CUDA(cudaMemsetAsync(q_.get(), 0, n * 8, s));
  }
  F3RG_CUDA(cudaMemcpyAsync(state_.get(), &h, sizeof h, cudaMemcpyHostToDevice, s));
  KState* S = state_.get<KState>();
  const CsrDev A = a_->csr();
  const TilesDev T = a_->tiles(2);
  double* x = x_.get<double>();
  double* r = r_.get<double>();
  double* p = p_.get<double>();
  double* v = q_.get<double>();  // CG: q; BiCGStab: v
  // M's sweeps are gated on the solver's stop flag like every kernel of a batch
  const int* stop = reinterpret_cast<const int*>(reinterpret_cast<const char*>(S) + offsetof(KState, stop));
  auto apply_m = [&](const double* in, double* out) {
    M_->enqueue(*work_, in, 2, out, 2, s, stop, 1, nullptr);
  };
  // CG after its checks: z = M r, rz', beta (src/cg.cpp:69-72), then p = z + beta p
  auto cg_next = [&]() {
    if (has_m()) {
      apply_m(r, z_.get<double>());
      F3RG_CUDA(launch_cg_rz(Launch{0, s}, r, z_.get<double>(), n, S, sync));
      F3RG_CUDA(launch_cg_p(Launch{0, s}, p, z_.get<double>(), n, S));
    } else {
      F3RG_CUDA(launch_cg_next(Launch{0, s}, S));
      F3RG_CUDA(launch_cg_p(Launch{0, s}, p, r, n, S));
    }
  };
  double* phat = has_m() ? z_.get<double>() : p;
  double* shat = has_m() ? shat_.get<double>() : s_.get<double>();
  const int batch = 8;  // iterations enqueued per host synchronisation
  for (;;) {
    for (int k = 0; k < batch; ++k) {
      if (which == 0) {
        F3RG_CUDA(launch_cg_spmv(Launch{0, s}, A, T, p, v, S, sync));
        F3RG_CUDA(launch_cg_update(Launch{0, s}, x, r, p, v, n, S, sync));
        cg_next();
      } else {
        F3RG_CUDA(launch_bi_rho(Launch{0, s}, rhat_.get<double>(), r, n, S, sync));
        F3RG_CUDA(launch_bi_p(Launch{0, s}, p, v, r, n, S));
        if (has_m()) apply_m(p, phat);  // phat = M p (src/cg.cpp:120)
        F3RG_CUDA(launch_bi_v(Launch{0, s}, A, T, phat, v, rhat_.get<double>(), S, sync));
        F3RG_CUDA(launch_bi_s(Launch{0, s}, s_.get<double>(), r, v, n, S));
        if (has_m()) apply_m(s_.get<double>(), shat);  // shat = M s (:131)
        F3RG_CUDA(launch_bi_t(Launch{0, s}, A, T, s_.get<double>(), shat, t_.get<double>(), S, sync));
        F3RG_CUDA(launch_bi_update(Launch{0, s}, x, r, phat, s_.get<double>(), shat, t_.get<double>(), n, S, sync));
      }
    }
    read(S, sizeof h);
    std::memcpy(&h, stage_host_, sizeof h);
    if (h.stop == KS_RUN) continue;
    if (h.stop == KS_TOL) {
      const double tr = true_rel(b, bnorm, s);
      if (tr < tol) {
        rep.converged = true;
        rep.final_true_residual = tr;
        break;
      }
      // the reference carries on with the iteration (cap test, then CG's z/rz/beta/p)
      F3RG_CUDA(launch_krylov_resume(Launch{0, s}, S));
      if (which == 0) cg_next();
      continue;
    }
    if (h.stop == KS_INDEFINITE) throw Error(ERR_SOLVER, "cg: indefinite operator detected");
    rep.flag = h.stop == KS_CAPPED ? "capped" : "breakdown";
    rep.final_true_residual = true_rel(b, bnorm, s);
    break;
  }
  rep.outer_iterations = h.it;
  rep.precond_invocations = h.precond;
  if (h.it > 0) {
    std::vector<double> hist(h.it);
    F3RG_CUDA(cudaMemcpyAsync(hist.data(), hist_.get<double>() + 1, h.it * 8, cudaMemcpyDeviceToHost, s));
    F3RG_CUDA(cudaStreamSynchronize(s));
    rep.residual_history.insert(rep.residual_history.end(), hist.begin(), hist.end());
  }
  if (x_out) F3RG_CUDA(cudaMemcpyAsync(x_out, x, n * 8, cudaMemcpyDeviceToDevice, s));
  F3RG_CUDA(cudaStreamSynchronize(s));
  rep.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return rep;
}

}  // namespace f3rg
