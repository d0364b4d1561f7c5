// precond.cpp -- block-Jacobi ILU(0)/IC(0): host factorisation (restating reference
// src/ilu.cpp:38-185), the level-set sweep schedules and the device apply.
#include "precond.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>

#include "engine.hpp"
#include "state.hpp"

namespace f3rg {

// ---- host factorisation -------------------------------------------------------------
namespace {

double round_to(int p, double x) {  // demote(x, p): one RNE rounding (precision.hpp:64-70)
  if (p == 2) return x;
  if (p == 1) return (double)(float)x;
  // binary16 from binary64 with one rounding (half.hpp:54-80): round the significand
  // to 11 bits at the binary16 exponent, subnormals on the fixed 2^-24 grid
  if (std::isnan(x) || std::isinf(x)) return x;
  const double a = std::fabs(x);
  if (a == 0.0) return x;
  int e;
  std::frexp(a, &e);  // a = f * 2^e, f in [0.5, 1)
  int q = e - 11;     // quantum exponent for 11 significant bits
  if (q < -24) q = -24;
  const double scaled = std::ldexp(a, -q);
  double r = std::nearbyint(scaled);  // RNE (default rounding mode)
  double out = std::ldexp(r, q);
  if (out >= 65520.0) out = INFINITY;  // 65504 + half an ulp rounds to inf
  else if (out > 65504.0) out = 65504.0;
  return std::copysign(out, x);
}

std::string block_row(const char* what, uint64_t b, uint64_t i) {
  return std::string(what) + " in block " + std::to_string(b) + ", row " + std::to_string(i);
}

// one diagonal block [lo, hi) of the working copy, factorised in place; returns ""
// or the reference's error message
struct Work {
  std::vector<uint32_t> ptr, idx, diag;
  std::vector<double> val;
};

std::string factor_block(Work& w, uint64_t b, uint32_t lo, uint32_t hi, bool symmetric) {
  if (!symmetric) {
    // ILU(0), IKJ order (src/ilu.cpp:88-106)
    std::vector<int64_t> pos(hi - lo, -1);
    for (uint32_t i = lo; i < hi; ++i) {
      for (uint32_t k = w.ptr[i]; k < w.ptr[i + 1]; ++k) pos[w.idx[k] - lo] = k;
      for (uint32_t k = w.ptr[i]; k < w.ptr[i + 1] && w.idx[k] < i; ++k) {
        const uint32_t r = w.idx[k];
        w.val[k] = w.val[k] / w.val[w.diag[r]];
        const double f = w.val[k];
        for (uint32_t q = w.diag[r] + 1; q < w.ptr[r + 1]; ++q) {
          const int64_t p = pos[w.idx[q] - lo];
          if (p >= 0) w.val[p] = w.val[p] - f * w.val[q];
        }
      }
      for (uint32_t k = w.ptr[i]; k < w.ptr[i + 1]; ++k) pos[w.idx[k] - lo] = -1;
      if (w.val[w.diag[i]] == 0.0) return block_row("zero pivot", b, i);
    }
  } else {
    // IC(0) on the lower pattern (src/ilu.cpp:108-137)
    for (uint32_t i = lo; i < hi; ++i) {
      for (uint32_t k = w.ptr[i]; k < w.ptr[i + 1]; ++k) {
        const uint32_t j = w.idx[k];
        double s = w.val[k];
        uint32_t a = w.ptr[i], c = w.ptr[j];
        while (a < w.ptr[i + 1] && c < w.ptr[j + 1] && w.idx[a] < j && w.idx[c] < j) {
          if (w.idx[a] == w.idx[c]) s = s - w.val[a++] * w.val[c++];
          else if (w.idx[a] < w.idx[c]) ++a;
          else ++c;
        }
        if (j < i) {
          w.val[k] = s / w.val[w.diag[j]];
        } else {
          if (s <= 0.0) return block_row("non-positive pivot", b, i);
          w.val[k] = std::sqrt(s);
        }
      }
    }
  }
  return "";
}

}  // namespace

HostFactors factorize_host(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals,
                           const IluConfig& cfg) {
  if (cfg.nblocks == 0 || cfg.nblocks > n) throw Error(ERR_FACTORIZATION, "nblocks must be in [1, n]");
  if (!(cfg.alpha > 0.0)) throw Error(ERR_FACTORIZATION, "alpha must be positive");
  HostFactors f;
  f.n = n;
  f.cfg = cfg;
  f.block_ranges.assign(cfg.nblocks + 1, 0);
  for (uint64_t b = 0; b < cfg.nblocks; ++b)
    f.block_ranges[b + 1] = f.block_ranges[b] + (uint32_t)(n / cfg.nblocks + (b < n % cfg.nblocks ? 1 : 0));

  // working copy restricted to the diagonal blocks (IC: lower triangle), diagonal
  // scaled by alpha (src/ilu.cpp:62-86)
  Work w;
  w.ptr.assign(n + 1, 0);
  w.diag.assign(n, 0);
  w.idx.reserve(rp[n]);
  w.val.reserve(rp[n]);
  for (uint64_t b = 0; b < cfg.nblocks; ++b) {
    const uint32_t lo = f.block_ranges[b], hi = f.block_ranges[b + 1];
    for (uint32_t i = lo; i < hi; ++i) {
      bool diag = false;
      for (uint32_t k = rp[i]; k < rp[i + 1]; ++k) {
        const uint32_t j = ci[k];
        if (j < lo || j >= hi || (cfg.symmetric && j > i)) continue;
        if (j == i) {
          diag = true;
          w.diag[i] = (uint32_t)w.idx.size();
          w.val.push_back(vals[k] * cfg.alpha);
        } else {
          w.val.push_back(vals[k]);
        }
        w.idx.push_back(j);
      }
      if (!diag) throw Error(ERR_FACTORIZATION, block_row("missing diagonal entry", b, i));
      w.ptr[i + 1] = (uint32_t)w.idx.size();
    }
  }
  // the blocks are independent: factorise them on parallel host threads; the first
  // failing block in block order reports (the reference's sequential loop would
  // have stopped there)
  std::vector<std::string> errs(cfg.nblocks);
  {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const uint64_t nt = std::min<uint64_t>(cfg.nblocks, hw);
    std::vector<std::thread> th;
    for (uint64_t t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        for (uint64_t b = t; b < cfg.nblocks; b += nt)
          errs[b] = factor_block(w, b, f.block_ranges[b], f.block_ranges[b + 1], cfg.symmetric);
      });
    for (auto& x : th) x.join();
  }
  for (const auto& e : errs)
    if (!e.empty()) throw Error(ERR_FACTORIZATION, e);

  // split into the stored factors (src/ilu.cpp:140-157)
  f.lp.assign(n + 1, 0);
  f.up.assign(n + 1, 0);
  for (uint64_t i = 0; i < n; ++i) {
    for (uint32_t k = w.ptr[i]; k < w.ptr[i + 1]; ++k) {
      if (cfg.symmetric || w.idx[k] < i) {
        f.li.push_back(w.idx[k]);
        f.lv.push_back(w.val[k]);
      } else {
        f.ui.push_back(w.idx[k]);
        f.uv.push_back(w.val[k]);
      }
    }
    f.lp[i + 1] = (uint32_t)f.li.size();
    f.up[i + 1] = (uint32_t)f.ui.size();
  }
  // every pivot must survive the cast to the apply precision (:159-172)
  for (uint64_t i = 0; i < n; ++i) {
    const double d = cfg.symmetric ? f.lv[f.lp[i + 1] - 1] : f.uv[f.up[i]];
    const double c = round_to(cfg.prec, d);
    if (c == 0.0 || !std::isfinite(c)) {
      uint64_t b = 0;
      while (f.block_ranges[b + 1] <= i) ++b;
      throw Error(ERR_FACTORIZATION, std::string("casting factors to ") + precision_name(cfg.prec) +
                                         " lost the diagonal of row " + std::to_string(i) + "; block " +
                                         std::to_string(b));
    }
  }
  for (auto& v : f.lv) v = round_to(cfg.prec, v);
  for (auto& v : f.uv) v = round_to(cfg.prec, v);
  return f;
}

// ---- device schedule --------------------------------------------------------------
static void* upload(const void* src, size_t bytes) {
  void* p = nullptr;
  F3RG_CUDA(cudaMalloc(&p, bytes ? bytes : 16));
  if (bytes) F3RG_CUDA(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice));
  return p;
}

static size_t psz(int p) { return p == 0 ? 2 : p == 1 ? 4 : 8; }

// factor values -> device array at precision p (exact: they are representable)
static void* upload_values(const std::vector<double>& v, int p) {
  void* d64 = upload(v.data(), v.size() * 8);
  if (p == 2) return d64;
  void* out = nullptr;
  F3RG_CUDA(cudaMalloc(&out, v.size() * psz(p) + 16));
  if (!v.empty()) F3RG_CUDA(launch_copy(2, p, Launch{}, d64, out, v.size()));
  F3RG_CUDA(cudaDeviceSynchronize());
  cudaFree(d64);
  return out;
}

void DevicePrecond::build_sweep(int k, const HostFactors& f) {
  const uint64_t n = f.n;
  const bool sym = f.cfg.symmetric;
  // row lists: entries in the reference's accumulation order, plus the divisor
  std::vector<uint32_t> rptr(n + 1, 0), ridx;
  std::vector<double> rval, rdg;
  const bool has_dg = k == 1 || sym;
  if (has_dg) rdg.assign(n, 0.0);
  if (k == 0) {
    for (uint64_t i = 0; i < n; ++i) {
      const uint32_t end = sym ? f.lp[i + 1] - 1 : f.lp[i + 1];
      for (uint32_t q = f.lp[i]; q < end; ++q) {
        ridx.push_back(f.li[q]);
        rval.push_back(f.lv[q]);
      }
      if (sym) rdg[i] = f.lv[f.lp[i + 1] - 1];
      rptr[i + 1] = (uint32_t)ridx.size();
    }
  } else if (!sym) {
    for (uint64_t i = 0; i < n; ++i) {
      for (uint32_t q = f.up[i] + 1; q < f.up[i + 1]; ++q) {
        ridx.push_back(f.ui[q]);
        rval.push_back(f.uv[q]);
      }
      rdg[i] = f.uv[f.up[i]];
      rptr[i + 1] = (uint32_t)ridx.size();
    }
  } else {
    // IC backward: column j of L below the diagonal, rows DESCENDING (the order the
    // reference's scatter loop, src/ilu.cpp:237-244, updates work[j] in)
    std::vector<uint32_t> cnt(n + 1, 0);
    for (uint64_t i = 0; i < n; ++i) {
      for (uint32_t q = f.lp[i]; q + 1 < f.lp[i + 1]; ++q) ++cnt[f.li[q] + 1];
      rdg[i] = f.lv[f.lp[i + 1] - 1];
    }
    for (uint64_t j = 0; j < n; ++j) rptr[j + 1] = rptr[j] + cnt[j + 1];
    ridx.resize(rptr[n]);
    rval.resize(rptr[n]);
    std::vector<uint32_t> fill(rptr.begin(), rptr.end() - 1);
    for (uint64_t i = n; i-- > 0;)
      for (uint32_t q = f.lp[i]; q + 1 < f.lp[i + 1]; ++q) {
        const uint32_t j = f.li[q];
        ridx[fill[j]] = (uint32_t)i;
        rval[fill[j]++] = f.lv[q];
      }
  }
  // dependency levels (forward: rows ascending; backward: descending)
  std::vector<uint32_t> lev(n, 0);
  uint32_t nlev = 0;
  for (uint64_t t = 0; t < n; ++t) {
    const uint64_t i = k == 0 ? t : n - 1 - t;
    uint32_t l = 0;
    for (uint32_t q = rptr[i]; q < rptr[i + 1]; ++q) l = std::max(l, lev[ridx[q]] + 1);
    lev[i] = l;
    nlev = std::max(nlev, l + 1);
  }
  // rows grouped by level (ascending row id inside a level), each level in slices of 32
  std::vector<uint32_t> lstart(nlev + 1, 0);
  for (uint64_t i = 0; i < n; ++i) ++lstart[lev[i] + 1];
  for (uint32_t l = 0; l < nlev; ++l) lstart[l + 1] += lstart[l];
  std::vector<uint32_t> order(n), lfill(lstart.begin(), lstart.end() - 1);
  for (uint64_t i = 0; i < n; ++i) order[lfill[lev[i]]++] = (uint32_t)i;
  uint64_t ns = 0;
  for (uint32_t l = 0; l < nlev; ++l) ns += (lstart[l + 1] - lstart[l] + 31) / 32;
  std::vector<uint32_t> rows(ns * 32, 0xffffffffu), cnt(ns * 32, 0), soff(ns + 1, 0);
  std::vector<double> dg(has_dg ? ns * 32 : 0, 1.0);
  uint64_t s = 0;
  for (uint32_t l = 0; l < nlev; ++l)
    for (uint32_t a = lstart[l]; a < lstart[l + 1]; a += 32, ++s) {
      uint32_t width = 0;
      for (uint32_t t = 0; t < 32 && a + t < lstart[l + 1]; ++t) {
        const uint32_t i = order[a + t];
        rows[s * 32 + t] = i;
        cnt[s * 32 + t] = rptr[i + 1] - rptr[i];
        width = std::max(width, cnt[s * 32 + t]);
        if (has_dg) dg[s * 32 + t] = rdg[i];
      }
      soff[s + 1] = soff[s] + width;
    }
  std::vector<uint32_t> col((uint64_t)soff[ns] * 32, 0);
  std::vector<double> val((uint64_t)soff[ns] * 32, 0.0);
  for (uint64_t q = 0; q < ns; ++q)
    for (uint32_t t = 0; t < 32; ++t) {
      const uint32_t i = rows[q * 32 + t];
      if (i == 0xffffffffu) continue;
      for (uint32_t e = 0; e < cnt[q * 32 + t]; ++e) {
        const uint64_t at = ((uint64_t)soff[q] + e) * 32 + t;
        col[at] = ridx[rptr[i] + e];
        val[at] = rval[rptr[i] + e];
      }
    }
  std::vector<uint32_t> slvl(ns), lns(nlev, 0);
  for (uint64_t q = 0, l = 0; l < nlev; ++l)
    for (uint32_t a = lstart[l]; a < lstart[l + 1]; a += 32, ++q) slvl[q] = (uint32_t)l, ++lns[l];
  nslices_[k] = (uint32_t)ns;
  nlev_[k] = nlev;
  buf_[k][6] = upload(slvl.data(), slvl.size() * 4);
  buf_[k][7] = upload(lns.data(), lns.size() * 4);
  buf_[k][0] = upload(rows.data(), rows.size() * 4);
  buf_[k][1] = upload(cnt.data(), cnt.size() * 4);
  buf_[k][2] = upload(soff.data(), soff.size() * 4);
  buf_[k][3] = upload(col.data(), col.size() * 4);
  buf_[k][4] = upload_values(val, cfg_.prec);
  buf_[k][5] = has_dg ? upload_values(dg, cfg_.prec) : nullptr;
}

DevicePrecond::DevicePrecond(uint64_t n) : identity_(true), n_(n) {}

DevicePrecond::DevicePrecond(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals,
                             const IluConfig& cfg)
    : identity_(false), n_(n), cfg_(cfg) {
  validate_csr(n, rp, ci);
  const HostFactors f = factorize_host(n, rp, ci, vals, cfg);
  block_ranges_ = f.block_ranges;
  try {
    build_sweep(0, f);
    build_sweep(1, f);
    own_ = make_work();
  } catch (...) {
    for (auto& b : buf_)
      for (auto& p : b)
        if (p) cudaFree(p), p = nullptr;
    throw;
  }
}

DevicePrecond::~DevicePrecond() {
  for (auto& b : buf_)
    for (auto& p : b)
      if (p) cudaFree(p);
}

SweepDev DevicePrecond::sweep(int k) const {
  SweepDev d;
  d.nslices = nslices_[k];
  d.nlevels = nlev_[k];
  d.rows = static_cast<const uint32_t*>(buf_[k][0]);
  d.cnt = static_cast<const uint32_t*>(buf_[k][1]);
  d.soff = static_cast<const uint32_t*>(buf_[k][2]);
  d.col = static_cast<const uint32_t*>(buf_[k][3]);
  d.val = buf_[k][4];
  d.dg = buf_[k][5];
  d.lvl = static_cast<const uint32_t*>(buf_[k][6]);
  d.lvl_ns = static_cast<const uint32_t*>(buf_[k][7]);
  static const uint32_t sleep_ns = [] {
    const char* e = std::getenv("F3RG_SWEEP_SLEEP");
    return e ? (uint32_t)std::atoi(e) : 512u;
  }();
  static const uint32_t ahead = [] {
    const char* e = std::getenv("F3RG_SWEEP_AHEAD");
    return e ? (uint32_t)std::atoi(e) : 4u;
  }();
  static const uint32_t poll = [] {
    const char* e = std::getenv("F3RG_SWEEP_POLL");
    return e ? (uint32_t)std::atoi(e) : 0u;
  }();
  d.poll = poll;
  d.sleep_ns = sleep_ns;
  d.ahead = ahead;
  d.n = n_;
  return d;
}

std::unique_ptr<SweepWork> DevicePrecond::make_work() const {
  return std::make_unique<SweepWork>(n_, nlev_[0], nlev_[1]);
}

void DevicePrecond::enqueue(SweepWork& w, const void* r, int pr, void* z, int pz, cudaStream_t s,
                            const int* gate_dead, int gate_n, const RichEpiH* re) const {
  if (identity_) {  // IdentityPrecond::apply = copy_into (src/ilu.cpp:33-36)
    F3RG_CUDA(launch_copy(pr, pz, Launch{0, s}, r, z, n_));
    return;
  }
  const int c = compute_prec(pr);
  w.prepare(c, s);
  const GateH gate{gate_dead, gate_n};
  F3RG_CUDA(launch_sweep_fwd(cfg_.prec, pr, Launch{0, s}, sweep(0), r, w.cells[0], w.level_done[0], w.ctl, gate));
  F3RG_CUDA(launch_sweep_bwd(cfg_.prec, c, pz, Launch{0, s}, sweep(1), w.cells[0], w.cells[1], z, w.level_done[1],
                             w.ctl + 1, gate, re ? *re : RichEpiH{}));
}

void DevicePrecond::apply(const void* r, int pr, void* z, int pz, cudaStream_t s) const {
  if (identity_) {
    F3RG_CUDA(launch_copy(pr, pz, Launch{0, s}, r, z, n_));
    return;
  }
  enqueue(*own_, r, pr, z, pz, s, nullptr, 0, nullptr);
}

// ---- per-user workspace -------------------------------------------------------------
SweepWork::SweepWork(uint64_t n, uint32_t nlev_fwd, uint32_t nlev_bwd) : n_(n) {
  const uint32_t nl[2] = {nlev_fwd, nlev_bwd};
  for (int k = 0; k < 2; ++k) {
    F3RG_CUDA(cudaMalloc(&cells[k], n * 12 + 64));
    F3RG_CUDA(cudaMemset(cells[k], 0, n * 12 + 64));
    F3RG_CUDA(cudaMalloc((void**)&level_done[k], (size_t)nl[k] * 4 + 64));
    F3RG_CUDA(cudaMemset(level_done[k], 0, (size_t)nl[k] * 4 + 64));
  }
  F3RG_CUDA(cudaMalloc((void**)&ctl, 2 * sizeof(SweepCtl)));
  F3RG_CUDA(cudaMemset(ctl, 0, 2 * sizeof(SweepCtl)));
  // test hook: start the epoch tags just below a 2^16 multiple (the tags skip those,
  // the launch counter does not), as a long-lived solver reaches after 65k applies
  if (const char* e = std::getenv("F3RG_SWEEP_EPOCH0")) {
    SweepCtl h[2] = {};
    h[0].epoch = h[1].epoch = (unsigned)std::strtoul(e, nullptr, 10);
    F3RG_CUDA(cudaMemcpy(ctl, h, sizeof h, cudaMemcpyHostToDevice));
  }
}

void SweepWork::prepare(int c, cudaStream_t s) {
  if (c == last_c_) return;
  if (last_c_ >= 0)
    for (auto& p : cells) F3RG_CUDA(cudaMemsetAsync(p, 0, n_ * 12 + 64, s));
  last_c_ = c;
}

SweepWork::~SweepWork() {
  for (int k = 0; k < 2; ++k) {
    if (cells[k]) cudaFree(cells[k]);
    if (level_done[k]) cudaFree(level_done[k]);
  }
  if (ctl) cudaFree(ctl);
}

}  // namespace f3rg
