// capi.cpp -- the C ABI of include/f3rg.h over the engine (engine.hpp).
// Exceptions never cross the boundary: each entry point maps f3rg::Error codes
// (1:1 with the reference's exception classes) to its return value and records
// the message for f3rg_last_error().
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/f3rg.h"
#include "engine.hpp"
#include "wsell_pk_layout.hpp"
#include "launch.hpp"

using namespace f3rg;

struct f3rg_matrix {
  std::shared_ptr<DeviceMatrix> m;
};

struct f3rg_solver {
  std::unique_ptr<Solver> s;
  Report last;
  DevBuf b, x;  // device staging of the host-buffer entry, allocated on first use
};

struct f3rg_richardson {
  std::shared_ptr<DeviceMatrix> a;
  int prec = 0, m = 1;
  DevBuf state, omegas, wused, wupd, calls, R, Za, Zb, P, dead, cnt, partials, counter, bar;
  std::shared_ptr<const DevicePrecond> M;  // null: identity
  std::unique_ptr<SweepWork> work;
};

struct f3rg_precond {
  std::shared_ptr<DevicePrecond> p;
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return F3RG_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return F3RG_EINTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return F3RG_EINTERNAL;
  }
}

void check_prec(int p) {
  if (p < 0 || p > 2) throw Error(ERR_DIMENSION, "precision tag must be 0 (f16), 1 (f32) or 2 (f64)");
}

cudaStream_t as_stream(uintptr_t s) { return reinterpret_cast<cudaStream_t>(s); }

void fill_report(const Report& r, f3rg_report* out) {
  if (!out) return;
  std::memset(out, 0, sizeof *out);
  out->converged = r.converged;
  out->outer_iterations = r.outer_iterations;
  out->precond_invocations = r.precond_invocations;
  out->final_true_residual = r.final_true_residual;
  out->wall_seconds = r.wall_seconds;
  out->n_history = r.residual_history.size();
  out->n_levels = r.level_iterations.size();
  out->n_omegas = r.omegas_final.size();
  std::strncpy(out->flag, r.flag.c_str(), sizeof out->flag - 1);
}

RunOptions to_opts(const f3rg_run_options* o) {
  RunOptions r;
  if (o) {
    r.tol = o->tol;
    r.max_outer_restarts = o->max_outer_restarts;
    r.max_outer_total = o->max_outer_total;
    r.reset_richardson_on_restart = o->reset_richardson_on_restart != 0;
  }
  return r;
}

// scratch for scalar results of kernel-level reductions
struct Scratch {
  DevBuf partials, counter, out;
  Scratch() {
    partials.alloc((size_t)max_partial_blocks() * 16 * sizeof(double));
    counter.alloc(64);
    out.alloc(64);
    F3RG_CUDA(cudaMemset(counter.get(), 0, 64));
  }
};
Scratch& scratch() {
  thread_local Scratch s;
  return s;
}

}  // namespace

extern "C" {

const char* f3rg_last_error(void) { return g_err.c_str(); }
const char* f3rg_version(void) { return "f3rg 0.1 (sm_100a)"; }

int f3rg_set_seq_reductions(int on) {
  const int old = f3rg::seq_reductions();
  f3rg::set_seq_reductions(on);
  return old;
}

void f3rg_default_run_options(f3rg_run_options* o) {
  o->tol = 1e-8;
  o->max_outer_restarts = 3;
  o->max_outer_total = 300;
  o->reset_richardson_on_restart = 0;
}

int f3rg_matrix_create(f3rg_matrix** out, const f3rg_csr* a) {
  return guarded([&] {
    if (!out || !a) throw Error(ERR_DIMENSION, "null argument");
    auto h = std::make_unique<f3rg_matrix>();
    h->m = std::make_shared<DeviceMatrix>(a->n, a->row_ptr, a->col_idx, a->values);
    *out = h.release();
  });
}

void f3rg_matrix_destroy(f3rg_matrix* a) { delete a; }
uint64_t f3rg_matrix_rows(const f3rg_matrix* a) { return a ? a->m->rows() : 0; }
uint64_t f3rg_matrix_nnz(const f3rg_matrix* a) { return a ? a->m->nnz() : 0; }
uint64_t f3rg_matrix_stream_bytes(const f3rg_matrix* a, int prec) {
  return a && prec >= 0 && prec <= 2 ? (uint64_t)a->m->stream_bytes(prec) : 0;
}

int f3rg_matrix_engine(const f3rg_matrix* a) { return a ? a->m->shape() : -1; }

int f3rg_wsell_pk_selfcheck(uint64_t n, const uint32_t* row_ptr, const uint32_t* col_idx, uint32_t ctas,
                            uint64_t* stats) {
  return guarded([&] {
   for (int cl = 1; cl >= 0; --cl) {  // both geometries; the statistics are the packed fp16 stream's (class 0)
    const int64_t kPkTW = pk_tw(cl), kPkW = pk_w(cl), kPkRing = pk_ring(cl);
    const uint32_t kPkLimit = pk_pad(cl), kPkPad = pk_pad(cl), kPkEsc = pk_esc(cl);
    PkLayoutHost L;
    try {
      pk_build_layout(n, row_ptr, col_idx, ctas, L, cl);
    } catch (const std::length_error& e) {
      throw Error(ERR_UNSUPPORTED, e.what());
    }
    const uint64_t nsl = L.soff.size() - 1;
    uint64_t pads = 0, far = 0, rows_seen = 0;
    auto fail = [&](uint64_t r, const char* what) {
      throw Error(ERR_DIMENSION, "packed layout: row " + std::to_string(r) + ": " + what);
    };
    if (L.cwin.size() != (size_t)ctas + 1 || L.cwin.front() != 0 ||
        (uint64_t)L.cwin.back() * kWsSortRows < n)
      fail(0, "CTA split does not cover the rows");
    for (uint64_t s = 0; s < nsl; ++s) {
      const uint32_t width = (L.soff[s + 1] - L.soff[s]) / 32u;
      if ((L.soff[s] & 127u) || (width & 3u)) fail(0, "slice offset / width not chunk aligned");
      for (uint32_t l = 0; l < 32; ++l) {
        const uint32_t r = L.row[s * 32 + l];
        auto at = [&](uint32_t pos) { return (uint64_t)L.soff[s] + (uint64_t)(pos >> 2) * 128u + l * 4u + (pos & 3u); };
        if (r == kWsPadIdx) {
          for (uint32_t pos = 0; pos < width; ++pos)
            if (L.code[at(pos)] != kPkPad || L.src[at(pos)] != kWsPadIdx) fail(s, "a lane without a row holds an entry");
          continue;
        }
        if (r / kWsSortRows != s / (kWsSortRows / 32)) fail(r, "row outside its sort window");
        ++rows_seen;
        const int64_t B = (int64_t)(r / (uint64_t)kPkTW) * kPkTW;
        const int64_t lo = std::max<int64_t>(0, B - kPkW), hi = std::min<int64_t>((int64_t)n, B + kPkTW + kPkW);
        uint32_t k = row_ptr[r], pos = 0;
        while (pos < width) {
          const uint32_t code = L.code[at(pos)], src = L.src[at(pos)];
          if (code >= kPkEsc) {  // escape pair: this slot carries no value, the next one the low half and the entry
            if ((pos & 3u) == 3u) fail(r, "escape pair split over two quads");
            if (src != kWsPadIdx) fail(r, "escape slot carries a value");
            if (k >= row_ptr[r + 1]) fail(r, "more entries than the CSR row");
            const uint32_t c = ((code - kPkEsc) << 16) | L.code[at(pos + 1)];
            if (c != col_idx[k] || L.src[at(pos + 1)] != k) fail(r, "far column / entry mismatch");
            const bool inband = (int64_t)c >= lo && (int64_t)c < hi && c % (uint32_t)kPkRing < kPkLimit;
            if (inband) fail(r, "band entry stored as far");
            ++far, ++k, pos += 2;
          } else if (src == kWsPadIdx) {
            if (code != kPkPad) fail(r, "padding slot with a ring code");
            ++pads, ++pos;
          } else {
            if (k >= row_ptr[r + 1] || src != k) fail(r, "entry out of order");
            const uint32_t c = col_idx[k];
            if (code != c % (uint32_t)kPkRing || code >= kPkLimit || (int64_t)c < lo || (int64_t)c >= hi)
              fail(r, "ring slot does not match the column / band");
            ++k, ++pos;
          }
        }
        if (k != row_ptr[r + 1]) fail(r, "row not fully stored");
      }
    }
    if (rows_seen != n) fail(0, "not every row is stored exactly once");
    if (far != L.far) fail(0, "far count mismatch");
    if (stats) stats[0] = L.E, stats[1] = far, stats[2] = nsl, stats[3] = pads;
   }
  });
}

int f3rg_matrix_values(const f3rg_matrix* a, int prec, double* out_host) {
  return guarded([&] {
    check_prec(prec);
    const uint64_t nnz = a->m->nnz();
    DevBuf tmp(nnz * 8 + 16);
    F3RG_CUDA(launch_copy(prec, 2, Launch{}, a->m->values(prec), tmp.get(), nnz));
    F3RG_CUDA(cudaMemcpy(out_host, tmp.get(), nnz * 8, cudaMemcpyDeviceToHost));
  });
}

int f3rg_spec_canonical(const char* spec, char* out, size_t cap) {
  return guarded([&] {
    const std::string s = parse_spec(spec ? spec : "").to_string();
    if (cap) {
      std::strncpy(out, s.c_str(), cap - 1);
      out[cap - 1] = 0;
    }
  });
}

// ---- primary preconditioner (include/f3r/ilu.hpp) ------------------------------------
namespace {
IluConfig to_cfg(const f3rg_ilu_config* c) {
  if (!c) throw Error(ERR_DIMENSION, "null ilu config");
  check_prec(c->apply_precision);
  IluConfig k;
  k.nblocks = c->nblocks;
  k.alpha = c->alpha;
  k.symmetric = c->symmetric != 0;
  k.prec = c->apply_precision;
  return k;
}

// the fp64 CSR of a device matrix, back in host memory (setup only)
void download(const DeviceMatrix& m, std::vector<uint32_t>& rp, std::vector<uint32_t>& ci, std::vector<double>& v) {
  const CsrDev c = m.csr_plain();
  rp.resize(m.rows() + 1);
  ci.resize(m.nnz());
  v.resize(m.nnz());
  F3RG_CUDA(cudaDeviceSynchronize());
  F3RG_CUDA(cudaMemcpy(rp.data(), c.rp, rp.size() * 4, cudaMemcpyDeviceToHost));
  if (m.nnz()) {
    F3RG_CUDA(cudaMemcpy(ci.data(), c.ci, ci.size() * 4, cudaMemcpyDeviceToHost));
    F3RG_CUDA(cudaMemcpy(v.data(), c.val[2], v.size() * 8, cudaMemcpyDeviceToHost));
  }
}
}  // namespace

int f3rg_ilu_factorize(f3rg_precond** out, const f3rg_csr* a, const f3rg_ilu_config* cfg) {
  return guarded([&] {
    if (!out || !a) throw Error(ERR_DIMENSION, "null argument");
    auto h = std::make_unique<f3rg_precond>();
    h->p = std::make_shared<DevicePrecond>(a->n, a->row_ptr, a->col_idx, a->values, to_cfg(cfg));
    *out = h.release();
  });
}

int f3rg_precond_identity(f3rg_precond** out, uint64_t n) {
  return guarded([&] {
    if (!out) throw Error(ERR_DIMENSION, "null argument");
    auto h = std::make_unique<f3rg_precond>();
    h->p = std::make_shared<DevicePrecond>(n);
    *out = h.release();
  });
}

void f3rg_precond_destroy(f3rg_precond* m) { delete m; }
uint64_t f3rg_precond_rows(const f3rg_precond* m) { return m ? m->p->rows() : 0; }

int f3rg_precond_info(const f3rg_precond* m, f3rg_ilu_config* cfg, uint32_t* levels, uint32_t* ranges,
                      uint64_t cap) {
  return guarded([&] {
    if (!m) throw Error(ERR_DIMENSION, "null argument");
    const DevicePrecond& p = *m->p;
    if (cfg) {
      cfg->nblocks = p.identity() ? 0 : p.config().nblocks;
      cfg->alpha = p.config().alpha;
      cfg->symmetric = p.config().symmetric;
      cfg->apply_precision = p.config().prec;
    }
    if (levels) levels[0] = p.nlevels(0), levels[1] = p.nlevels(1);
    const auto& br = p.block_ranges();
    for (uint64_t i = 0; ranges && i < br.size() && i < cap; ++i) ranges[i] = br[i];
  });
}

int f3rg_precond_apply(const f3rg_precond* m, const void* r, int pr, void* z, int pz, uintptr_t stream) {
  return guarded([&] {
    if (!m) throw Error(ERR_DIMENSION, "null argument");
    check_prec(pr), check_prec(pz);
    m->p->apply(r, pr, z, pz, as_stream(stream));
  });
}

int f3rg_ilu_factorize_host(const f3rg_csr* a, const f3rg_ilu_config* cfg, uint64_t* nnz_lower, uint64_t* nnz_upper,
                            uint32_t* lp, uint32_t* li, double* lv, uint32_t* up, uint32_t* ui, double* uv) {
  return guarded([&] {
    if (!a) throw Error(ERR_DIMENSION, "null argument");
    validate_csr(a->n, a->row_ptr, a->col_idx);
    const HostFactors f = factorize_host(a->n, a->row_ptr, a->col_idx, a->values, to_cfg(cfg));
    if (nnz_lower) *nnz_lower = f.li.size();
    if (nnz_upper) *nnz_upper = f.ui.size();
    if (lp) std::memcpy(lp, f.lp.data(), f.lp.size() * 4);
    if (li) std::memcpy(li, f.li.data(), f.li.size() * 4);
    if (lv) std::memcpy(lv, f.lv.data(), f.lv.size() * 8);
    if (up) std::memcpy(up, f.up.data(), f.up.size() * 4);
    if (ui) std::memcpy(ui, f.ui.data(), f.ui.size() * 4);
    if (uv) std::memcpy(uv, f.uv.data(), f.uv.size() * 8);
  });
}

int f3rg_solver_create_m(f3rg_solver** out, const f3rg_matrix* a, const char* spec, const f3rg_precond* m) {
  return guarded([&] {
    if (!out || !a || !spec || !m) throw Error(ERR_DIMENSION, "null argument");
    auto h = std::make_unique<f3rg_solver>();
    const int kind = m->p->identity() ? PK_IDENTITY : m->p->config().symmetric ? PK_IC0 : PK_ILU0;
    h->s = std::make_unique<Solver>(parse_spec(spec), a->m, kind, nullptr, m->p);
    *out = h.release();
  });
}

int f3rg_solver_create(f3rg_solver** out, const f3rg_matrix* a, const char* spec, int precond_kind) {
  return guarded([&] {
    if (!out || !a || !spec) throw Error(ERR_DIMENSION, "null argument");
    auto h = std::make_unique<f3rg_solver>();
    const Spec sp = parse_spec(spec);
    std::shared_ptr<const DevicePrecond> M;
    if (precond_kind == PK_ILU0 || precond_kind == PK_IC0) {
      // factorise from the spec terminal with the reference bench's defaults
      // (blocks 4, alpha 1, fp64 apply; src/bench.cpp:160-177, include/f3r/bench.hpp:31-34)
      IluConfig cfg;
      cfg.symmetric = precond_kind == PK_IC0;
      cfg.nblocks = sp.has_precond && sp.precond.has_blocks ? sp.precond.blocks : 4;
      cfg.alpha = sp.has_precond && sp.precond.has_alpha ? sp.precond.alpha : 1.0;
      cfg.prec = sp.has_precond && sp.precond.has_prec ? sp.precond.prec : 2;
      std::vector<uint32_t> rp, ci;
      std::vector<double> v;
      download(*a->m, rp, ci, v);
      M = std::make_shared<DevicePrecond>(a->m->rows(), rp.data(), ci.data(), v.data(), cfg);
    } else if (precond_kind != PK_IDENTITY) {
      throw Error(ERR_DIMENSION, "precond_kind must be F3RG_PRECOND_ILU0, _IC0 or _IDENTITY");
    }
    h->s = std::make_unique<Solver>(sp, a->m, precond_kind, nullptr, M);
    *out = h.release();
  });
}

void f3rg_solver_destroy(f3rg_solver* s) { delete s; }
const char* f3rg_solver_id(const f3rg_solver* s) { return s ? s->s->id().c_str() : ""; }

int f3rg_solve_device(f3rg_solver* s, const double* b, double* x, const f3rg_run_options* o, f3rg_report* rep,
                      uintptr_t stream) {
  return guarded([&] {
    s->last = s->s->run(b, x, to_opts(o), as_stream(stream));
    fill_report(s->last, rep);
  });
}

int f3rg_solve(f3rg_solver* s, const double* b_host, double* x_host, const f3rg_run_options* o, f3rg_report* rep) {
  return guarded([&] {
    const uint64_t n = s->s->rows();
    if (!s->b.get()) s->b.alloc(n * 8 + 16), s->x.alloc(n * 8 + 16);
    cudaStream_t st = s->s->stream();
    F3RG_CUDA(cudaMemcpyAsync(s->b.get(), b_host, n * 8, cudaMemcpyHostToDevice, st));
    s->last = s->s->run(s->b.get<double>(), x_host ? s->x.get<double>() : nullptr, to_opts(o), st);
    if (x_host) {
      F3RG_CUDA(cudaMemcpyAsync(x_host, s->x.get(), n * 8, cudaMemcpyDeviceToHost, st));
      F3RG_CUDA(cudaStreamSynchronize(st));
    }
    fill_report(s->last, rep);
  });
}

int f3rg_solver_reset_state(f3rg_solver* s, uintptr_t stream) {
  return guarded([&] { s->s->reset_state(as_stream(stream)); });
}

int f3rg_solver_history(const f3rg_solver* s, double* out, uint64_t cap) {
  const auto& h = s->last.residual_history;
  for (uint64_t i = 0; i < h.size() && i < cap; ++i) out[i] = h[i];
  return F3RG_OK;
}

int f3rg_solver_level_iterations(const f3rg_solver* s, uint64_t* out, uint64_t cap) {
  const auto& h = s->last.level_iterations;
  for (uint64_t i = 0; i < h.size() && i < cap; ++i) out[i] = h[i];
  return F3RG_OK;
}

int f3rg_solver_omegas(f3rg_solver* s, double* out, uint64_t cap) {
  return guarded([&] {
    const auto w = s->s->innermost_omegas();
    for (uint64_t i = 0; i < w.size() && i < cap; ++i) out[i] = w[i];
  });
}

uint64_t f3rg_solver_omega_count(const f3rg_solver* s) {
  uint64_t n = 0;
  guarded([&] { n = s->s->innermost_omegas().size(); });
  return n;
}

int f3rg_solver_collectives(const f3rg_solver* s, uint64_t* halos, uint64_t* reductions) {
  if (!s || !halos || !reductions) return F3RG_EDIMENSION;
  *halos = s->s->halos();
  *reductions = s->s->reductions();
  return F3RG_OK;
}

int f3rg_solver_set_profile(f3rg_solver* s, int on) {
  s->s->set_profile(on != 0);
  return F3RG_OK;
}

int f3rg_solver_profile_entry(const f3rg_solver* s, uint64_t i, char* name, size_t cap, double* ms,
                              uint64_t* launches, double* bytes) {
  return guarded([&] {
    const auto r = s->s->profile_results();
    if (i >= r.size()) throw Error(ERR_DIMENSION, "profile entry out of range");
    if (cap) {
      std::strncpy(name, r[i].name.c_str(), cap - 1);
      name[cap - 1] = 0;
    }
    *ms = r[i].ms;
    *launches = r[i].launches;
    *bytes = r[i].bytes;
  });
}

// ---- kernel-level -----------------------------------------------------------------
int f3rg_spmv(const f3rg_matrix* a, int pa, const void* x, int px, void* y, int py, uintptr_t stream) {
  return guarded([&] {
    check_prec(pa), check_prec(px), check_prec(py);
    F3RG_CUDA(launch_spmv(pa, px, py, Launch{0, as_stream(stream)}, a->m->csr(), a->m->tiles(pa), x, y));
  });
}

int f3rg_dot(const void* x, int px, const void* y, int py, uint64_t n, int floor_p, double* out, uintptr_t stream) {
  return guarded([&] {
    check_prec(px), check_prec(py), check_prec(floor_p);
    auto& sc = scratch();
    cudaStream_t s = as_stream(stream);
    F3RG_CUDA(launch_dot(px, py, floor_p, Launch{0, s}, x, y, n, sc.out.get<double>(),
                         SyncH{sc.partials.get<double>(), sc.counter.get<unsigned>()}));
    F3RG_CUDA(cudaMemcpyAsync(out, sc.out.get(), 8, cudaMemcpyDeviceToHost, s));
    F3RG_CUDA(cudaStreamSynchronize(s));
  });
}

int f3rg_norm2(const void* x, int px, uint64_t n, double* out, uintptr_t stream) {
  return guarded([&] {
    check_prec(px);
    auto& sc = scratch();
    cudaStream_t s = as_stream(stream);
    F3RG_CUDA(launch_norm2(px, Launch{0, s}, x, n, sc.out.get<double>(),
                           SyncH{sc.partials.get<double>(), sc.counter.get<unsigned>()}));
    F3RG_CUDA(cudaMemcpyAsync(out, sc.out.get(), 8, cudaMemcpyDeviceToHost, s));
    F3RG_CUDA(cudaStreamSynchronize(s));
  });
}

int f3rg_axpy(double alpha, const void* x, int px, void* y, int py, uint64_t n, uintptr_t stream) {
  return guarded([&] {
    check_prec(px), check_prec(py);
    F3RG_CUDA(launch_axpy(px, py, Launch{0, as_stream(stream)}, alpha, x, y, n));
  });
}

int f3rg_add_scaled(const void* x, int px, double alpha, const void* y, int py, void* out, int po, uint64_t n,
                    uintptr_t stream) {
  return guarded([&] {
    check_prec(px), check_prec(py), check_prec(po);
    F3RG_CUDA(launch_add_scaled(px, py, po, Launch{0, as_stream(stream)}, x, alpha, y, out, n));
  });
}

int f3rg_copy(const void* x, int px, void* y, int py, uint64_t n, uintptr_t stream) {
  return guarded([&] {
    check_prec(px), check_prec(py);
    F3RG_CUDA(launch_copy(px, py, Launch{0, as_stream(stream)}, x, y, n));
  });
}

int f3rg_scale(double alpha, void* x, int px, uint64_t n, uintptr_t stream) {
  return guarded([&] {
    check_prec(px);
    F3RG_CUDA(launch_scale(px, Launch{0, as_stream(stream)}, alpha, x, n));
  });
}

int f3rg_fill(void* x, int px, uint64_t n, double value, uintptr_t stream) {
  return guarded([&] {
    check_prec(px);
    F3RG_CUDA(launch_fill(px, Launch{0, as_stream(stream)}, x, n, value));
  });
}

// ---- Richardson ---------------------------------------------------------------------
int f3rg_richardson_create(f3rg_richardson** out, const f3rg_matrix* a, int prec, int m, uint64_t cycle) {
  return guarded([&] {
    check_prec(prec);
    if (m < 1) throw Error(ERR_SOLVER, "richardson: m must be >= 1");
    auto r = std::make_unique<f3rg_richardson>();
    r->a = a->m;
    r->prec = prec;
    r->m = m;
    const uint64_t n = a->m->rows();
    const size_t vb = n * (prec == 0 ? 2 : prec == 1 ? 4 : 8) + 16;
    r->omegas.alloc((size_t)m * 8);
    r->wused.alloc((size_t)m * 8);
    r->wupd.alloc((size_t)m * 4);
    r->calls.alloc(32);
    r->R.alloc(vb);
    r->Za.alloc(vb);
    r->Zb.alloc(vb);
    r->dead.alloc(64);
    r->cnt.alloc(CNT_N * 8);
    r->partials.alloc((size_t)max_partial_blocks() * 16 * 8);
    r->counter.alloc(64);
    r->bar.alloc(64);
    for (DevBuf* b : {&r->dead, &r->cnt, &r->counter, &r->bar}) F3RG_CUDA(cudaMemset(b->get(), 0, b->bytes()));
    RichState h;
    h.m = m;
    h.cycle = cycle;
    h.omegas = r->omegas.get<double>();
    h.wused = r->wused.get<double>();
    h.wupd = r->wupd.get<int>();
    h.calls = r->calls.get<unsigned long long>();
    h.R = r->R.get();
    h.Za = r->Za.get();
    h.Zb = r->Zb.get();
    r->state.alloc(sizeof h);
    F3RG_CUDA(cudaMemcpy(r->state.get(), &h, sizeof h, cudaMemcpyHostToDevice));
    std::vector<double> w((size_t)m, 1.0);
    F3RG_CUDA(cudaMemcpy(r->omegas.get(), w.data(), w.size() * 8, cudaMemcpyHostToDevice));
    const unsigned long long c[4] = {1ull, 0ull, 0ull, 0ull};
    F3RG_CUDA(cudaMemcpy(r->calls.get(), c, sizeof c, cudaMemcpyHostToDevice));
    *out = r.release();
  });
}

void f3rg_richardson_destroy(f3rg_richardson* r) { delete r; }

int f3rg_richardson_set_omegas(f3rg_richardson* r, const double* w) {
  return guarded([&] {
    F3RG_CUDA(cudaDeviceSynchronize());
    F3RG_CUDA(cudaMemcpy(r->omegas.get(), w, (size_t)r->m * 8, cudaMemcpyHostToDevice));
    // a pageable H2D cudaMemcpy may return before its DMA lands; applies run on
    // other (non-blocking) streams, so wait for it here
    F3RG_CUDA(cudaDeviceSynchronize());
  });
}

int f3rg_richardson_state(f3rg_richardson* r, double* omegas, uint64_t* counters) {
  return guarded([&] {
    F3RG_CUDA(cudaDeviceSynchronize());
    if (omegas) F3RG_CUDA(cudaMemcpy(omegas, r->omegas.get(), (size_t)r->m * 8, cudaMemcpyDeviceToHost));
    unsigned long long c[4];
    F3RG_CUDA(cudaMemcpy(c, r->calls.get(), sizeof c, cudaMemcpyDeviceToHost));
    if (counters) counters[0] = c[0], counters[1] = c[1], counters[2] = c[2];
  });
}

int f3rg_richardson_set_precond(f3rg_richardson* r, const f3rg_precond* m) {
  return guarded([&] {
    if (!r) throw Error(ERR_DIMENSION, "null argument");
    if (m && m->p->rows() != r->a->rows()) throw Error(ERR_DIMENSION, "preconditioner size does not match the matrix");
    F3RG_CUDA(cudaDeviceSynchronize());
    r->M = m ? m->p : nullptr;
    if (r->M && !r->M->identity()) {
      const uint64_t n = r->a->rows();
      r->P.alloc(n * (r->prec == 0 ? 2 : r->prec == 1 ? 4 : 8) + 16);
      r->work = r->M->make_work();
    }
  });
}

int f3rg_richardson_apply(f3rg_richardson* r, const void* v, void* z, uintptr_t stream) {
  return guarded([&] {
    const int p = r->prec;
    if (r->M && !r->M->identity()) {
      // richardson_apply with op.precondition = M (src/richardson.cpp:10-54): the
      // launch sequence of Solver::enqueue_richardson_m
      cudaStream_t s = as_stream(stream);
      const uint64_t n = r->a->rows();
      const GateH gate{r->dead.get<int>(), 0};
      const SyncH sync{r->partials.get<double>(), r->counter.get<unsigned>()};
      auto phase = [&](int ph, int k) {
        F3RG_CUDA(launch_richm_phase(p, p, p, Launch{0, s}, r->a->csr(), r->a->tiles(p), ph, k, v, nullptr, z, n,
                                     r->state.get<RichState>(), r->R.get(), r->P.get(), r->Za.get(), gate, 0,
                                     r->cnt.get<unsigned long long>(), sync));
      };
      phase(RM_START_H, 0);
      for (int k = 0; k < r->m; ++k) {
        if (k > 0) phase(RM_RESID_H, k);
        RichEpiH re{r->state.get<RichState>(), k, k > 0 ? r->Za.get() : nullptr, k + 1 == r->m ? z : r->Za.get()};
        r->M->enqueue(*r->work, r->R.get(), p, r->P.get(), p, s, nullptr, 0, &re);
        phase(RM_DOTS_H, k);
        phase(RM_UPDATE_H, k);
      }
      phase(RM_BOOK_H, 0);
      return;
    }
    F3RG_CUDA(launch_richardson(p, p, p, Launch{0, as_stream(stream)}, r->a->csr(), r->a->tiles(p), v, nullptr, z,
                                r->a->rows(), r->state.get<RichState>(), GateH{r->dead.get<int>(), 0}, 0,
                                r->cnt.get<unsigned long long>(),
                                SyncH{r->partials.get<double>(), r->counter.get<unsigned>()}, r->bar.get<unsigned>(),
                                r->bar.get<unsigned>() + 1, nullptr));
  });
}

}  // extern "C"

// ---- restarted fp64 FGMRES(m) with M (reference fgmres_restarted) ------------------------
extern "C" int f3rg_fgmres_solve(const f3rg_matrix* a, const f3rg_precond* m, int restart, const double* b_host,
                                 double* x_host, double tol, uint64_t max_precond, f3rg_report* rep, double* history,
                                 uint64_t hist_cap) {
  return guarded([&] {
    if (!a || !b_host || !m) throw Error(ERR_DIMENSION, "null argument");
    if (restart < 1) throw Error(ERR_SOLVER, "restart length must be >= 1");
    const uint64_t n = a->m->rows();
    const int kind = m->p->identity() ? PK_IDENTITY : m->p->config().symmetric ? PK_IC0 : PK_ILU0;
    Solver s(parse_spec("F" + std::to_string(restart) + ":f64/f64"), a->m, kind, nullptr, m->p);
    DevBuf b(n * 8 + 16), x(n * 8 + 16);
    F3RG_CUDA(cudaMemcpy(b.get(), b_host, n * 8, cudaMemcpyHostToDevice));
    RunOptions o;
    o.tol = tol;
    o.restart_budget = max_precond;
    Report r = s.run(b.get<double>(), x_host ? x.get<double>() : nullptr, o, nullptr);
    if (max_precond == 0) {  // the reference caps before the first cycle
      r.outer_iterations = 0;
      r.flag = "capped";
    }
    r.solver_id = "fgmres" + std::to_string(restart);
    r.level_iterations.clear();
    r.omegas_final.clear();
    if (x_host) F3RG_CUDA(cudaMemcpy(x_host, x.get(), n * 8, cudaMemcpyDeviceToHost));
    fill_report(r, rep);
    for (uint64_t i = 0; history && i < r.residual_history.size() && i < hist_cap; ++i) history[i] = r.residual_history[i];
  });
}

// ---- fp64 CG / BiCGStab -------------------------------------------------------------
extern "C" int f3rg_krylov_solve_m(const f3rg_matrix* a, const f3rg_precond* m, int which, const double* b_host,
                                   double* x_host, double tol, uint64_t max_precond, f3rg_report* rep,
                                   double* history, uint64_t hist_cap) {
  return guarded([&] {
    if (!a || !b_host) throw Error(ERR_DIMENSION, "null argument");
    const uint64_t n = a->m->rows();
    KrylovSolver ks(a->m, m ? m->p : nullptr);
    DevBuf b(n * 8 + 16), x(n * 8 + 16);
    F3RG_CUDA(cudaMemcpy(b.get(), b_host, n * 8, cudaMemcpyHostToDevice));
    const Report r = ks.solve(which, b.get<double>(), x.get<double>(), tol, max_precond, nullptr);
    if (x_host) F3RG_CUDA(cudaMemcpy(x_host, x.get(), n * 8, cudaMemcpyDeviceToHost));
    fill_report(r, rep);
    for (uint64_t i = 0; history && i < r.residual_history.size() && i < hist_cap; ++i)
      history[i] = r.residual_history[i];
  });
}

extern "C" int f3rg_krylov_solve(const f3rg_matrix* a, int which, const double* b_host, double* x_host, double tol,
                                 uint64_t max_precond, f3rg_report* rep, double* history, uint64_t hist_cap) {
  return f3rg_krylov_solve_m(a, nullptr, which, b_host, x_host, tol, max_precond, rep, history, hist_cap);
}

// ---- row-block partition ----------------------------------------
struct f3rg_comm {
  int P = 1;
  std::unique_ptr<LocalGroup> local;
  std::vector<std::unique_ptr<LocalExchange>> lex;
  std::unique_ptr<NcclExchange> nccl;
  uint64_t n = 0;
};

extern "C" {

int f3rg_part_plan(const f3rg_csr* a, int P, int rank, f3rg_part_info* info, uint32_t* halo, uint64_t* recv_off,
                   uint64_t* recv_cnt, uint64_t* send_cnt, uint32_t* send_idx, uint32_t* local_rp,
                   uint32_t* local_ci) {
  return guarded([&] {
    if (!a || !info) throw Error(ERR_DIMENSION, "null argument");
    validate_csr(a->n, a->row_ptr, a->col_idx);
    const PartPlan p = make_plan(a->n, a->row_ptr, a->col_idx, P, rank);
    info->r0 = p.r0;
    info->r1 = p.r1;
    info->n_lo = p.n_lo;
    info->n_hi = p.n_hi;
    info->pad = p.pad;
    info->off = p.off();
    info->n_ext = p.n_ext();
    info->ld = p.ld();
    info->nnz_local = p.ci.size();
    info->nnz_begin = p.nnz_begin;
    uint64_t nsend = 0;
    for (const auto& v : p.send_idx) nsend += v.size();
    info->n_send = nsend;
    if (halo) std::memcpy(halo, p.halo.data(), p.halo.size() * 4);
    for (int q = 0; q < P; ++q) {
      if (recv_off) recv_off[q] = p.recv_off[q];
      if (recv_cnt) recv_cnt[q] = p.recv_cnt[q];
      if (send_cnt) send_cnt[q] = p.send_idx[q].size();
    }
    if (send_idx) {
      uint64_t o = 0;
      for (const auto& v : p.send_idx) {
        std::memcpy(send_idx + o, v.data(), v.size() * 4);
        o += v.size();
      }
    }
    if (local_rp) std::memcpy(local_rp, p.rp.data(), p.rp.size() * 4);
    if (local_ci) std::memcpy(local_ci, p.ci.data(), p.ci.size() * 4);
  });
}

int f3rg_comm_local(f3rg_comm** out, const f3rg_csr* a, int P) {
  return guarded([&] {
    if (!out || !a) throw Error(ERR_DIMENSION, "null argument");
    validate_csr(a->n, a->row_ptr, a->col_idx);
    auto c = std::make_unique<f3rg_comm>();
    c->P = P;
    c->n = a->n;
    c->local = std::make_unique<LocalGroup>(P);
    c->local->set_plans(a->n, a->row_ptr, a->col_idx);
    for (int r = 0; r < P; ++r) c->lex.push_back(std::make_unique<LocalExchange>(c->local.get(), r));
    *out = c.release();
  });
}

int f3rg_nccl_unique_id(void* out128) {
  return guarded([&] {
    if (!out128) throw Error(ERR_DIMENSION, "null argument");
    NcclExchange::unique_id(out128);
  });
}

int f3rg_comm_nccl(f3rg_comm** out, const f3rg_csr* a, int P, int rank, const void* unique_id) {
  return guarded([&] {
    if (!out || !a || !unique_id) throw Error(ERR_DIMENSION, "null argument");
    validate_csr(a->n, a->row_ptr, a->col_idx);
    auto c = std::make_unique<f3rg_comm>();
    c->P = P;
    c->n = a->n;
    c->nccl = std::make_unique<NcclExchange>(P, rank, unique_id, a->n, a->row_ptr, a->col_idx);
    *out = c.release();
  });
}

void f3rg_comm_destroy(f3rg_comm* c) { delete c; }

int f3rg_solver_create_part(f3rg_solver** out, f3rg_comm* c, const f3rg_csr* a, const char* spec, int precond_kind,
                            int rank) {
  return guarded([&] {
    if (!out || !c || !a || !spec) throw Error(ERR_DIMENSION, "null argument");
    if (a->n != c->n) throw Error(ERR_DIMENSION, "matrix differs from the one the communicator was planned for");
    Exchange* ex = nullptr;
    if (c->local) {
      if (rank < 0 || rank >= c->P) throw Error(ERR_DIMENSION, "rank out of range");
      ex = c->lex[rank].get();
    } else {
      if (rank != c->nccl->rank()) throw Error(ERR_DIMENSION, "rank differs from the communicator's");
      ex = c->nccl.get();
    }
    const PartPlan& p = ex->plan();
    auto m = std::make_shared<DeviceMatrix>(p.n_own(), p.rp.data(), p.ci.data(), a->values + p.nnz_begin, p.n_ext());
    auto h = std::make_unique<f3rg_solver>();
    h->s = std::make_unique<Solver>(parse_spec(spec), m, precond_kind, ex);
    *out = h.release();
  });
}

int f3rg_solve_local(f3rg_comm* c, f3rg_solver** solvers, const double* b_host, double* x_host,
                     const f3rg_run_options* o, f3rg_report* reps) {
  return guarded([&] {
    if (!c || !c->local || !solvers || !b_host) throw Error(ERR_DIMENSION, "local solve needs a local communicator");
    const int P = c->P;
    std::vector<int> codes((size_t)P, F3RG_OK);
    std::vector<std::string> msgs((size_t)P);
    std::vector<std::thread> th;
    const RunOptions opts = to_opts(o);
    for (int r = 0; r < P; ++r) {
      th.emplace_back([&, r] {
        try {
          f3rg_solver* s = solvers[r];
          const PartPlan& p = c->local->plans[r];
          const uint64_t n = p.n_own();
          if (s->s->rows() != n || s->s->exchange() != c->lex[r].get())
            throw Error(ERR_DIMENSION, "solver " + std::to_string(r) + " is not rank " + std::to_string(r));
          cudaStream_t st = c->local->stream;
          if (!s->b.get()) s->b.alloc(n * 8 + 16), s->x.alloc(n * 8 + 16);
          F3RG_CUDA(cudaMemcpyAsync(s->b.get(), b_host + p.r0, n * 8, cudaMemcpyHostToDevice, st));
          s->last = s->s->run(s->b.get<double>(), x_host ? s->x.get<double>() : nullptr, opts, st);
          if (x_host) {
            F3RG_CUDA(cudaMemcpyAsync(x_host + p.r0, s->x.get(), n * 8, cudaMemcpyDeviceToHost, st));
            F3RG_CUDA(cudaStreamSynchronize(st));
          }
          if (reps) fill_report(s->last, reps + r);
        } catch (const Error& e) {
          codes[r] = e.code, msgs[r] = e.what();
          c->local->fail();
        } catch (const std::exception& e) {
          codes[r] = F3RG_EINTERNAL, msgs[r] = e.what();
          c->local->fail();
        }
      });
    }
    for (auto& t : th) t.join();
    for (int r = 0; r < P; ++r)
      if (codes[r] != F3RG_OK && msgs[r].find("a peer rank failed") == std::string::npos)
        throw Error(codes[r], "rank " + std::to_string(r) + ": " + msgs[r]);
    for (int r = 0; r < P; ++r)
      if (codes[r] != F3RG_OK) throw Error(codes[r], "rank " + std::to_string(r) + ": " + msgs[r]);
  });
}

int f3rg_local_spmv(const f3rg_csr* a, int P, int pa, int px, int py, const double* x_host, double* y_host) {
  return guarded([&] {
    check_prec(pa), check_prec(px), check_prec(py);
    if (!a || !x_host || !y_host) throw Error(ERR_DIMENSION, "null argument");
    validate_csr(a->n, a->row_ptr, a->col_idx);
    LocalGroup g(P);
    g.set_plans(a->n, a->row_ptr, a->col_idx);
    const size_t esx = px == 0 ? 2 : px == 1 ? 4 : 8, esy = py == 0 ? 2 : py == 1 ? 4 : 8;
    std::vector<std::shared_ptr<DeviceMatrix>> mats;
    std::vector<DevBuf> xs((size_t)P), ys((size_t)P);
    DevBuf tmp(a->n * 8 + 16);
    for (int r = 0; r < P; ++r) {
      const PartPlan& p = g.plans[r];
      mats.push_back(
          std::make_shared<DeviceMatrix>(p.n_own(), p.rp.data(), p.ci.data(), a->values + p.nnz_begin, p.n_ext()));
      xs[r].alloc(p.ld() * esx + 16);
      ys[r].alloc(p.n_own() * esy + 16);
      F3RG_CUDA(cudaMemset(xs[r].get(), 0, xs[r].bytes()));
      F3RG_CUDA(cudaMemcpy(tmp.get(), x_host + p.r0, p.n_own() * 8, cudaMemcpyHostToDevice));
      F3RG_CUDA(launch_copy(2, px, Launch{}, tmp.get(), xs[r].get<char>() + p.off() * esx, p.n_own()));
      g.ptrs[r] = xs[r].get();
    }
    for (int r = 0; r < P; ++r) g.gather_into(r, xs[r].get(), px, nullptr);
    for (int r = 0; r < P; ++r) {
      const PartPlan& p = g.plans[r];
      F3RG_CUDA(launch_spmv(pa, px, py, Launch{}, mats[r]->csr(), mats[r]->tiles(pa), xs[r].get(), ys[r].get()));
      F3RG_CUDA(launch_copy(py, 2, Launch{}, ys[r].get(), tmp.get(), p.n_own()));
      F3RG_CUDA(cudaMemcpy(y_host + p.r0, tmp.get(), p.n_own() * 8, cudaMemcpyDeviceToHost));
    }
  });
}

int f3rg_solve_part_device(f3rg_solver* s, const double* b_own, double* x_own, const f3rg_run_options* o,
                           f3rg_report* rep, uintptr_t stream) {
  return guarded([&] {
    if (!s || !s->s->exchange()) throw Error(ERR_DIMENSION, "not a partitioned solver");
    s->last = s->s->run(b_own, x_own, to_opts(o), as_stream(stream));
    fill_report(s->last, rep);
  });
}

}  // extern "C"

namespace f3rg {
void set_last_error(const std::string& m) { g_err = m; }
}  // namespace f3rg

// ---- diagonal scaling on the device (reference diagonal_scale, src/scaling.cpp:11-38) ----
extern "C" int f3rg_matrix_create_scaled(f3rg_matrix** out, const f3rg_csr* a, const double* b_host,
                                         double* b_scaled_host, double* d_host) {
  return guarded([&] {
    if (!out || !a) throw Error(ERR_DIMENSION, "null argument");
    const uint64_t n = a->n;
    DevBuf d(n * 8 + 16);
    auto h = std::make_unique<f3rg_matrix>();
    DeviceMatrix::Scale sc;
    sc.d_dev = d.get<double>();
    h->m = std::make_shared<DeviceMatrix>(n, a->row_ptr, a->col_idx, a->values, sc);
    if (b_host && b_scaled_host) {
      DevBuf b(n * 8 + 16), bs(n * 8 + 16);
      F3RG_CUDA(cudaMemcpy(b.get(), b_host, n * 8, cudaMemcpyHostToDevice));
      F3RG_CUDA(launch_scale_rhs(Launch{}, b.get<double>(), d.get<double>(), bs.get<double>(), n));
      F3RG_CUDA(cudaMemcpy(b_scaled_host, bs.get(), n * 8, cudaMemcpyDeviceToHost));
    }
    if (d_host) F3RG_CUDA(cudaMemcpy(d_host, d.get(), n * 8, cudaMemcpyDeviceToHost));
    *out = h.release();
  });
}
