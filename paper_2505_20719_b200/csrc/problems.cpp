// problems.cpp -- synthetic problem generators (include/f3rg_problems.h).
// Host setup code: builds the fp64 CSR of each BASELINE.json configuration with
// the reference's conventions and seeds. Compiled with
// -ffp-contract=off so b = A x_true and the diagonal scaling round exactly like
// the reference (src/csr.cpp:23-37, src/scaling.cpp:11-38).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/f3rg.h"
#include "../../include/f3rg_problems.h"
#include "engine.hpp"

namespace {

// SplitMix64 (Vigna's constants; the reference's include/f3r/rng.hpp:15-32 uses the same stream)
struct Mix64 {
  uint64_t s;
  explicit Mix64(uint64_t seed) : s(seed) {}
  uint64_t next() {
    s += 0x9e3779b97f4a7c15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double unit() { return (double)(next() >> 11) * 0x1.0p-53; }  // [0, 1)
  double gauss() {  // Box-Muller on two draws; 1-u keeps the log argument in (0, 1]
    const double u1 = unit(), u2 = unit();
    return std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(6.283185307179586 * u2);
  }
};

struct Csr {
  uint64_t n = 0;
  std::vector<uint32_t> rp, ci;
  std::vector<double> val;
};

// 7-point pattern with per-entry value callback v(i, j, k, dir) where dir in
// {0:-z, 1:-y, 2:-x, 3:self, 4:+x, 5:+y, 6:+z} (ascending column order)
template <class F>
Csr seven_point(int64_t nx, int64_t ny, int64_t nz, F&& v) {
  Csr a;
  a.n = (uint64_t)(nx * ny * nz);
  a.rp.assign(a.n + 1, 0);
  // row lengths first (parallel fill afterwards)
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        const uint64_t row = (uint64_t)(i + nx * (j + ny * k));
        a.rp[row + 1] = 1u + (k > 0) + (j > 0) + (i > 0) + (i + 1 < nx) + (j + 1 < ny) + (k + 1 < nz);
      }
  for (uint64_t r = 0; r < a.n; ++r) a.rp[r + 1] += a.rp[r];
  a.ci.resize(a.rp[a.n]);
  a.val.resize(a.rp[a.n]);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        const int64_t row = i + nx * (j + ny * k);
        uint32_t p = a.rp[row];
        auto put = [&](int64_t col, int dir) {
          a.ci[p] = (uint32_t)col;
          a.val[p] = v(i, j, k, dir);
          ++p;
        };
        if (k > 0) put(row - nx * ny, 0);
        if (j > 0) put(row - nx, 1);
        if (i > 0) put(row - 1, 2);
        put(row, 3);
        if (i + 1 < nx) put(row + 1, 4);
        if (j + 1 < ny) put(row + nx, 5);
        if (k + 1 < nz) put(row + nx * ny, 6);
      }
  return a;
}

// HPCG/HPGMP 27-point operator, semantics of the reference generate_stencil
// (src/stencil.cpp:55-101): diag 26, off -1, z face neighbours -1 +/- beta.
Csr stencil27(int64_t nx, int64_t ny, int64_t nz, double beta) {
  Csr a;
  a.n = (uint64_t)(nx * ny * nz);
  a.rp.assign(a.n + 1, 0);
  auto cnt = [](int64_t c, int64_t n) { return (int64_t)1 + (c > 0) + (c + 1 < n); };
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i)
        a.rp[(uint64_t)(i + nx * (j + ny * k)) + 1] = (uint32_t)(cnt(i, nx) * cnt(j, ny) * cnt(k, nz));
  for (uint64_t r = 0; r < a.n; ++r) a.rp[r + 1] += a.rp[r];
  a.ci.resize(a.rp[a.n]);
  a.val.resize(a.rp[a.n]);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        const int64_t row = i + nx * (j + ny * k);
        uint32_t p = a.rp[row];
        for (int dz = -1; dz <= 1; ++dz) {
          if (k + dz < 0 || k + dz >= nz) continue;
          for (int dy = -1; dy <= 1; ++dy) {
            if (j + dy < 0 || j + dy >= ny) continue;
            for (int dx = -1; dx <= 1; ++dx) {
              if (i + dx < 0 || i + dx >= nx) continue;
              double v = -1.0;
              if (!dx && !dy && !dz) v = 26.0;
              else if (!dx && !dy && dz == 1) v = -1.0 + beta;
              else if (!dx && !dy && dz == -1) v = -1.0 - beta;
              a.ci[p] = (uint32_t)((i + dx) + nx * ((j + dy) + ny * (k + dz)));
              a.val[p] = v;
              ++p;
            }
          }
        }
      }
  return a;
}

// Config 4: face coefficients k = exp(sigma*g), g ~ N(0,1) i.i.d. from one
// SplitMix64(seed) stream, drawn x-faces, then y-faces, then z-faces, each in
// lexicographic order (face index fastest along its own axis); z faces x zscale.
// A cell's diagonal sums its six faces (Dirichlet faces included) in the order
// x-, x+, y-, y+, z-, z+; off-diagonals are -k of the shared face. SPD.
Csr aniso7(int64_t nx, int64_t ny, int64_t nz, double sigma, double zscale, uint64_t seed) {
  Mix64 r(seed);
  std::vector<double> kx((size_t)((nx + 1) * ny * nz)), ky((size_t)(nx * (ny + 1) * nz)),
      kz((size_t)(nx * ny * (nz + 1)));
  for (auto& v : kx) v = std::exp(sigma * r.gauss());
  for (auto& v : ky) v = std::exp(sigma * r.gauss());
  for (auto& v : kz) v = std::exp(sigma * r.gauss()) * zscale;
  auto fx = [&](int64_t i, int64_t j, int64_t k) { return kx[(size_t)(i + (nx + 1) * (j + ny * k))]; };
  auto fy = [&](int64_t i, int64_t j, int64_t k) { return ky[(size_t)(i + nx * (j + (ny + 1) * k))]; };
  auto fz = [&](int64_t i, int64_t j, int64_t k) { return kz[(size_t)(i + nx * (j + ny * k))]; };
  return seven_point(nx, ny, nz, [&](int64_t i, int64_t j, int64_t k, int dir) {
    switch (dir) {
      case 0: return -fz(i, j, k);
      case 1: return -fy(i, j, k);
      case 2: return -fx(i, j, k);
      case 4: return -fx(i + 1, j, k);
      case 5: return -fy(i, j + 1, k);
      case 6: return -fz(i, j, k + 1);
      default: {
        double s = fx(i, j, k);
        s = s + fx(i + 1, j, k);
        s = s + fy(i, j, k);
        s = s + fy(i, j + 1, k);
        s = s + fz(i, j, k);
        s = s + fz(i, j, k + 1);
        return s;
      }
    }
  });
}

// Config 5: per-row stream SplitMix64(seed ^ (0xD1B54A32D192ED03 * (row + 1))).
// Row length L ~ lognormal (mu = ln 30 - s^2/2, s = 0.5; rejection to [5, 200]),
// L-1 off-diagonal columns: 5% uniform in [0, n), else row + round(N(0, band^2));
// out-of-range / diagonal / duplicate draws are redrawn. Values U[-1, 1] in
// ascending column order; diagonal = 1.1 * sum |off| (strict diagonal dominance).
struct RowGen {
  uint64_t n, seed;
  double band, frac_long;
  Mix64 stream(uint64_t row) const { return Mix64(seed ^ (0xD1B54A32D192ED03ull * (row + 1))); }
  static uint32_t length(Mix64& r) {
    const double s = 0.5, mu = std::log(30.0) - 0.5 * s * s;
    for (;;) {
      const double L = std::floor(std::exp(mu + s * r.gauss()) + 0.5);
      if (L >= 5.0 && L <= 200.0) return (uint32_t)L;
    }
  }
};

Csr unstructured(uint64_t n, uint64_t seed) {
  RowGen g{n, seed, 5000.0, 0.05};
  Csr a;
  a.n = n;
  a.rp.assign(n + 1, 0);
  const uint64_t cap = n < 200 ? n : 200;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    Mix64 r = g.stream((uint64_t)i);
    a.rp[(uint64_t)i + 1] = std::min<uint32_t>(RowGen::length(r), (uint32_t)cap);
  }
  for (uint64_t i = 0; i < n; ++i) a.rp[i + 1] += a.rp[i];
  a.ci.resize(a.rp[n]);
  a.val.resize(a.rp[n]);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    Mix64 r = g.stream((uint64_t)i);
    (void)RowGen::length(r);
    const uint32_t L = a.rp[i + 1] - a.rp[i];
    uint32_t* cols = &a.ci[a.rp[i]];
    cols[0] = (uint32_t)i;
    uint32_t have = 1;
    while (have < L) {
      int64_t c;
      if (r.unit() < g.frac_long) {
        c = (int64_t)(r.next() % n);
      } else {
        c = i + (int64_t)std::llround(g.band * r.gauss());
      }
      if (c < 0 || c >= (int64_t)n) continue;
      bool dup = false;
      for (uint32_t q = 0; q < have; ++q) dup = dup || cols[q] == (uint32_t)c;
      if (dup) continue;
      cols[have++] = (uint32_t)c;
    }
    std::sort(cols, cols + L);
    double* v = &a.val[a.rp[i]];
    double off = 0.0;
    uint32_t dpos = 0;
    for (uint32_t q = 0; q < L; ++q) {
      if (cols[q] == (uint32_t)i) {
        dpos = q;
        continue;
      }
      v[q] = 2.0 * r.unit() - 1.0;
      off = off + std::fabs(v[q]);
    }
    v[dpos] = 1.1 * off;
  }
  return a;
}

}  // namespace

struct f3rg_problem {
  Csr a;
  std::vector<double> b, d;
};

namespace {
thread_local std::string g_perr;
}

extern "C" {

int f3rg_problem_generate(f3rg_problem** out, int kind, const uint64_t grid[3], double param, uint64_t seed) {
  try {
    auto p = std::make_unique<f3rg_problem>();
    const int64_t nx = (int64_t)grid[0], ny = (int64_t)grid[1], nz = (int64_t)grid[2];
    switch (kind) {
      case F3RG_GEN_POISSON7:
        p->a = seven_point(nx, ny, nz, [](int64_t, int64_t, int64_t, int dir) { return dir == 3 ? 6.0 : -1.0; });
        break;
      case F3RG_GEN_STENCIL27:
        p->a = stencil27(nx, ny, nz, param);
        break;
      case F3RG_GEN_CONVDIFF7:
        // -Laplace(u) + v.grad(u), h = 1, nu = 1, v = (1,1,1): Pe_cell = |v_i| h / (2 nu) = 0.5;
        // first-order upwind (v > 0 -> backward differences): diag 6 + 3, upwind -2, downwind -1
        p->a = seven_point(nx, ny, nz, [](int64_t, int64_t, int64_t, int dir) {
          return dir == 3 ? 9.0 : (dir < 3 ? -2.0 : -1.0);
        });
        break;
      case F3RG_GEN_ANISO7:
        p->a = aniso7(nx, ny, nz, 1.5, 1e-2, seed);
        break;
      case F3RG_GEN_UNSTRUCTURED:
        p->a = unstructured(grid[0], seed);
        break;
      default:
        throw f3rg::Error(F3RG_EDIMENSION, "unknown generator kind");
    }
    if (p->a.rp.back() >= (1ull << 31)) throw f3rg::Error(F3RG_EDIMENSION, "matrix exceeds 32-bit index range");
    *out = p.release();
    return 0;
  } catch (const f3rg::Error& e) {
    g_perr = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_perr = e.what();
    return F3RG_EINTERNAL;
  }
}

void f3rg_problem_destroy(f3rg_problem* p) { delete p; }

int f3rg_problem_finalize(f3rg_problem* p, int mode, uint64_t seed) {
  Csr& a = p->a;
  const uint64_t n = a.n;
  // d_i = 1 / sqrt(|a_ii|) (src/scaling.cpp:19-27)
  p->d.assign(n, 0.0);
  for (uint64_t i = 0; i < n; ++i) {
    double aii = 0.0;
    bool found = false;
    for (uint32_t k = a.rp[i]; k < a.rp[i + 1]; ++k)
      if (a.ci[k] == i) aii = a.val[k], found = true;
    if (!found || aii == 0.0) return F3RG_EFACTORIZATION;
    p->d[i] = 1.0 / std::sqrt(std::fabs(aii));
  }
  p->b.assign(n, 0.0);
  if (mode == 0) {
    std::vector<double> xt(n);
    Mix64 r(seed);
    for (auto& v : xt) v = 2.0 * r.unit() - 1.0;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
      double acc = 0.0;
      for (uint32_t k = a.rp[i]; k < a.rp[i + 1]; ++k) acc = acc + a.val[k] * xt[a.ci[k]];
      p->b[i] = acc;
    }
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; ++i)
    for (uint32_t k = a.rp[i]; k < a.rp[i + 1]; ++k) a.val[k] = a.val[k] * p->d[i] * p->d[a.ci[k]];
  if (mode == 0) {
    for (uint64_t i = 0; i < n; ++i) p->b[i] = p->b[i] * p->d[i];
  } else {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
      double acc = 0.0;
      for (uint32_t k = a.rp[i]; k < a.rp[i + 1]; ++k) acc = acc + a.val[k] * 1.0;
      p->b[i] = acc;
    }
  }
  return 0;
}

int f3rg_problem_arrays(const f3rg_problem* p, uint64_t* n, uint64_t* nnz, const uint32_t** row_ptr,
                        const uint32_t** col_idx, const double** values, const double** b, const double** d) {
  *n = p->a.n;
  *nnz = p->a.rp.back();
  *row_ptr = p->a.rp.data();
  *col_idx = p->a.ci.data();
  *values = p->a.val.data();
  *b = p->b.empty() ? nullptr : p->b.data();
  *d = p->d.empty() ? nullptr : p->d.data();
  return 0;
}

}  // extern "C"
