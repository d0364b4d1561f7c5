/* oracle/f3r_oracle.c -- TEST INFRASTRUCTURE ONLY (see f3r_oracle.h).
 *
 * A plain-C restatement of the reference's hot path, written from its
 * documented semantics:
 *   binary16         include/f3r/half.hpp:27-150   (RNE, no FTZ, canonical NaN 0x7e00)
 *   promotion rule   include/f3r/precision.hpp:22,59-84
 *   BLAS-1           src/vector_ops.cpp:20-173     (sequential reductions, no FMA)
 *   SpMV             src/csr.cpp:23-37             (row-sequential, accumulator = promote(A, x))
 *   FGMRES cycle     src/fgmres.cpp:21-161         (CGS, Givens, back-substitution)
 *   Richardson       src/richardson.cpp:10-54      (adaptive weight, cumulative average)
 *   nesting / run    src/nesting.cpp:46-352
 * Vectors are double arrays holding values representable at their precision
 * tag; "compute at precision c" means the operands are widened exactly and each
 * product/sum is rounded to c (for c = binary16 via binary32, which the
 * reference also does and which equals a correctly rounded binary16 op).
 */
#include "f3r_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ binary16 */

uint16_t or_half_from_double(double x) {
  if (isnan(x)) return 0x7e00u; /* canonical quiet NaN, sign dropped */
  _Float16 h = (_Float16)x;     /* libgcc __truncdfhf2: one RNE rounding from binary64 */
  uint16_t b;
  memcpy(&b, &h, 2);
  return b;
}

uint16_t or_half_from_float(float x) {
  if (isnan(x)) return 0x7e00u;
  _Float16 h = (_Float16)x; /* vcvtps2ph / __truncsfhf2: RNE */
  uint16_t b;
  memcpy(&b, &h, 2);
  return b;
}

float or_float_from_half(uint16_t b) {
  if ((b & 0x7c00u) == 0x7c00u && (b & 0x3ffu)) return NAN;
  _Float16 h;
  memcpy(&h, &b, 2);
  return (float)h;
}

static inline double h_of_f(float f) { return (double)or_float_from_half(or_half_from_float(f)); }
static inline double h_of_d(double d) { return (double)or_float_from_half(or_half_from_double(d)); }

double or_round(int p, double x) {
  if (p == OR_P64) return x;
  if (p == OR_P32) return (double)(float)x;
  return h_of_d(x);
}

static inline int maxp(int a, int b) { return a > b ? a : b; }

/* one correctly rounded op at precision c on operands already at c */
static inline double mul_c(int c, double a, double b) {
  if (c == OR_P64) return a * b;
  const float f = (float)a * (float)b;
  return c == OR_P32 ? (double)f : h_of_f(f);
}
static inline double add_c(int c, double a, double b) {
  if (c == OR_P64) return a + b;
  const float f = (float)a + (float)b;
  return c == OR_P32 ? (double)f : h_of_f(f);
}
static inline double sub_c(int c, double a, double b) {
  if (c == OR_P64) return a - b;
  const float f = (float)a - (float)b;
  return c == OR_P32 ? (double)f : h_of_f(f);
}
static inline double div_c(int c, double a, double b) {
  if (c == OR_P64) return a / b;
  const float f = (float)a / (float)b;
  return c == OR_P32 ? (double)f : h_of_f(f);
}
static inline double sqrt_c(int c, double a) {
  if (c == OR_P64) return sqrt(a);
  const float f = sqrtf((float)a);
  return c == OR_P32 ? (double)f : h_of_f(f);
}
static inline double hypot_c(int c, double a, double b) {
  if (c == OR_P64) return hypot(a, b);
  const float f = hypotf((float)a, (float)b);
  return c == OR_P32 ? (double)f : h_of_f(f);
}

/* -------------------------------------------------------------------- BLAS-1 */

void or_spmv(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals, int pa, const double* x,
             int px, double* y, int py) {
  const int c = maxp(pa, px);
  /* values and x are exact at their own precision, hence exact at c >= both */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    double acc = 0.0;
    if (c == OR_P64) {
      for (uint32_t k = rp[i]; k < rp[i + 1]; ++k) acc = acc + vals[k] * x[ci[k]];
    } else if (c == OR_P32) {
      float a = 0.0f;
      for (uint32_t k = rp[i]; k < rp[i + 1]; ++k) a = a + (float)vals[k] * (float)x[ci[k]];
      acc = a;
    } else {
      for (uint32_t k = rp[i]; k < rp[i + 1]; ++k) acc = add_c(OR_P16, acc, mul_c(OR_P16, vals[k], x[ci[k]]));
    }
    y[i] = or_round(py, acc);
  }
}

/* Summation order of the dots (experiments only): 0 = the reference's sequential
 * index order (src/vector_ops.cpp:20-28, the default), 1 = pairwise (blocks of 256
 * summed sequentially, then a balanced tree), at the same precision C. Used to show
 * that outer-count differences at large n come from the order alone. */
static int g_pairwise = 0;
void or_set_pairwise_dots(int on) { g_pairwise = on; }

static double dot_seq(int c, const double* x, const double* y, uint64_t lo, uint64_t hi) {
  double acc = 0.0;
  if (c == OR_P64) {
    for (uint64_t i = lo; i < hi; ++i) acc = acc + x[i] * y[i];
  } else if (c == OR_P32) {
    float a = 0.0f;
    for (uint64_t i = lo; i < hi; ++i) a = a + (float)x[i] * (float)y[i];
    acc = a;
  } else {
    for (uint64_t i = lo; i < hi; ++i) acc = add_c(OR_P16, acc, mul_c(OR_P16, x[i], y[i]));
  }
  return acc;
}

static double dot_pairwise(int c, const double* x, const double* y, uint64_t lo, uint64_t hi) {
  if (hi - lo <= 256) return dot_seq(c, x, y, lo, hi);
  const uint64_t mid = lo + (hi - lo) / 2;
  return add_c(c, dot_pairwise(c, x, y, lo, mid), dot_pairwise(c, x, y, mid, hi));
}

double or_dot(const double* x, int px, const double* y, int py, uint64_t n, int floor_p) {
  const int c = maxp(floor_p, maxp(px, py));
  return g_pairwise ? dot_pairwise(c, x, y, 0, n) : dot_seq(c, x, y, 0, n);
}

double or_norm2(const double* x, int px, uint64_t n) {
  const double s = or_dot(x, px, x, px, n, OR_P16);
  /* square root at the storage precision: sqrt(Half(s)) / sqrt(float(s)) / sqrt(s) */
  return sqrt_c(px, or_round(px, s));
}

void or_axpy(double alpha, const double* x, int px, double* y, int py, uint64_t n) {
  const int c = maxp(px, py);
  const double a = or_round(c, alpha);
  for (uint64_t i = 0; i < n; ++i) y[i] = or_round(py, add_c(c, mul_c(c, a, x[i]), y[i]));
}

void or_add_scaled(const double* x, int px, double alpha, const double* y, int py, double* out, int po,
                   uint64_t n) {
  const int c = maxp(maxp(px, py), po);
  const double a = or_round(c, alpha);
  for (uint64_t i = 0; i < n; ++i) out[i] = or_round(po, add_c(c, x[i], mul_c(c, a, y[i])));
}

void or_copy(const double* x, int px, double* y, int py, uint64_t n) {
  (void)px;
  for (uint64_t i = 0; i < n; ++i) y[i] = or_round(py, x[i]);
}

void or_scale(double alpha, double* x, int px, uint64_t n) {
  const double a = or_round(px, alpha);
  for (uint64_t i = 0; i < n; ++i) x[i] = mul_c(px, a, x[i]);
}

/* ------------------------------------------- block-Jacobi ILU(0) / IC(0) */
/* Restates BlockJacobiIlu0 (reference src/ilu.cpp:38-263, include/f3r/ilu.hpp:44-84):
 * contiguous row blocks (remainder to the leading blocks, :47-54), each diagonal
 * block factorised at fp64 with zero fill on a working copy whose diagonal is
 * scaled by alpha (:62-86); ILU in IKJ order (:88-106), IC on the lower pattern
 * (:108-137); factors split and rounded to the apply precision (:140-183). */

static double* vnew(uint64_t n) { return (double*)calloc(n ? n : 1, sizeof(double)); }

struct or_ilu {
  uint64_t n, nblocks;
  int symmetric, prec;
  uint32_t* br;                 /* nblocks + 1 row offsets */
  uint32_t *lp, *li, *upp, *ui; /* lower / upper CSR (upper empty for IC) */
  double *lv, *uv;              /* values, exactly representable at prec */
};

static int ilu_fail(char* err, size_t cap, const char* msg) {
  if (err && cap) snprintf(err, cap, "%s", msg);
  return 5;
}

static uint64_t ilu_block_of(const or_ilu* m, uint64_t row) {
  uint64_t b = 0;
  while (m->br[b + 1] <= row) ++b;
  return b;
}

void or_ilu_free(or_ilu* m) {
  if (!m) return;
  free(m->br);
  free(m->lp);
  free(m->li);
  free(m->upp);
  free(m->ui);
  free(m->lv);
  free(m->uv);
  free(m);
}

int or_ilu_factorize(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals, uint64_t nblocks,
                     double alpha, int symmetric, int prec, or_ilu** out, char* err, size_t errcap) {
  char msg[256];
  *out = NULL;
  if (nblocks == 0 || nblocks > n) return ilu_fail(err, errcap, "nblocks must be in [1, n]");
  if (!(alpha > 0.0)) return ilu_fail(err, errcap, "alpha must be positive");
  or_ilu* m = (or_ilu*)calloc(1, sizeof *m);
  m->n = n;
  m->nblocks = nblocks;
  m->symmetric = symmetric;
  m->prec = prec;
  m->br = (uint32_t*)malloc((nblocks + 1) * sizeof(uint32_t));
  m->br[0] = 0;
  for (uint64_t b = 0; b < nblocks; ++b) m->br[b + 1] = m->br[b] + (uint32_t)(n / nblocks + (b < n % nblocks));

  /* working rows: in-block entries (IC: j <= i only), diagonal scaled by alpha */
  const uint64_t nnz = rp[n];
  uint32_t* wp = (uint32_t*)calloc(n + 1, sizeof(uint32_t));
  uint32_t* wi = (uint32_t*)malloc((nnz ? nnz : 1) * sizeof(uint32_t));
  double* wv = (double*)malloc((nnz ? nnz : 1) * sizeof(double));
  uint32_t* wd = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
  uint64_t w = 0;
  int rc = 0;
  for (uint64_t b = 0; b < nblocks && !rc; ++b) {
    const uint32_t lo = m->br[b], hi = m->br[b + 1];
    for (uint32_t i = lo; i < hi; ++i) {
      int diag = 0;
      for (uint32_t k = rp[i]; k < rp[i + 1]; ++k) {
        const uint32_t j = ci[k];
        if (j < lo || j >= hi || (symmetric && j > i)) continue;
        if (j == i) {
          diag = 1;
          wd[i] = (uint32_t)w;
          wv[w] = vals[k] * alpha;
        } else {
          wv[w] = vals[k];
        }
        wi[w++] = j;
      }
      if (!diag) {
        snprintf(msg, sizeof msg, "missing diagonal entry in block %llu, row %u", (unsigned long long)b, i);
        rc = ilu_fail(err, errcap, msg);
        break;
      }
      wp[i + 1] = (uint32_t)w;
    }
  }
  if (!rc && !symmetric) {
    /* ILU(0): row i eliminates with every earlier row of its pattern, in order */
    int64_t* pos = (int64_t*)malloc((n ? n : 1) * sizeof(int64_t));
    for (uint64_t i = 0; i < n; ++i) pos[i] = -1;
    for (uint64_t b = 0; b < nblocks && !rc; ++b) {
      for (uint32_t i = m->br[b]; i < m->br[b + 1]; ++i) {
        for (uint32_t k = wp[i]; k < wp[i + 1]; ++k) pos[wi[k]] = k;
        for (uint32_t k = wp[i]; k < wp[i + 1] && wi[k] < i; ++k) {
          const uint32_t r = wi[k];
          wv[k] = wv[k] / wv[wd[r]];
          const double f = wv[k];
          for (uint32_t q = wd[r] + 1; q < wp[r + 1]; ++q)
            if (pos[wi[q]] >= 0) wv[pos[wi[q]]] = wv[pos[wi[q]]] - f * wv[q];
        }
        for (uint32_t k = wp[i]; k < wp[i + 1]; ++k) pos[wi[k]] = -1;
        if (wv[wd[i]] == 0.0) {
          snprintf(msg, sizeof msg, "zero pivot in block %llu, row %u", (unsigned long long)b, i);
          rc = ilu_fail(err, errcap, msg);
          break;
        }
      }
    }
    free(pos);
  } else if (!rc) {
    /* IC(0): l_ij = (a_ij - sum_{k<j} l_ik l_jk) / l_jj, l_ii = sqrt(a_ii - sum l_ik^2);
     * the sums walk the two rows' common columns below j in ascending order */
    for (uint64_t b = 0; b < nblocks && !rc; ++b) {
      for (uint32_t i = m->br[b]; i < m->br[b + 1] && !rc; ++i) {
        for (uint32_t k = wp[i]; k < wp[i + 1]; ++k) {
          const uint32_t j = wi[k];
          double s = wv[k];
          uint32_t a = wp[i], c = wp[j];
          while (a < wp[i + 1] && c < wp[j + 1] && wi[a] < j && wi[c] < j) {
            if (wi[a] == wi[c]) s = s - wv[a++] * wv[c++];
            else if (wi[a] < wi[c]) ++a;
            else ++c;
          }
          if (j < i) {
            wv[k] = s / wv[wd[j]];
          } else if (s <= 0.0) {
            snprintf(msg, sizeof msg, "non-positive pivot in block %llu, row %u", (unsigned long long)b, i);
            rc = ilu_fail(err, errcap, msg);
            break;
          } else {
            wv[k] = sqrt(s);
          }
        }
      }
    }
  }
  if (!rc) {
    /* split: IC keeps the whole lower row (diagonal last), ILU the strict lower
     * part and the upper part with its diagonal first */
    m->lp = (uint32_t*)calloc(n + 1, sizeof(uint32_t));
    m->upp = (uint32_t*)calloc(n + 1, sizeof(uint32_t));
    m->li = (uint32_t*)malloc((w ? w : 1) * sizeof(uint32_t));
    m->ui = (uint32_t*)malloc((w ? w : 1) * sizeof(uint32_t));
    m->lv = (double*)malloc((w ? w : 1) * sizeof(double));
    m->uv = (double*)malloc((w ? w : 1) * sizeof(double));
    uint64_t nl = 0, nu = 0;
    for (uint64_t i = 0; i < n; ++i) {
      for (uint32_t k = wp[i]; k < wp[i + 1]; ++k) {
        if (symmetric || wi[k] < i) {
          m->li[nl] = wi[k];
          m->lv[nl++] = wv[k];
        } else {
          m->ui[nu] = wi[k];
          m->uv[nu++] = wv[k];
        }
      }
      m->lp[i + 1] = (uint32_t)nl;
      m->upp[i + 1] = (uint32_t)nu;
    }
    static const char* pname[3] = {"f16", "f32", "f64"};
    for (uint64_t i = 0; i < n && !rc; ++i) {
      const double d = symmetric ? m->lv[m->lp[i + 1] - 1] : m->uv[m->upp[i]];
      const double cast = or_round(prec, d);
      if (cast == 0.0 || !isfinite(cast)) {
        snprintf(msg, sizeof msg, "casting factors to %s lost the diagonal of row %llu; block %llu", pname[prec],
                 (unsigned long long)i, (unsigned long long)ilu_block_of(m, i));
        rc = ilu_fail(err, errcap, msg);
      }
    }
    for (uint64_t k = 0; k < nl; ++k) m->lv[k] = or_round(prec, m->lv[k]);
    for (uint64_t k = 0; k < nu; ++k) m->uv[k] = or_round(prec, m->uv[k]);
  }
  free(wp);
  free(wi);
  free(wv);
  free(wd);
  if (rc) {
    or_ilu_free(m);
    return rc;
  }
  *out = m;
  return 0;
}

uint64_t or_ilu_count(const or_ilu* m, int upper) { return upper ? m->upp[m->n] : m->lp[m->n]; }

void or_ilu_export(const or_ilu* m, int upper, uint32_t* ptr, uint32_t* idx, double* vals) {
  const uint32_t* p = upper ? m->upp : m->lp;
  const uint64_t nz = p[m->n];
  memcpy(ptr, p, (m->n + 1) * sizeof(uint32_t));
  memcpy(idx, upper ? m->ui : m->li, nz * sizeof(uint32_t));
  memcpy(vals, upper ? m->uv : m->lv, nz * sizeof(double));
}

/* BlockJacobiIlu0::apply (src/ilu.cpp:187-263): per block, at C = promote(prec,
 * pr); every multiply and subtract rounds to C. IC's backward sweep scatters row
 * i's x_i into the earlier rows (column-oriented, :237-244). */
void or_ilu_apply(const or_ilu* m, const double* r, int pr, double* z, int pz) {
  const int c = maxp(m->prec, pr);
  double* t = vnew(m->n);
  for (uint64_t b = 0; b < m->nblocks; ++b) {
    const uint32_t lo = m->br[b], hi = m->br[b + 1];
    if (!m->symmetric) {
      for (uint32_t i = lo; i < hi; ++i) {
        double acc = r[i];
        for (uint32_t k = m->lp[i]; k < m->lp[i + 1]; ++k) acc = sub_c(c, acc, mul_c(c, m->lv[k], t[m->li[k]]));
        t[i] = acc;
      }
      for (uint32_t i = hi; i-- > lo;) {
        double acc = t[i];
        for (uint32_t k = m->upp[i] + 1; k < m->upp[i + 1]; ++k)
          acc = sub_c(c, acc, mul_c(c, m->uv[k], t[m->ui[k]]));
        t[i] = div_c(c, acc, m->uv[m->upp[i]]);
      }
    } else {
      for (uint32_t i = lo; i < hi; ++i) {
        double acc = r[i];
        const uint32_t dk = m->lp[i + 1] - 1;
        for (uint32_t k = m->lp[i]; k < dk; ++k) acc = sub_c(c, acc, mul_c(c, m->lv[k], t[m->li[k]]));
        t[i] = div_c(c, acc, m->lv[dk]);
      }
      for (uint32_t i = hi; i-- > lo;) {
        const uint32_t dk = m->lp[i + 1] - 1;
        const double xi = div_c(c, t[i], m->lv[dk]);
        t[i] = xi;
        for (uint32_t k = m->lp[i]; k < dk; ++k) t[m->li[k]] = sub_c(c, t[m->li[k]], mul_c(c, m->lv[k], xi));
      }
    }
  }
  for (uint64_t i = 0; i < m->n; ++i) z[i] = or_round(pz, t[i]);
  free(t);
}

/* --------------------------------------------------------------- the solver */

typedef struct {
  uint64_t n;
  const uint32_t* rp;
  const uint32_t* ci;
  const double* vals[3]; /* replicas by precision tag */
  const or_level* lv;
  int D;
  uint64_t precond_invocations;
  uint64_t level_inv[16];
  uint64_t level_it[16];
  /* Richardson state per level */
  double* omegas[16];
  uint64_t call_count[16], update_count[16], degenerate[16];
  const or_ilu* M; /* primary preconditioner; NULL = IdentityPrecond */
} ctx_t;


static void multiply(ctx_t* c, int d, const double* x, int px, double* y, int py) {
  or_spmv(c->n, c->rp, c->ci, c->vals[c->lv[d].pa], c->lv[d].pa, x, px, y, py);
}

static void inner_solve(ctx_t* c, int d, const double* rhs, int prhs, double* out, int pout);

/* LevelOperator::precondition (src/nesting.cpp:53-64) of level d */
static void precondition(ctx_t* c, int d, const double* v, int pv, double* z, int pz) {
  const int child = d + 1;
  if (child >= c->D) { /* PrimarySolver (src/nesting.cpp:70-83): M applies itself */
    c->precond_invocations++;
    if (c->M) or_ilu_apply(c->M, v, pv, z, pz);
    else or_copy(v, pv, z, pz, c->n); /* IdentityPrecond (src/ilu.cpp:33-36) */
    return;
  }
  const int cp = c->lv[child].pv;
  if (cp == pv) {
    inner_solve(c, child, v, pv, z, pz);
    return;
  }
  double* down = vnew(c->n);
  double* out = vnew(c->n);
  or_copy(v, pv, down, cp, c->n);
  inner_solve(c, child, down, cp, out, cp);
  or_copy(out, cp, z, pz, c->n);
  free(down);
  free(out);
}

typedef struct {
  int iterations;
  double residual_norm;
  int happy, diverged, divergence_step;
  int n_est;
  double* est; /* m+1 */
} cycle_res;

/* fgmres_cycle / cycle_impl<W> (src/fgmres.cpp:21-148); W = prec of b.
 * If d < 0 the operator is (A_pa, identity) on matrix `vals_override`. */
static cycle_res cycle(ctx_t* c, int d, const double* b, int W, double* x, int px, int m, int use_tol,
                       double rel_tol, int x_is_zero) {
  const uint64_t n = c->n;
  cycle_res res;
  memset(&res, 0, sizeof res);
  res.divergence_step = -1;
  res.est = (double*)calloc((size_t)m + 2, sizeof(double));
  double* r = vnew(n);
  if (x_is_zero) {
    or_copy(b, W, r, W, n);
  } else {
    double* ax = vnew(n);
    multiply(c, d, x, px, ax, W);
    or_add_scaled(b, W, -1.0, ax, W, r, W, n);
    free(ax);
  }
  const double beta = or_norm2(r, W, n);
  res.est[res.n_est++] = beta;
  res.residual_norm = beta;
  if (beta == 0.0 || !isfinite(beta)) {
    res.diverged = !isfinite(beta);
    res.divergence_step = res.diverged ? 0 : -1;
    free(r);
    return res;
  }
  double bnorm = beta;
  if (!x_is_zero) {
    double* bc = vnew(n);
    or_copy(b, W, bc, W, n);
    bnorm = or_norm2(bc, W, n);
    free(bc);
  }
  double** V = (double**)calloc((size_t)m + 1, sizeof(double*));
  double** Z = (double**)calloc((size_t)m, sizeof(double*));
  double* H = (double*)calloc((size_t)(m + 1) * (size_t)m, sizeof(double)); /* column j at H + j*(m+1) */
  double* g = (double*)calloc((size_t)m + 1, sizeof(double));
  double* cs = (double*)calloc((size_t)m, sizeof(double));
  double* sn = (double*)calloc((size_t)m, sizeof(double));
  or_scale(div_c(W, 1.0, or_round(W, beta)), r, W, n);
  V[0] = r;
  int nv = 1;
  g[0] = or_round(W, beta);

  for (int j = 0; j < m; ++j) {
    double* z = vnew(n);
    precondition(c, d, V[j], W, z, W);
    double* w = vnew(n);
    multiply(c, d, z, W, w, W);
    double* h = H + (size_t)j * (size_t)(m + 1);
    for (int i = 0; i <= j; ++i) h[i] = or_round(W, or_dot(w, W, V[i], W, n, OR_P16));
    for (int i = 0; i <= j; ++i) or_axpy(-h[i], V[i], W, w, W, n);
    const double wnorm = or_norm2(w, W, n);
    h[j + 1] = or_round(W, wnorm);
    int bad = !isfinite(wnorm);
    for (int i = 0; i <= j + 1; ++i) bad = bad || !isfinite(h[i]);
    if (bad) {
      res.diverged = 1;
      res.divergence_step = j;
      free(z);
      free(w);
      break;
    }
    const int happy = wnorm == 0.0;
    if (!happy) {
      or_scale(div_c(W, 1.0, or_round(W, wnorm)), w, W, n);
      V[nv++] = w;
    } else {
      free(w);
    }
    Z[j] = z;
    for (int i = 0; i < j; ++i) {
      const double t = add_c(W, mul_c(W, cs[i], h[i]), mul_c(W, sn[i], h[i + 1]));
      h[i + 1] = add_c(W, mul_c(W, -sn[i], h[i]), mul_c(W, cs[i], h[i + 1]));
      h[i] = t;
    }
    const double hj = h[j], hj1 = h[j + 1];
    const double rho = hypot_c(W, hj, hj1);
    if (rho == 0.0) {
      cs[j] = 1.0;
      sn[j] = 0.0;
    } else {
      cs[j] = div_c(W, hj, rho);
      sn[j] = div_c(W, hj1, rho);
    }
    h[j] = rho;
    h[j + 1] = 0.0;
    g[j + 1] = mul_c(W, -sn[j], g[j]);
    g[j] = mul_c(W, cs[j], g[j]);
    res.iterations++;
    const double estimate = fabs(g[j + 1]);
    res.est[res.n_est++] = estimate;
    res.residual_norm = estimate;
    if (happy) {
      res.happy = 1;
      break;
    }
    if (use_tol && estimate < rel_tol * bnorm) break;
  }
  const int k = res.iterations;
  if (k > 0) {
    double* y = (double*)calloc((size_t)k, sizeof(double));
    for (int i = k - 1; i >= 0; --i) {
      double acc = g[i];
      for (int l = i + 1; l < k; ++l) acc = sub_c(W, acc, mul_c(W, H[(size_t)l * (size_t)(m + 1) + (size_t)i], y[l]));
      y[i] = div_c(W, acc, H[(size_t)i * (size_t)(m + 1) + (size_t)i]);
    }
    for (int i = 0; i < k; ++i) or_axpy(y[i], Z[i], W, x, px, n);
    free(y);
  }
  for (int i = 0; i < nv; ++i) free(V[i]);
  for (int i = 0; i < m; ++i) free(Z[i]);
  free(V);
  free(Z);
  free(H);
  free(g);
  free(cs);
  free(sn);
  return res;
}

/* richardson_apply (src/richardson.cpp:10-54); wp = precision of z */
static void richardson(ctx_t* c, int d, int mk, uint64_t cycle_len, double* omegas, uint64_t* call_count,
                       uint64_t* update_count, uint64_t* degenerate, const double* v, int pv, double* z, int wp) {
  const uint64_t n = c->n;
  const int update_call = cycle_len != 0 && (*call_count % cycle_len) == 0;
  for (uint64_t i = 0; i < n; ++i) z[i] = 0.0;
  double* r = vnew(n);
  double* p = vnew(n);
  double* s = vnew(n);
  or_copy(v, pv, r, wp, n);
  for (int k = 0; k < mk; ++k) {
    if (k > 0) {
      multiply(c, d, z, wp, s, wp);
      or_add_scaled(v, pv, -1.0, s, wp, r, wp, n);
    }
    precondition(c, d, r, wp, p, wp);
    if (update_call) {
      multiply(c, d, p, wp, s, wp);
      const double num = or_dot(r, wp, s, wp, n, OR_P32);
      const double den = or_dot(s, wp, s, wp, n, OR_P32);
      if (den == 0.0 || !isfinite(num) || !isfinite(den)) {
        (*degenerate)++;
        or_axpy(omegas[k], p, wp, z, wp, n);
      } else {
        const int dp = maxp(OR_P32, wp);
        const double wprime = dp == OR_P32 ? (double)((float)num / (float)den) : num / den;
        or_axpy(wprime, p, wp, z, wp, n);
        const double done = (double)(*call_count / cycle_len - 1);
        omegas[k] = (done * omegas[k] + wprime) / (done + 1.0);
      }
    } else {
      or_axpy(omegas[k], p, wp, z, wp, n);
    }
  }
  if (update_call) (*update_count)++;
  (*call_count)++;
  free(r);
  free(p);
  free(s);
}

static void inner_solve(ctx_t* c, int d, const double* rhs, int prhs, double* out, int pout) {
  const or_level* L = &c->lv[d];
  c->level_inv[d]++;
  if (L->kind == 0) {
    for (uint64_t i = 0; i < c->n; ++i) out[i] = 0.0;
    cycle_res res = cycle(c, d, rhs, prhs, out, pout, L->m, 0, 0.0, 1);
    c->level_it[d] += (uint64_t)res.iterations;
    free(res.est);
  } else {
    richardson(c, d, L->m, L->cycle, c->omegas[d], &c->call_count[d], &c->update_count[d], &c->degenerate[d], rhs,
               prhs, out, pout);
    c->level_it[d] += (uint64_t)L->m;
  }
}

static void reset_rich(ctx_t* c, int d) {
  const or_level* L = &c->lv[d];
  for (int k = 0; k < L->m; ++k) c->omegas[d][k] = L->has_omega ? L->omega : 1.0;
  c->call_count[d] = 1;
  c->update_count[d] = 0;
  c->degenerate[d] = 0;
}

static double true_rel(ctx_t* c, const double* b, const double* x, int px, double bnorm) {
  const uint64_t n = c->n;
  double* x64 = vnew(n);
  double* ax = vnew(n);
  double* r = vnew(n);
  or_copy(x, px, x64, OR_P64, n);
  or_spmv(n, c->rp, c->ci, c->vals[OR_P64], OR_P64, x64, OR_P64, ax, OR_P64);
  or_add_scaled(b, OR_P64, -1.0, ax, OR_P64, r, OR_P64, n);
  const double t = or_norm2(r, OR_P64, n) / bnorm;
  free(x64);
  free(ax);
  free(r);
  return t;
}

static void push_hist(or_report* rep, double* hist, uint64_t cap, double v) {
  if (rep->n_history < cap) hist[rep->n_history] = v;
  rep->n_history++;
}

int or_solve(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals64, const or_level* levels,
             int nlevels, const double* b, double tol, int max_outer_restarts, uint64_t max_outer_total,
             int reset_richardson, double* x_out, double* history, uint64_t hist_cap, or_report* rep) {
  return or_solve_m(n, rp, ci, vals64, levels, nlevels, NULL, b, tol, max_outer_restarts, max_outer_total,
                    reset_richardson, x_out, history, hist_cap, rep);
}

int or_solve_m(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals64, const or_level* levels,
               int nlevels, const or_ilu* M, const double* b, double tol, int max_outer_restarts,
               uint64_t max_outer_total, int reset_richardson, double* x_out, double* history, uint64_t hist_cap,
               or_report* rep) {
  if (M && M->n != n) return 2;
  if (nlevels < 1 || nlevels > 16) return 3;
  for (int d = 0; d < nlevels; ++d)
    if (levels[d].m < 1) return 3;
  /* precision must not increase with depth (src/nesting.cpp:184-194) */
  for (int d = 1; d < nlevels; ++d)
    if (levels[d].pa > levels[d - 1].pa || levels[d].pv > levels[d - 1].pv) return 3;
  const uint64_t nnz = rp[n];
  double* v32 = (double*)malloc((nnz ? nnz : 1) * sizeof(double));
  double* v16 = (double*)malloc((nnz ? nnz : 1) * sizeof(double));
  for (uint64_t k = 0; k < nnz; ++k) {
    v32[k] = or_round(OR_P32, vals64[k]);
    v16[k] = or_round(OR_P16, vals64[k]);
  }
  ctx_t c;
  memset(&c, 0, sizeof c);
  c.n = n;
  c.rp = rp;
  c.ci = ci;
  c.vals[OR_P16] = v16;
  c.vals[OR_P32] = v32;
  c.vals[OR_P64] = vals64;
  c.lv = levels;
  c.D = nlevels;
  c.M = M;
  for (int d = 0; d < nlevels; ++d) {
    c.omegas[d] = (double*)calloc((size_t)levels[d].m, sizeof(double));
    reset_rich(&c, d);
  }
  memset(rep, 0, sizeof *rep);
  rep->n_levels = (uint64_t)nlevels;

  const int top_vec = levels[0].pv;
  double* x = vnew(n); /* at top_vec, zero */
  const double bnorm = or_norm2(b, OR_P64, n);
  if (bnorm == 0.0) {
    rep->converged = 1;
    push_hist(rep, history, hist_cap, 0.0);
  } else {
    push_hist(rep, history, hist_cap, 1.0);
    int executions = 0;
    const int max_exec = 1 + (max_outer_restarts > 0 ? max_outer_restarts : 0);
    if (levels[0].kind == 0) {
      const int m1 = levels[0].m;
      for (;;) {
        const uint64_t remaining = max_outer_total - rep->outer_iterations;
        if (remaining == 0) {
          strcpy(rep->flag, "capped");
          break;
        }
        const int len = (int)((uint64_t)m1 < remaining ? (uint64_t)m1 : remaining);
        c.level_inv[0]++;
        cycle_res res = cycle(&c, 0, b, OR_P64, x, top_vec, len, 1, tol, executions == 0);
        c.level_it[0] += (uint64_t)res.iterations;
        rep->outer_iterations += (uint64_t)res.iterations;
        for (int i = 1; i < res.n_est; ++i) push_hist(rep, history, hist_cap, res.est[i] / bnorm);
        const int diverged = res.diverged, step = res.divergence_step;
        const double rn = res.residual_norm;
        free(res.est);
        if (diverged) {
          snprintf(rep->flag, sizeof rep->flag, "divergence at outer step %d", step);
          break;
        }
        if (rn < tol * bnorm && true_rel(&c, b, x, top_vec, bnorm) < tol) {
          rep->converged = 1;
          break;
        }
        if (++executions >= max_exec) {
          strcpy(rep->flag, "capped");
          break;
        }
        if (reset_richardson)
          for (int d = 1; d < nlevels; ++d) reset_rich(&c, d);
      }
    } else {
      /* Richardson outermost (src/nesting.cpp:312-343) */
      const or_level* L = &levels[0];
      double* om = (double*)calloc((size_t)L->m, sizeof(double));
      for (int k = 0; k < L->m; ++k) om[k] = L->has_omega ? L->omega : 1.0;
      uint64_t cc = 1, uc = 0, dg = 0;
      double* r = vnew(n);
      double* z = vnew(n);
      double* ax = vnew(n);
      or_copy(b, OR_P64, r, top_vec, n);
      for (;;) {
        if (rep->outer_iterations >= max_outer_total) {
          strcpy(rep->flag, "capped");
          break;
        }
        c.level_inv[0]++;
        richardson(&c, 0, L->m, L->cycle, om, &cc, &uc, &dg, r, top_vec, z, top_vec);
        c.level_it[0] += (uint64_t)L->m;
        or_axpy(1.0, z, top_vec, x, top_vec, n);
        rep->outer_iterations++;
        multiply(&c, 0, x, top_vec, ax, top_vec);
        or_add_scaled(b, OR_P64, -1.0, ax, top_vec, r, top_vec, n);
        const double rel = or_norm2(r, top_vec, n) / bnorm;
        push_hist(rep, history, hist_cap, rel);
        if (!isfinite(rel)) {
          strcpy(rep->flag, "divergence");
          break;
        }
        if (rel < tol && true_rel(&c, b, x, top_vec, bnorm) < tol) {
          rep->converged = 1;
          break;
        }
      }
      free(om);
      free(r);
      free(z);
      free(ax);
    }
    rep->final_true_residual = true_rel(&c, b, x, top_vec, bnorm);
  }
  rep->precond_invocations = c.precond_invocations;
  for (int d = 0; d < nlevels; ++d) rep->level_iterations[d] = c.level_it[d];
  /* innermost Richardson weights (src/nesting.cpp:233-243): deepest inner level */
  for (int d = nlevels - 1; d >= 1; --d) {
    if (levels[d].kind == 1) {
      rep->n_omegas = (uint64_t)levels[d].m;
      for (int k = 0; k < levels[d].m && k < 64; ++k) rep->omegas[k] = c.omegas[d][k];
      break;
    }
  }
  if (x_out) or_copy(x, top_vec, x_out, OR_P64, n);
  free(x);
  for (int d = 0; d < nlevels; ++d) free(c.omegas[d]);
  free(v32);
  free(v16);
  return 0;
}

void or_richardson_apply(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals_p, int p, int m,
                         uint64_t cycle_len, double* omegas, uint64_t* counters, const double* v, double* z) {
  or_richardson_apply_m(n, rp, ci, vals_p, p, m, cycle_len, NULL, omegas, counters, v, z);
}

void or_richardson_apply_m(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals_p, int p, int m,
                           uint64_t cycle_len, const or_ilu* M, double* omegas, uint64_t* counters, const double* v,
                           double* z) {
  or_level lv = {1, m, p, p, cycle_len, 0, 0.0};
  ctx_t c;
  memset(&c, 0, sizeof c);
  c.n = n;
  c.rp = rp;
  c.ci = ci;
  c.vals[p] = vals_p;
  c.lv = &lv;
  c.D = 1;
  c.M = M;
  richardson(&c, 0, m, cycle_len, omegas, &counters[0], &counters[1], &counters[2], v, p, z, p);
}

int or_fgmres_cycle(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals_pa, int pa, int pw,
                    const double* b, double* x, int m, double rel_tol, int use_tol, int x_is_zero, int* iterations,
                    double* estimates, int* flags) {
  if (m < 1) return 3;
  or_level lv = {0, m, pa, pw, 0, 0, 0.0};
  ctx_t c;
  memset(&c, 0, sizeof c);
  c.n = n;
  c.rp = rp;
  c.ci = ci;
  c.vals[pa] = vals_pa;
  c.lv = &lv;
  c.D = 1;
  cycle_res res = cycle(&c, 0, b, pw, x, pw, m, use_tol, rel_tol, x_is_zero);
  *iterations = res.iterations;
  for (int i = 0; i < res.n_est; ++i) estimates[i] = res.est[i];
  flags[0] = res.happy;
  flags[1] = res.diverged;
  flags[2] = res.divergence_step;
  free(res.est);
  return 0;
}

/* ----------------------------------------------------------- spec grammar */

static int prec_tok(const char* s, int len) {
  if (len == 3 && !strncmp(s, "f64", 3)) return OR_P64;
  if (len == 3 && !strncmp(s, "f32", 3)) return OR_P32;
  if (len == 3 && !strncmp(s, "f16", 3)) return OR_P16;
  return -1;
}

static void trim(const char** s, const char** e) {
  while (*s < *e && (**s == ' ' || **s == '\t')) (*s)++;
  while (*e > *s && ((*e)[-1] == ' ' || (*e)[-1] == '\t')) (*e)--;
}

int or_parse_spec(const char* spec, or_level* levels, int cap) {
  int nl = 0;
  const char* p = spec;
  for (;;) {
    const char* e = strchr(p, '>');
    const char* end = e ? e : p + strlen(p);
    const char* s = p;
    trim(&s, &end);
    if (s == end) return -1;
    if (*s == 'F' || *s == 'R') {
      if (nl >= cap) return -1;
      or_level L;
      memset(&L, 0, sizeof L);
      L.kind = *s == 'R';
      L.cycle = 64;
      const char* colon = memchr(s, ':', (size_t)(end - s));
      if (!colon) return -1;
      char* num_end;
      L.m = (int)strtol(s + 1, &num_end, 10);
      if (num_end != colon || L.m < 1) return -1;
      const char* rest = colon + 1;
      if (!L.kind) {
        const char* slash = memchr(rest, '/', (size_t)(end - rest));
        if (!slash) return -1;
        const char *a0 = rest, *a1 = slash, *b0 = slash + 1, *b1 = end;
        trim(&a0, &a1);
        trim(&b0, &b1);
        L.pa = prec_tok(a0, (int)(a1 - a0));
        L.pv = prec_tok(b0, (int)(b1 - b0));
        if (L.pa < 0 || L.pv < 0) return -1;
      } else {
        const char* q = rest;
        int first = 1;
        while (q <= end) {
          const char* comma = memchr(q, ',', (size_t)(end - q));
          const char* qe = comma ? comma : end;
          const char *t0 = q, *t1 = qe;
          trim(&t0, &t1);
          if (first) {
            L.pa = L.pv = prec_tok(t0, (int)(t1 - t0));
            if (L.pa < 0) return -1;
            first = 0;
          } else {
            const char* eq = memchr(t0, '=', (size_t)(t1 - t0));
            if (!eq) return -1;
            const char *k0 = t0, *k1 = eq, *v0 = eq + 1, *v1 = t1;
            trim(&k0, &k1);
            trim(&v0, &v1);
            char buf[64];
            const size_t vl = (size_t)(v1 - v0) < sizeof buf - 1 ? (size_t)(v1 - v0) : sizeof buf - 1;
            memcpy(buf, v0, vl);
            buf[vl] = 0;
            if (k1 - k0 == 1 && *k0 == 'c') {
              L.cycle = strtoull(buf, NULL, 10);
            } else if (k1 - k0 == 5 && !strncmp(k0, "omega", 5)) {
              L.has_omega = 1;
              L.omega = strtod(buf, NULL);
            } else {
              return -1;
            }
          }
          if (!comma) break;
          q = comma + 1;
        }
      }
      levels[nl++] = L;
    } else {
      /* terminal: identity, ilu0(...) or ic0(...); like the reference's, it only
       * names M -- the caller passes the preconditioner itself */
      if (e) return -1;
      if (!(end - s == 8 && !strncmp(s, "identity", 8)) && strncmp(s, "ilu0", 4) && strncmp(s, "ic0", 3)) return -1;
    }
    if (!e) break;
    p = e + 1;
  }
  return nl > 0 ? nl : -1;
}
