/* oracle/f3r_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's hot-path arithmetic (the CPU oracle the
 * CUDA path is checked against). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it; the product never does.
 *
 * Parity pin: every function here is checked bit-for-bit against the UNMODIFIED
 * reference (oracle/_ref/libf3r_ref.so, built from /root/reference/proj/src by
 * oracle/Makefile) through golden vectors in tests/golden/ (made by
 * tests/golden/make_golden.py) -- see tests/test_oracle_golden.py.
 *
 * Conventions: a vector is a double array whose entries are exactly
 * representable at its precision tag (0 = binary16, 1 = binary32, 2 = binary64);
 * every store rounds (RNE, no flush-to-zero) to the destination's precision.
 */
#ifndef F3R_ORACLE_H
#define F3R_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_P16 = 0, OR_P32 = 1, OR_P64 = 2 };

/* binary16 conversions (reference include/f3r/half.hpp:27-100) */
uint16_t or_half_from_double(double x);
uint16_t or_half_from_float(float x);
float or_float_from_half(uint16_t h);
double or_round(int p, double x); /* demote(x, p) of include/f3r/precision.hpp:64-70 */

/* BLAS-1 and SpMV (reference src/vector_ops.cpp, src/csr.cpp:23-37) */
void or_spmv(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals, int pa, const double* x,
             int px, double* y, int py);
double or_dot(const double* x, int px, const double* y, int py, uint64_t n, int floor_p);
void or_set_pairwise_dots(int on); /* experiments: pairwise instead of sequential dots */
double or_norm2(const double* x, int px, uint64_t n);
void or_axpy(double alpha, const double* x, int px, double* y, int py, uint64_t n);
void or_add_scaled(const double* x, int px, double alpha, const double* y, int py, double* out, int po,
                   uint64_t n);
void or_copy(const double* x, int px, double* y, int py, uint64_t n);
void or_scale(double alpha, double* x, int px, uint64_t n);

/* Block-Jacobi ILU(0)/IC(0) primary preconditioner (reference src/ilu.cpp:38-263).
 * or_ilu_factorize returns 0, or 5 (FactorizationError) with the reference's
 * message in err. Factor values are exactly representable at `prec`. */
typedef struct or_ilu or_ilu;
int or_ilu_factorize(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals, uint64_t nblocks,
                     double alpha, int symmetric, int prec, or_ilu** out, char* err, size_t errcap);
void or_ilu_free(or_ilu* m);
void or_ilu_apply(const or_ilu* m, const double* r, int pr, double* z, int pz);
/* stored factors: upper = 0 the lower factor (IC: with its diagonal last), 1 the
 * upper factor (ILU, diagonal first) */
uint64_t or_ilu_count(const or_ilu* m, int upper);
void or_ilu_export(const or_ilu* m, int upper, uint32_t* ptr, uint32_t* idx, double* vals);

/* Nested solver (reference src/nesting.cpp, src/fgmres.cpp, src/richardson.cpp)
 * with the primary preconditioner M = identity (or_solve) or a block-Jacobi
 * ILU(0)/IC(0) (or_solve_m, M != NULL). */
typedef struct {
  int kind; /* 0 = FGMRES, 1 = Richardson */
  int m;
  int pa; /* matrix precision */
  int pv; /* vector precision (Richardson: both) */
  uint64_t cycle;
  int has_omega;
  double omega;
} or_level;

typedef struct {
  int converged;
  uint64_t outer_iterations;
  uint64_t precond_invocations;
  double final_true_residual;
  uint64_t n_levels;
  uint64_t level_iterations[16];
  uint64_t n_history;
  uint64_t n_omegas;
  double omegas[64];
  char flag[128];
} or_report;

/* Parses the reference grammar (include/f3r/solver_spec.hpp:9-15) into levels;
 * returns the level count, or -1 on a parse error. The terminal must be
 * `identity` or absent. */
int or_parse_spec(const char* spec, or_level* levels, int cap);

/* Solve A x = b with the nest `levels` (matrix given at fp64; lower replicas are
 * element-wise RNE demotions, src/csr.cpp:83-92). history has room for hist_cap
 * entries. Returns 0 on success, nonzero on a contract error. */
int or_solve(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals64, const or_level* levels,
             int nlevels, const double* b, double tol, int max_outer_restarts, uint64_t max_outer_total,
             int reset_richardson, double* x_out, double* history, uint64_t hist_cap, or_report* rep);

int or_solve_m(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals64, const or_level* levels,
               int nlevels, const or_ilu* M, const double* b, double tol, int max_outer_restarts,
               uint64_t max_outer_total, int reset_richardson, double* x_out, double* history, uint64_t hist_cap,
               or_report* rep);

void or_richardson_apply_m(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals_p, int p, int m,
                           uint64_t cycle_len, const or_ilu* M, double* omegas, uint64_t* counters, const double* v,
                           double* z);

/* One richardson_apply with (A_p, M = I) and a persistent state
 * (src/richardson.cpp:10-54). state layout: omegas[m], then counters
 * call_count, update_count, degenerate (as doubles). */
void or_richardson_apply(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals_p, int p, int m,
                         uint64_t cycle, double* omegas, uint64_t* counters, const double* v, double* z);

/* One fgmres_cycle (src/fgmres.cpp:21-161) against (A_pa, M = I), vectors at pw. */
int or_fgmres_cycle(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals_pa, int pa, int pw,
                    const double* b, double* x, int m, double rel_tol, int use_tol, int x_is_zero, int* iterations,
                    double* estimates, int* flags);

#ifdef __cplusplus
}
#endif
#endif
