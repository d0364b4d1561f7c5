/* f3rg_problems.h -- host-side synthetic problem generators for the five
 * BASELINE.json configurations and the reference's HPCG/HPGMP
 * stencil (src/stencil.cpp:55-101). Setup code, untimed; not part of the solve
 * boundary. All follow the reference conventions: lexicographic x-fastest
 * numbering, strictly increasing columns per row, out-of-grid neighbours omitted,
 * SplitMix64 streams (include/f3r/rng.hpp:15-32), symmetric diagonal scaling
 * D^-1/2 A D^-1/2 (src/scaling.cpp:11-38). */
#ifndef F3RG_PROBLEMS_H
#define F3RG_PROBLEMS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct f3rg_problem f3rg_problem;

enum {
  F3RG_GEN_POISSON7 = 1,     /* config 1: diag 6, off -1 (nx, ny, nz) */
  F3RG_GEN_STENCIL27 = 2,    /* config 2: reference generate_stencil (nx, ny, nz powers of 2; beta) */
  F3RG_GEN_CONVDIFF7 = 3,    /* config 3: upwind, cell Peclet 0.5: diag 9, upwind -2, downwind -1 */
  F3RG_GEN_ANISO7 = 4,       /* config 4: k = exp(N(0, 1.5^2)) per face, z faces x1e-2 */
  F3RG_GEN_UNSTRUCTURED = 5  /* config 5: lognormal row lengths, banded Gaussian + 5% long range */
};

/* Generates the fp64 matrix A (unscaled) of `kind`. grid[3] = (nx, ny, nz) for the
 * stencils, grid[0] = n for UNSTRUCTURED. param: beta (STENCIL27), ignored otherwise.
 * seed: the problem's random stream (ANISO7 face field, UNSTRUCTURED pattern). */
int f3rg_problem_generate(f3rg_problem** out, int kind, const uint64_t grid[3], double param, uint64_t seed);
void f3rg_problem_destroy(f3rg_problem* p);

/* right-hand side: mode 0 -> x_true_i = 2u-1 from SplitMix64(seed), b = A x_true;
 * then (A, b) <- diagonal_scale(A, b).  mode 1 -> scale A first, b = A~ * 1. */
int f3rg_problem_finalize(f3rg_problem* p, int mode, uint64_t seed);

/* views owned by the handle (valid until destroy) */
int f3rg_problem_arrays(const f3rg_problem* p, uint64_t* n, uint64_t* nnz, const uint32_t** row_ptr,
                        const uint32_t** col_idx, const double** values, const double** b, const double** d);

#ifdef __cplusplus
}
#endif
#endif
