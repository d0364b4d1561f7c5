/* f3rg.h -- C ABI of the B200-native F3R hot path (fp64 FGMRES > fp32 FGMRES >
 * fp16-matrix FGMRES > fp16 Richardson, arXiv 2505.20719).
 *
 * This is the drop-in boundary for the reference's solve path. The reference is a
 * C++ library (/root/reference/proj); its per-vector virtuals
 * (LinearOperator::multiply/precondition, include/f3r/operator.hpp:19-27) run
 * ~10^4 times per solve, so the device boundary sits one level up, at the
 * ComposedSolver (include/f3r/nesting.hpp:55-77): one call solves the whole nest.
 * Kernel-level entry points replace the reference's BLAS-1/SpMV free functions and
 * are what the parity tests call. Plain pointers and sizes only; no torch types.
 *
 * Precision tags: 0 = binary16, 1 = binary32, 2 = binary64 (reference enum
 * f3r::Precision, include/f3r/precision.hpp:20).
 *
 * Error convention (reference include/f3r/errors.hpp:12-38): every function
 * returns 0 on success or one of the F3RG_E* codes, matching the exception class
 * the reference throws; f3rg_last_error() returns the message of the calling
 * thread's last failure. Non-convergence is NOT an error (reference
 * src/nesting.cpp:283-306): it is report.converged == 0 plus report.flag.
 *
 * Ownership (reference include/f3r/nesting.hpp:51-54): host arrays passed in are
 * borrowed for the duration of the call only; the library owns every device copy.
 * A solver handle is not re-entrant (one host thread at a time, Richardson weights
 * mutate), distinct handles may share one matrix handle and run concurrently.
 */
#ifndef F3RG_H
#define F3RG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  F3RG_OK = 0,
  F3RG_EDIMENSION = 2,     /* f3r::DimensionError */
  F3RG_ESOLVER = 3,        /* f3r::SolverError */
  F3RG_EPARSE = 4,         /* f3r::ParseError */
  F3RG_EFACTORIZATION = 5, /* f3r::FactorizationError */
  F3RG_ECUDA = 6,          /* CUDA runtime failure (no reference counterpart) */
  F3RG_EUNSUPPORTED = 7,   /* valid reference input not implemented on the device */
  F3RG_EINTERNAL = 9
};

enum { F3RG_P16 = 0, F3RG_P32 = 1, F3RG_P64 = 2 };
enum { F3RG_PRECOND_ILU0 = 0, F3RG_PRECOND_IC0 = 1, F3RG_PRECOND_IDENTITY = 2 };

typedef struct f3rg_matrix f3rg_matrix; /* SparseCsr + PrecisionReplicas on the device */
typedef struct f3rg_solver f3rg_solver; /* ComposedSolver on the device */

/* fp64 CSR in host memory; u32 indices (reference include/f3r/csr.hpp:23-67) */
typedef struct {
  uint64_t n;
  const uint32_t* row_ptr; /* n+1 */
  const uint32_t* col_idx; /* row_ptr[n] */
  const double* values;    /* row_ptr[n] */
} f3rg_csr;

/* reference RunOptions, include/f3r/nesting.hpp:29-38 */
typedef struct {
  double tol;
  int32_t max_outer_restarts;
  uint64_t max_outer_total;
  int32_t reset_richardson_on_restart;
} f3rg_run_options;

/* reference ConvergenceReport, include/f3r/report.hpp:18-30 (fixed-size view; the
 * variable-length fields are fetched with f3rg_solver_history / _level_iterations /
 * _omegas) */
typedef struct {
  int32_t converged;
  uint64_t outer_iterations;
  uint64_t precond_invocations;
  double final_true_residual;
  double wall_seconds;
  uint64_t n_history;
  uint64_t n_levels;
  uint64_t n_omegas;
  char flag[128];
} f3rg_report;

const char* f3rg_last_error(void);
const char* f3rg_version(void);
void f3rg_default_run_options(f3rg_run_options* opts); /* tol 1e-8, 3, 300, 0 */
/* Validation mode: every dot / norm of the single-GPU solve is summed sequentially in
 * index order, exactly as the reference's dot_core (src/vector_ops.cpp:20-28), instead
 * of the default fixed-shape tree. Slow (one dependent add per element); for parity
 * runs on long vectors. Applies to solvers and kernels launched (or graphs captured)
 * after the call; the default comes from F3RG_SEQ_REDUCTIONS. Returns the old value. */
int f3rg_set_seq_reductions(int on);

/* ---- matrices (replaces SparseCsr(...) + make_replicas, src/csr.cpp:40-69,130-136) */
int f3rg_matrix_create(f3rg_matrix** out, const f3rg_csr* a64);
void f3rg_matrix_destroy(f3rg_matrix* a);
uint64_t f3rg_matrix_rows(const f3rg_matrix* a);
uint64_t f3rg_matrix_nnz(const f3rg_matrix* a);
/* bytes one device pass over replica `prec` streams (values + the compressed column
 * stream in use + row pointers); the reference's u32 CSR is nnz*(s+4) + 4(n+1) */
uint64_t f3rg_matrix_stream_bytes(const f3rg_matrix* a, int prec);
/* SpMV engine the matrix was laid out for: 0 row tiles (regular), 1 row tiles (short
 * rows), 2 row tiles over the row-sorted copy (gather-bound), 3 windowed SELL
 * (gather-bound, square, one rank); F3RG_SHAPE / F3RG_SORT_ROWS / F3RG_WSELL force */
int f3rg_matrix_engine(const f3rg_matrix* a);
/* Host-side self-check of the packed windowed SELL layout (csrc/wsell_pk_layout.hpp) the fp16
 * passes of engine 3 stream: builds the layout of the CSR pattern for `ctas` CTAs (no GPU needed)
 * and decodes every row back -- slot codes, escape pairs of far columns, padding -- against the
 * CSR row, in order. stats (4 values, may be null): slots, far entries, slices, padding slots.
 * Returns 0, or F3RG_EDIMENSION with the first mismatch in f3rg_last_error(). */
int f3rg_wsell_pk_selfcheck(uint64_t n, const uint32_t* row_ptr, const uint32_t* col_idx, uint32_t ctas,
                            uint64_t* stats);
/* replica values widened to fp64 into host memory (nnz doubles) */
int f3rg_matrix_values(const f3rg_matrix* a, int prec, double* out_host);

/* ---- problem setup -------------------------------------------
 * f3rg_matrix_create_scaled: diagonal_scale(A, b) (src/scaling.cpp:11-38) computed on
 * the device from the UNSCALED fp64 CSR -- d_i = 1/sqrt|a_ii|, a~_ij = (a_ij d_i) d_j,
 * b~ = b d, bit-identical to the reference -- and the replicas of the scaled matrix.
 * b_host / b_scaled_host / d_host (n each) are optional. F3RG_EFACTORIZATION on a
 * missing or zero diagonal, with the reference's message. */
int f3rg_matrix_create_scaled(f3rg_matrix** out, const f3rg_csr* a64, const double* b_host, double* b_scaled_host,
                              double* d_host);
/* Matrix Market coordinate files (read_matrix_market / write_matrix_market,
 * src/matrix_market.cpp:33-127): real / integer / pattern, general / symmetric;
 * F3RG_EPARSE with the reference's messages. The host CSR is owned by the handle;
 * f3rg_host_csr_view points an f3rg_csr at its arrays. */
typedef struct f3rg_host_csr f3rg_host_csr;
int f3rg_read_matrix_market(const char* path, f3rg_host_csr** out);
int f3rg_host_csr_view(const f3rg_host_csr* h, f3rg_csr* view);
uint64_t f3rg_host_csr_nnz(const f3rg_host_csr* h);
void f3rg_host_csr_destroy(f3rg_host_csr* h);
int f3rg_write_matrix_market(const char* path, const f3rg_csr* a64);

/* ---- solver spec grammar (replaces parse_solver_spec / SolverSpec::to_string,
 *      src/solver_spec.cpp:147-212) */
int f3rg_spec_canonical(const char* spec, char* out, size_t cap);

/* ---- primary preconditioner M (replaces IdentityPrecond and
 *      BlockJacobiIlu0::factorize / apply, include/f3r/ilu.hpp:25-84,
 *      src/ilu.cpp:33-263). The factorisation runs on the host at fp64 exactly as
 *      the reference's; the triangular sweeps of apply run on the device, bit-exact
 *      (level-scheduled, sync-free). Errors: F3RG_EFACTORIZATION with the
 *      reference's message (missing diagonal, zero / non-positive pivot, a pivot
 *      lost in the cast to the apply precision, nblocks / alpha out of range). */
typedef struct f3rg_precond f3rg_precond;
/* reference IluConfig, include/f3r/ilu.hpp:44-49 */
typedef struct {
  uint64_t nblocks;
  double alpha;
  int32_t symmetric;       /* 1: IC(0), 0: ILU(0) */
  int32_t apply_precision; /* F3RG_P16 / _P32 / _P64 */
} f3rg_ilu_config;
int f3rg_ilu_factorize(f3rg_precond** out, const f3rg_csr* a64, const f3rg_ilu_config* cfg);
int f3rg_precond_identity(f3rg_precond** out, uint64_t n);
void f3rg_precond_destroy(f3rg_precond* m);
uint64_t f3rg_precond_rows(const f3rg_precond* m);
/* config (nblocks 0 = identity), sweep depths levels[2] (forward, backward) and
 * block_ranges (nblocks + 1 row offsets, up to cap); any output may be NULL */
int f3rg_precond_info(const f3rg_precond* m, f3rg_ilu_config* cfg, uint32_t* levels, uint32_t* block_ranges,
                      uint64_t cap);
/* Preconditioner::apply: z = M r; device vectors r (prec_r) and z (prec_z); computes
 * at promote(apply_precision, prec_r) like the reference */
int f3rg_precond_apply(const f3rg_precond* m, const void* r, int prec_r, void* z, int prec_z, uintptr_t stream);
/* the host factorisation alone (no device work): stored factors as the reference
 * keeps them -- lower (IC: diagonal last in each row) and upper (ILU: diagonal
 * first). Call with NULL arrays for the sizes; lp / up have n + 1 entries. */
int f3rg_ilu_factorize_host(const f3rg_csr* a64, const f3rg_ilu_config* cfg, uint64_t* nnz_lower,
                            uint64_t* nnz_upper, uint32_t* lp, uint32_t* li, double* lv, uint32_t* up, uint32_t* ui,
                            double* uv);

/* ---- composed solver (replaces build(spec, replicas, M) + ComposedSolver::run,
 *      src/nesting.cpp:176-352,354-357).
 *      f3rg_solver_create_m: with a preconditioner from f3rg_ilu_factorize /
 *      f3rg_precond_identity (shared: it may be destroyed before the solver).
 *      f3rg_solver_create: IDENTITY, or ILU0/IC0 factorised here from the spec
 *      terminal's parameters with the reference bench's defaults (blocks 4,
 *      alpha 1, f64; src/bench.cpp:150-177). */
int f3rg_solver_create(f3rg_solver** out, const f3rg_matrix* a, const char* spec, int precond_kind);
int f3rg_solver_create_m(f3rg_solver** out, const f3rg_matrix* a, const char* spec, const f3rg_precond* m);
void f3rg_solver_destroy(f3rg_solver* s);
const char* f3rg_solver_id(const f3rg_solver* s);
/* b, x: HOST fp64 arrays of length n (x may be NULL); copies happen inside */
int f3rg_solve(f3rg_solver* s, const double* b_host, double* x_host, const f3rg_run_options* opts,
               f3rg_report* rep);
/* b, x: DEVICE fp64 arrays (x may be NULL); stream: cudaStream_t or 0 (own stream) */
int f3rg_solve_device(f3rg_solver* s, const double* b_dev, double* x_dev, const f3rg_run_options* opts,
                      f3rg_report* rep, uintptr_t stream);
/* restore a freshly built solver's state (Richardson weights and call counters,
 * include/f3r/richardson.hpp:26-46; they persist across solves exactly as in the
 * reference's ComposedSolver); stream-ordered on `stream` (0 = own stream) */
int f3rg_solver_reset_state(f3rg_solver* s, uintptr_t stream);
/* report vectors of the LAST solve (host memory, up to cap entries) */
int f3rg_solver_history(const f3rg_solver* s, double* out, uint64_t cap);
int f3rg_solver_level_iterations(const f3rg_solver* s, uint64_t* out, uint64_t cap);
int f3rg_solver_omegas(f3rg_solver* s, double* out, uint64_t cap); /* innermost_omegas() */
uint64_t f3rg_solver_omega_count(const f3rg_solver* s);           /* its length (0: no Richardson level) */
/* per-kernel timing of the next solve (CUDA events around each launch; the solve
 * runs eagerly instead of through the captured graph) */
int f3rg_solver_set_profile(f3rg_solver* s, int on);
/* kernel i of the last profiled solve: name, total ms, launches, algorithmic bytes */
int f3rg_solver_profile_entry(const f3rg_solver* s, uint64_t i, char* name, size_t cap, double* ms,
                              uint64_t* launches, double* bytes);
/* row-block partition: halo exchanges and cross-rank reductions (allgathers) the last
 * profiled solve enqueued on this rank (0 on one rank) */
int f3rg_solver_collectives(const f3rg_solver* s, uint64_t* halos, uint64_t* reductions);

/* ---- kernel-level entry points (device pointers, stream = cudaStream_t or 0) ---
 * Each mirrors one reference free function, same argument meaning. */
int f3rg_spmv(const f3rg_matrix* a, int prec_a, const void* x, int prec_x, void* y, int prec_y,
              uintptr_t stream); /* spmv, src/csr.cpp:138-147 */
int f3rg_dot(const void* x, int prec_x, const void* y, int prec_y, uint64_t n, int floor_prec, double* out_host,
             uintptr_t stream); /* dot_at_least, src/vector_ops.cpp:154-164 */
int f3rg_norm2(const void* x, int prec_x, uint64_t n, double* out_host, uintptr_t stream); /* norm2 :166 */
int f3rg_axpy(double alpha, const void* x, int prec_x, void* y, int prec_y, uint64_t n,
              uintptr_t stream); /* axpy :114 */
int f3rg_add_scaled(const void* x, int prec_x, double alpha, const void* y, int prec_y, void* out, int prec_out,
                    uint64_t n, uintptr_t stream); /* add_scaled :131 */
int f3rg_copy(const void* x, int prec_x, void* y, int prec_y, uint64_t n, uintptr_t stream); /* copy_into :87 */
int f3rg_scale(double alpha, void* x, int prec_x, uint64_t n, uintptr_t stream);            /* scale_in_place :104 */
int f3rg_fill(void* x, int prec_x, uint64_t n, double value, uintptr_t stream);             /* fill :77 */

/* ---- Richardson with persistent state (richardson_apply + RichardsonState,
 *      src/richardson.cpp:10-54, include/f3r/richardson.hpp:26-46); M = identity
 *      unless f3rg_richardson_set_precond names one */
typedef struct f3rg_richardson f3rg_richardson;
int f3rg_richardson_create(f3rg_richardson** out, const f3rg_matrix* a, int prec, int m, uint64_t cycle);
void f3rg_richardson_destroy(f3rg_richardson* r);
int f3rg_richardson_set_omegas(f3rg_richardson* r, const double* omegas_host);
/* omegas[m]; counters[3] = call_count, update_count, degenerate_events */
int f3rg_richardson_state(f3rg_richardson* r, double* omegas_host, uint64_t* counters_host);
/* v, z: device vectors at the Richardson precision */
int f3rg_richardson_apply(f3rg_richardson* r, const void* v, void* z, uintptr_t stream);
/* op.precondition = M for the following applies (NULL: identity again); the
 * RichardsonInner-over-PrimarySolver operator of src/nesting.cpp:46-83 */
int f3rg_richardson_set_precond(f3rg_richardson* r, const f3rg_precond* m);

/* ---- the reference's fp64 competitor solvers (src/cg.cpp:22-171: cg_solve,
 *      bicgstab_solve) on the device; f3rg_krylov_solve: M = identity. which: 0 = CG, 1 = BiCGStab.
 *      b, x: HOST fp64 arrays (x may be NULL). history (optional, hist_cap entries)
 *      receives the relative residuals, entry 0 = 1 (ConvergenceReport semantics).
 *      CG on an indefinite operator returns F3RG_ESOLVER, as the reference throws
 *      SolverError; breakdown / cap are report flags ("breakdown", "capped"). */
int f3rg_krylov_solve(const f3rg_matrix* a, int which, const double* b_host, double* x_host, double tol,
                      uint64_t max_precond_invocations, f3rg_report* rep, double* history, uint64_t hist_cap);
/* the same with the preconditioner M (cg_solve / bicgstab_solve(a, M, b, opts)): m from
 * f3rg_ilu_factorize / f3rg_precond_identity, NULL = identity */
int f3rg_krylov_solve_m(const f3rg_matrix* a, const f3rg_precond* m, int which, const double* b_host, double* x_host,
                        double tol, uint64_t max_precond_invocations, f3rg_report* rep, double* history,
                        uint64_t hist_cap);

/* ---- the reference's restarted fp64 FGMRES(m) with a terminal preconditioner
 *      (src/fgmres.cpp:163-222: fgmres_restarted; the bench's "fgmres64"). Cycles of
 *      `restart` steps from the current iterate until tol (estimate AND fp64 true
 *      residual) or max_precond_invocations applications of M ("capped"). m: a
 *      preconditioner from f3rg_precond_identity / f3rg_ilu_factorize. */
int f3rg_fgmres_solve(const f3rg_matrix* a, const f3rg_precond* m, int restart, const double* b_host, double* x_host,
                      double tol, uint64_t max_precond_invocations, f3rg_report* rep, double* history,
                      uint64_t hist_cap);

/* ---- row-block partition over P ranks ---------
 * Rows split by the reference's rule (src/ilu.cpp:47-54: base = n/P, remainder to the
 * leading blocks). Each rank keeps its rows of A and of every Krylov vector; SpMV
 * inputs use the rank's "ext" layout [pad | lo halo | owned | hi halo] (halo = remote
 * columns referenced by its rows, ascending); dots/norms are rank-local sums combined
 * in rank order, so every rank holds bitwise-identical Hessenberg/Givens scalars. */
typedef struct {
  uint64_t r0, r1;         /* owned rows */
  uint64_t n_lo, n_hi;     /* halo entries below / above the owned rows */
  uint64_t pad, off;       /* ext layout: owned rows start at off = pad + n_lo */
  uint64_t n_ext, ld;      /* ext length; vector stride of a basis */
  uint64_t nnz_local;      /* nonzeros of the owned rows */
  uint64_t nnz_begin;      /* global position of the first of them */
  uint64_t n_send;         /* total entries this rank sends per halo exchange */
} f3rg_part_info;

/* rank `rank`'s plan (host only, no device work). Optional outputs (NULL to skip):
 * halo[n_lo + n_hi] global columns; recv_off/recv_cnt/send_cnt[P]; send_idx[n_send]
 * owned-local indices, peers in rank order; local_rp[r1 - r0 + 1]; local_ci[nnz_local]
 * (ext columns) */
int f3rg_part_plan(const f3rg_csr* a, int P, int rank, f3rg_part_info* info, uint32_t* halo, uint64_t* recv_off,
                   uint64_t* recv_cnt, uint64_t* send_cnt, uint32_t* send_idx, uint32_t* local_rp,
                   uint32_t* local_ci);

typedef struct f3rg_comm f3rg_comm;
/* P ranks as host threads of this process, all on the current device, one stream
 * (the one-GPU test vehicle of the partition; data flow as with NCCL) */
int f3rg_comm_local(f3rg_comm** out, const f3rg_csr* a, int P);
/* one rank per process over NCCL (libnccl.so.2 resolved at run time; F3RG_NCCL_LIB
 * overrides). unique_id: 128 bytes from f3rg_nccl_unique_id on one rank, shared. */
int f3rg_nccl_unique_id(void* out128);
int f3rg_comm_nccl(f3rg_comm** out, const f3rg_csr* a, int P, int rank, const void* unique_id);
void f3rg_comm_destroy(f3rg_comm* c);
/* a ComposedSolver over rank `rank`'s rows (a: the GLOBAL fp64 CSR, host) */
int f3rg_solver_create_part(f3rg_solver** out, f3rg_comm* c, const f3rg_csr* a, const char* spec, int precond_kind,
                            int rank);
/* local communicator: solve with all P rank solvers (one host thread each); b, x:
 * global host vectors; reps[P] */
int f3rg_solve_local(f3rg_comm* c, f3rg_solver** solvers, const double* b_host, double* x_host,
                     const f3rg_run_options* opts, f3rg_report* reps);
/* NCCL communicator: this rank's solve; b_own, x_own: device vectors of its rows */
int f3rg_solve_part_device(f3rg_solver* s, const double* b_own, double* x_own, const f3rg_run_options* opts,
                           f3rg_report* rep, uintptr_t stream);
/* y = A x through the partition (P rank-local SpMVs on the current device after a
 * halo exchange); x, y: global host fp64 vectors, values rounded to px / from py */
int f3rg_local_spmv(const f3rg_csr* a, int P, int pa, int px, int py, const double* x_host, double* y_host);

#ifdef __cplusplus
}
#endif
#endif /* F3RG_H */
