// launch.hpp -- host-side launchers: map runtime precision tags (0 = f16, 1 = f32,
// 2 = f64) onto the kernel template instantiations. Implemented in launch_*.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace f3rg {

struct CsrDev;
struct TilesDev;
struct LevelState;
struct RichState;
struct StepInfo;
struct IoSlot;

struct GateH {
  const int* dead;
  int n;
};
struct SyncH {
  double* partials;
  unsigned* counter;
};

// cross-rank reduction stage (levels.cuh Dist); mode 0 = single rank
struct DistH {
  int mode = 0;
  int P = 1;
  double* loc = nullptr;
  const double* all = nullptr;
};

struct Launch {
  int grid = 0;  // 0: launcher picks (persistent, occupancy-sized)
  cudaStream_t stream = nullptr;
};

// grid used for streaming (BLAS-1 style) kernels and for tile kernels (per value
// precision and whether the kernel is the cooperative Richardson one)
int stream_grid();
// sequential index-order reductions (validation mode, common.cuh seq_sums): the
// value in effect when a kernel is launched or captured into a graph
int seq_reductions();
void set_seq_reductions(int on);
int max_partial_blocks();
int sm_count();

// ---- FGMRES level ------------------------------------------------------------------
cudaError_t launch_level_start(int ps, int pw, Launch l, void* src, const double* src_scale, int writeback, void* dst,
                               uint64_t n, LevelState* L, int* dead, GateH gate, int level, unsigned long long* cnt,
                               SyncH sync, const IoSlot* io, DistH dist = {});
cudaError_t launch_copy_scaled(int pw, Launch l, void* v, const double* scale, void* z, uint64_t n, GateH gate,
                               unsigned long long* cnt);
// dots: per-CTA partials (grid x 16 doubles); defer: leave their reduction to k_cgs.
// V: slot 0 of the basis (owned rows), ld: slot stride; z: the SpMV input (ext layout)
cudaError_t launch_spmv_dots(int pa, int pz, int pw, Launch l, const CsrDev& A, const TilesDev& T, const void* z,
                             void* V, uint64_t ld, int j, LevelState* L, GateH gate, SyncH sync, double* dots,
                             int defer, int* grid_out, DistH dist = {});
cudaError_t launch_multi_dot(int pw, Launch l, const void* V, uint64_t n, int j, int k0, LevelState* L, GateH gate,
                             SyncH sync, uint64_t ldv = 0, DistH dist = {});
cudaError_t launch_cgs(int pw, Launch l, void* V, uint64_t n, int j, LevelState* L, int* dead, GateH gate, int level,
                       int outer, int use_tol, StepInfo* info, SyncH sync, const double* dots, int dots_grid,
                       uint64_t ldv = 0, DistH dist = {});
cudaError_t launch_level_finish(int pz, int pw, int px, Launch l, const void* Z, uint64_t n, LevelState* L, void* x,
                                int x_is_zero, GateH gate, int level, unsigned long long* cnt, int count_iterations,
                                const IoSlot* io, uint64_t ldz = 0);
cudaError_t launch_residual(int pa, int px, int pw, Launch l, const CsrDev& A, const TilesDev& T, const void* x,
                            const double* b, void* r, LevelState* L, double* out_norm, SyncH sync, DistH dist = {});
cudaError_t launch_set_outer(Launch l, LevelState* L, double bnorm, double tol);

// ---- Richardson (cooperative) ----------------------------------------------------
cudaError_t launch_richardson(int pa, int pw, int pv, Launch l, const CsrDev& A, const TilesDev& T, const void* v,
                              const double* v_scale, void* out, uint64_t n, RichState* RS, GateH gate, int level,
                              unsigned long long* cnt, SyncH sync, unsigned* bar_count, unsigned* bar_gen,
                              const IoSlot* io, uint64_t voff = 0, int flags = 0);
// one phase of a partitioned Richardson call (richardson.cuh k_rich_phase, PH_*)
enum { PH_RESID_H = 0, PH_DOTS_H = 1, PH_UPDATE_H = 2, PH_BOOK_H = 3 };
cudaError_t launch_rich_phase(int pa, int pw, int pv, Launch l, const CsrDev& A, const TilesDev& T, int phase, int k,
                              const void* v, const double* v_scale, uint64_t off, void* out, uint64_t n,
                              RichState* RS, void* R, void* Za, GateH gate, int level, unsigned long long* cnt,
                              SyncH sync, DistH dist);

// ---- Richardson with a block-Jacobi ILU(0)/IC(0) M (richardson.cuh k_richm_phase) ----
enum { RM_START_H = 0, RM_RESID_H = 1, RM_DOTS_H = 2, RM_UPDATE_H = 3, RM_BOOK_H = 4 };
cudaError_t launch_richm_phase(int pa, int pw, int pv, Launch l, const CsrDev& A, const TilesDev& T, int phase, int k,
                               const void* v, const double* v_scale, void* out, uint64_t n, RichState* RS, void* R,
                               void* P, void* Za, GateH gate, int level, unsigned long long* cnt, SyncH sync);

// ---- block-Jacobi ILU(0)/IC(0) sweeps (trsv.cuh) ------------------------------------
struct SweepDev;
struct SweepCtl;
struct RichEpiH {
  const RichState* RS = nullptr;
  int k = 0;
  const void* zin = nullptr;
  void* zout = nullptr;
};
// forward sweep: t = L \ r (r at pin; factor precision pf; C = max(pf, pin))
cudaError_t launch_sweep_fwd(int pf, int pin, Launch l, const SweepDev& S, const void* r, void* cells,
                             unsigned* level_done, SweepCtl* ctl, GateH gate);
// backward sweep at compute precision pc: z = U \ t rounded to pout (+ fused Richardson update)
cudaError_t launch_sweep_bwd(int pf, int pc, int pout, Launch l, const SweepDev& S, const void* fcells, void* cells,
                             void* out, unsigned* level_done, SweepCtl* ctl, GateH gate, RichEpiH re);

// ---- fp64 CG / BiCGStab (krylov.cuh) ----------------------------------------------
struct KState;
int red_grid();
cudaError_t launch_cg_spmv(Launch l, const CsrDev& A, const TilesDev& T, const double* p, double* q, KState* S,
                           SyncH sync);
cudaError_t launch_cg_update(Launch l, double* x, double* r, const double* p, const double* q, uint64_t n, KState* S,
                             SyncH sync);
cudaError_t launch_cg_next(Launch l, KState* S);
cudaError_t launch_cg_rz(Launch l, const double* r, const double* z, uint64_t n, KState* S, SyncH sync);
cudaError_t launch_cg_p(Launch l, double* p, const double* r, uint64_t n, const KState* S);
cudaError_t launch_bi_rho(Launch l, const double* rhat, const double* r, uint64_t n, KState* S, SyncH sync);
cudaError_t launch_bi_p(Launch l, double* p, const double* v, const double* r, uint64_t n, const KState* S);
cudaError_t launch_bi_v(Launch l, const CsrDev& A, const TilesDev& T, const double* p, double* v, const double* rhat,
                        KState* S, SyncH sync);
cudaError_t launch_bi_s(Launch l, double* s, const double* r, const double* v, uint64_t n, const KState* S);
cudaError_t launch_bi_t(Launch l, const CsrDev& A, const TilesDev& T, const double* s, const double* shat, double* t,
                        KState* S, SyncH sync);
cudaError_t launch_bi_update(Launch l, double* x, double* r, const double* p, const double* s, const double* shat,
                             const double* t, uint64_t n, KState* S, SyncH sync);
cudaError_t launch_krylov_resume(Launch l, KState* S);

// ---- problem setup on the device (launch_setup.cu) ----------------------------------
// diagonal scaling in place: d_i = 1/sqrt|a_ii|, a_ij = (a_ij d_i) d_j; *bad = first
// row with a zero diagonal (the caller initialises it to ~0)
cudaError_t launch_diag_scale(Launch l, const uint32_t* rp, const uint32_t* ci, double* vals, const uint32_t* dpos,
                              double* d, uint64_t n, unsigned long long* bad);
cudaError_t launch_scale_rhs(Launch l, const double* b, const double* d, double* out, uint64_t n);

// ---- BLAS-1 / SpMV (kernel-level entry points) ----------------------------------
cudaError_t launch_fill(int p, Launch l, void* x, uint64_t n, double value);
cudaError_t launch_copy(int px, int py, Launch l, const void* x, void* y, uint64_t n);
cudaError_t launch_scale(int p, Launch l, double alpha, void* x, uint64_t n);
cudaError_t launch_axpy(int px, int py, Launch l, double alpha, const void* x, void* y, uint64_t n);
cudaError_t launch_add_scaled(int px, int py, int po, Launch l, const void* x, double alpha, const void* y, void* out,
                              uint64_t n);
// dot at C = max(floor, px, py) -> *out (device); norm: sqrt at precision px of the
// result rounded to px (norm2 semantics, x == y)
cudaError_t launch_dot(int px, int py, int floor_p, Launch l, const void* x, const void* y, uint64_t n, double* out,
                       SyncH sync, DistH dist = {});
cudaError_t launch_norm2(int px, Launch l, const void* x, uint64_t n, double* out, SyncH sync, DistH dist = {});
cudaError_t launch_permute_rows(Launch l, int esize, const uint32_t* rp_old, const uint32_t* rp_new,
                                const uint32_t* perm, const void* src, void* dst, uint64_t n);
// windowed SELL layout: out[e] = in[src[e]] (esize bytes, bit copy), or the pad
// (all ones if pad_ones, else zero) where src[e] == 0xffffffff
cudaError_t launch_ws_scatter(Launch l, int esize, const uint32_t* src, const void* in, void* out, uint64_t cnt,
                              bool pad_ones);
// windowed SELL layout: the encoded column stream of ring class cl (launch_setup.cu k_ws_encode)
cudaError_t launch_ws_encode(Launch l, const uint32_t* src, const uint32_t* ci, const uint32_t* soff,
                             const uint32_t* cwin, uint32_t G, uint64_t nsl, uint64_t n, int cl, uint32_t* out);
// packed windowed layout: out[e] = code[e] | fp16 bits of val16[src[e]] << 16 (+0 where src[e] == 0xffffffff)
cudaError_t launch_pk_pack(Launch l, const uint32_t* src, const uint16_t* code, const void* val16, uint32_t* out,
                           uint64_t cnt);
cudaError_t launch_pack16(Launch l, const void* val16, const uint16_t* dcol, uint32_t* out, uint64_t nnz);
// dst[i] = src[idx[i]], i < cnt, at precision p (halo pack / gather)
cudaError_t launch_gather(int p, Launch l, const void* src, const uint32_t* idx, uint64_t cnt, void* dst);
cudaError_t launch_spmv(int pa, int px, int py, Launch l, const CsrDev& A, const TilesDev& T, const void* x, void* y);

}  // namespace f3rg
