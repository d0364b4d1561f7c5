// engine.hpp -- host-side C++ of the f3rg engine: error classes, the solver-spec
// grammar, device-resident CSR replicas with their tile tables, and the composed
// solver that drives the device level chain. The public boundary is the C ABI in
// include/f3rg.h (capi.cpp); this header is internal.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "partition.hpp"
#include "precond.hpp"
#include "state.hpp"

namespace f3rg {

// error codes shared with include/f3rg.h
enum ErrCode {
  ERR_OK = 0,
  ERR_DIMENSION = 2,      // f3r::DimensionError
  ERR_SOLVER = 3,         // f3r::SolverError
  ERR_PARSE = 4,          // f3r::ParseError
  ERR_FACTORIZATION = 5,  // f3r::FactorizationError
  ERR_CUDA = 6,           // CUDA runtime failure (no reference counterpart)
  ERR_UNSUPPORTED = 7,    // valid reference input this device build does not implement
  ERR_INTERNAL = 9
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what);
#define F3RG_CUDA(x) ::f3rg::cuda_check((x), #x)

// ---- device memory ----------------------------------------------------------------
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t bytes) { alloc(bytes); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr, o.n_ = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_, n_ = o.n_;
      o.p_ = nullptr, o.n_ = 0;
    }
    return *this;
  }
  void alloc(size_t bytes);
  void release();
  template <class T = void>
  T* get() const {
    return static_cast<T*>(p_);
  }
  size_t bytes() const { return n_; }

 private:
  void* p_ = nullptr;
  size_t n_ = 0;
};

// ---- solver spec (reference include/f3r/solver_spec.hpp:30-62) ---------------------
enum LevelKind { LK_FGMRES = 0, LK_RICHARDSON = 1 };
enum PrecondKind { PK_ILU0 = 0, PK_IC0 = 1, PK_IDENTITY = 2 };

struct LevelSpec {
  int kind = LK_FGMRES;
  int m = 1;
  int pa = 2;  // matrix precision (Richardson: its one precision)
  int pv = 2;  // vector precision
  unsigned long long cycle = 64;
  bool has_omega = false;
  double omega = 1.0;
};

struct PrecondSpec {
  bool has_kind = false;
  int kind = PK_ILU0;
  bool has_blocks = false;
  unsigned long long blocks = 0;
  bool has_alpha = false;
  double alpha = 1.0;
  bool has_prec = false;
  int prec = 2;
};

struct Spec {
  std::vector<LevelSpec> levels;
  bool has_precond = false;
  PrecondSpec precond;
  std::string to_string() const;  // canonical form (src/solver_spec.cpp:165-212)
};

Spec parse_spec(const std::string& text);  // throws Error(ERR_PARSE)
const char* precision_name(int p);

// ---- tiles ----------------------------------------------------------------------------
// Contiguous row ranges with <= max_rows rows and <= max_nnz nonzeros; a row longer
// than max_nnz forms its own tile. Outputs r0/k0 of length ntiles+1.
void build_tiles(uint64_t n, const uint32_t* rp, uint32_t max_rows, uint32_t max_nnz, std::vector<uint32_t>& r0,
                 std::vector<uint32_t>& k0);
uint32_t tile_max_nnz(int pa, int shape = 0);
uint32_t tile_max_rows();

// ---- device matrix (reference SparseCsr + PrecisionReplicas, include/f3r/csr.hpp) ----
class DeviceMatrix {
 public:
  // validates like SparseCsr::validate (src/csr.cpp:51-69) and uploads one shared
  // index copy plus the fp64 / fp32 / fp16 value replicas (RNE demotions, :83-92).
  // ncols > n: a rank's rows of a partitioned matrix, columns in its ext layout
  DeviceMatrix(uint64_t n, const uint32_t* row_ptr, const uint32_t* col_idx, const double* values,
               uint64_t ncols = 0);
  // the same for diagonal_scale(A) (src/scaling.cpp:11-38) computed on the device from
  // the unscaled values: the replicas are those of the scaled matrix; d (n) is left
  // in d_dev (device, may be null). Throws Error(ERR_FACTORIZATION) like the reference
  struct Scale {
    double* d_dev = nullptr;
  };
  DeviceMatrix(uint64_t n, const uint32_t* row_ptr, const uint32_t* col_idx, const double* values, Scale scale);
  uint64_t rows() const { return n_; }
  uint64_t nnz() const { return nnz_; }
  // the CSR the tile kernels stream, always paired with tiles(p): the row-sorted
  // copy when the matrix has one (tiles(p).perm), else the matrix as uploaded
  CsrDev csr() const;
  CsrDev csr_plain() const;  // the matrix in its own row order
  TilesDev tiles(int p) const;
  bool sorted_rows() const { return perm_.get() != nullptr; }
  const void* values(int p) const { return val_[p].get(); }
  bool d16() const { return dcol_.get() != nullptr; }  // 16-bit delta column stream in use
  // bytes one pass over replica pa streams: values, the column stream in use, row_ptr
  double stream_bytes(int pa) const;
  int shape() const { return shape_; }  // 0 regular, 1 short rows, 2 gather-bound, 3 windowed SELL
  uint64_t ws_entries() const { return ws_E_; }
  uint64_t pk_slots() const { return pk_E_; }  // slots of the packed layout (0: none)  // stored entries of the windowed layout (0: none)

 private:
  void init(const uint32_t* row_ptr, const uint32_t* col_idx, const double* values, uint64_t ncols,
            const Scale* scale);
  uint64_t n_ = 0, nnz_ = 0;
  DevBuf rp_, ci_, val_[3], tr0_[3], tk0_[3], dcol_, first_, pk_;
  DevBuf perm_, srp_, sci_, sval_[3], sdcol_, sfirst_, spk_;  // row-sorted copy (irregular rows)
  DevBuf ws_soff_, ws_row_, ws_enc_[3], ws_val_[3], ws_cwin_;  // windowed SELL layout (shape 3)
  uint64_t ws_E_ = 0;
  uint32_t ws_G_ = 0;
  void build_wsell(const uint32_t* row_ptr);
  // packed layout of the fp16 replica for the 2-byte-ring passes (wsell_pk_layout.hpp)
  DevBuf pk_soff_, pk_row_, pk_words_, pk_cwin_;
  uint64_t pk_E_ = 0, pk_far_ = 0;
  // ... and the class-1 layout (4-byte rings) of all three replicas: codes + values
  DevBuf pk1_soff_, pk1_row_, pk1_cwin_, pk1_code_, pk1_val_[3];
  uint64_t pk1_E_ = 0;
  void build_wsell_pk(const uint32_t* row_ptr, const uint32_t* col_idx);
  uint32_t ntiles_[3] = {0, 0, 0};
  uint32_t l2hint_ = 0;  // L2 eviction priorities for the passes (init)
  int shape_ = 0;
};

void validate_csr(uint64_t n, const uint32_t* rp, const uint32_t* ci, uint64_t ncols = 0);

// ---- cross-rank exchange of the row-block partition ------------
// Every rank calls the same sequence of halo()/allgather() (its host control flow
// depends only on replicated scalars), so the exchanges always pair up.
class Exchange {
 public:
  virtual ~Exchange() = default;
  virtual int size() const = 0;
  virtual int rank() const = 0;
  virtual const PartPlan& plan() const = 0;
  // fill the halo entries of an ext-layout vector (precision prec) from the peers
  virtual void halo(void* ext, int prec, cudaStream_t s) = 0;
  // loc[0..16) of every rank -> all[r * 16 + k]; then the caller launches the tail;
  // then done_reduce()
  virtual void allgather(double* loc, double* all, cudaStream_t s) = 0;
  virtual void done_reduce(cudaStream_t) {}
  // where this rank's kernels publish their totals (allgather's loc) and read all
  virtual double* loc_buf() = 0;
  virtual double* all_buf() = 0;
  // stream the rank's solver must use (nullptr: its own)
  virtual cudaStream_t stream() const { return nullptr; }
  // exchanges are pure stream work (capturable into the inner CUDA graph)
  virtual bool capturable() const { return false; }
};

// P ranks of one process sharing the current device and ONE stream (each rank's
// solver runs on its own host thread). Halo entries are gathered straight from the
// peers' owned rows. Test vehicle for the partition on a one-GPU box: the data flow
// and arithmetic are those of the multi-process NCCL backend.
class LocalGroup {
 public:
  LocalGroup(int P);
  ~LocalGroup();
  int P;
  cudaStream_t stream = nullptr;
  std::vector<PartPlan> plans;
  // sidx[q][p]: device copy of plans[q].send_idx[p]
  std::vector<std::vector<DevBuf>> sidx;
  std::vector<void*> ptrs;  // ext pointers published at a halo exchange
  DevBuf all;               // P x 16 doubles: row r is rank r's loc
  void barrier();
  void fail();              // a rank failed: release everyone (barrier() then throws)
  // rank r's halo entries of an ext vector, gathered from the owned rows the peers
  // published in ptrs[] (precision prec)
  void gather_into(int r, void* ext, int prec, cudaStream_t s);
  void set_plans(uint64_t n, const uint32_t* rp, const uint32_t* ci);

 private:
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  unsigned long long gen_ = 0;
  bool failed_ = false;
};

class LocalExchange : public Exchange {
 public:
  LocalExchange(LocalGroup* g, int r) : g_(g), r_(r) {}
  int size() const override { return g_->P; }
  int rank() const override { return r_; }
  const PartPlan& plan() const override { return g_->plans[r_]; }
  void halo(void* ext, int prec, cudaStream_t s) override;
  void allgather(double* loc, double* all, cudaStream_t s) override;
  void done_reduce(cudaStream_t s) override;
  double* loc_buf() override { return g_->all.get<double>() + (size_t)r_ * 16; }
  double* all_buf() override { return g_->all.get<double>(); }
  cudaStream_t stream() const override { return g_->stream; }

 private:
  LocalGroup* g_;
  int r_;
};

// one rank per process (torch.distributed launch), NCCL point-to-point halos and
// allgather, loaded at run time from the libnccl.so.2 the process already maps
class NcclExchange : public Exchange {
 public:
  NcclExchange(int P, int rank, const void* unique_id, uint64_t n, const uint32_t* rp, const uint32_t* ci);
  ~NcclExchange() override;
  int size() const override { return plan_.P; }
  int rank() const override { return plan_.rank; }
  const PartPlan& plan() const override { return plan_; }
  void halo(void* ext, int prec, cudaStream_t s) override;
  void allgather(double* loc, double* all, cudaStream_t s) override;
  double* loc_buf() override { return loc_.get<double>(); }
  double* all_buf() override { return all_.get<double>(); }
  bool capturable() const override { return true; }
  static void unique_id(void* out128);

 private:
  PartPlan plan_;
  void* comm_ = nullptr;
  std::vector<DevBuf> sidx_;  // per peer: owned indices to send
  std::vector<uint64_t> soff_;
  DevBuf sendbuf_, loc_, all_;
};

// ---- composed solver (reference include/f3r/nesting.hpp:55-77) ------------------------
struct RunOptions {
  double tol = 1e-8;
  int max_outer_restarts = 3;
  unsigned long long max_outer_total = 300;
  bool reset_richardson_on_restart = false;
  // > 0: the reference's fgmres_restarted driver instead of ComposedSolver::run
  // (src/fgmres.cpp:163-222): cycles repeat until tol or this many applications of
  // the outermost level's preconditioner; no restart cap
  unsigned long long restart_budget = 0;
};

struct Report {
  bool converged = false;
  unsigned long long outer_iterations = 0;
  unsigned long long precond_invocations = 0;
  std::vector<unsigned long long> level_iterations;
  std::vector<double> residual_history;
  double final_true_residual = 0.0;
  double wall_seconds = 0.0;
  std::vector<double> omegas_final;
  std::string flag;
  std::string solver_id;
};

class Solver {
 public:
  // ex != nullptr: this solver is one rank of a row-block partition; `a` holds the
  // rank's rows (columns in its ext layout) and every vector is the rank's slice
  // m: the primary preconditioner (reference ComposedSolver(spec, replicas, M),
  // src/nesting.cpp:176-215); null = IdentityPrecond. precond_kind is checked
  // against it (an ILU/IC kind with no factorised M is ERR_UNSUPPORTED).
  Solver(const Spec& spec, std::shared_ptr<DeviceMatrix> a, int precond_kind, Exchange* ex = nullptr,
         std::shared_ptr<const DevicePrecond> m = nullptr);
  ~Solver();
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;

  // b, x: device fp64 vectors of length n (x may be null). stream 0 = own stream.
  Report run(const double* b_dev, double* x_dev, const RunOptions& opts, cudaStream_t stream);
  // back to a freshly built solver's state (Richardson weights 1 or fixed, call
  // counters 1), stream-ordered; equivalent to constructing a new ComposedSolver
  void reset_state(cudaStream_t stream);
  std::vector<double> innermost_omegas();
  std::vector<unsigned long long> level_invocations();
  const std::string& id() const { return id_; }
  uint64_t rows() const { return a_->rows(); }
  cudaStream_t stream() const { return own_stream_; }
  Exchange* exchange() const { return ex_; }
  // per-kernel timing of the NEXT run (CUDA events around every launch, eager mode)
  void set_profile(bool on) { profile_ = on; }
  struct KernelTime {
    std::string name;
    double ms;
    unsigned long long launches;
    double bytes;  // algorithmic bytes over all launches
  };
  std::vector<KernelTime> profile_results() const;
  // halo exchanges and cross-rank reductions (allgathers) the last eager (profiled)
  // run enqueued; graph replays do not count (row-block partition)
  unsigned long long halos() const { return n_halo_; }
  unsigned long long reductions() const { return n_reduce_; }

 private:
  struct Level;
  void build_levels();
  cudaGraphExec_t capture_invocation();  // one L2 invocation as a CUDA graph
  cudaGraphExec_t invocation_graph();     // ... the variant for the current upd_from_
  void enqueue_fgmres(int l, void* src, const double* src_scale, void* dst, const IoSlot* io, cudaStream_t s);
  void enqueue_child_step(int l, int j, cudaStream_t s, bool top);
  void reset_richardson(int l, cudaStream_t s);
  double read_double(const double* dev, cudaStream_t s);
  Report run_fgmres_top(const double* b, const RunOptions& opts, cudaStream_t s, double bnorm, Report rep);
  Report run_richardson_top(const double* b, const RunOptions& opts, cudaStream_t s, double bnorm, Report rep);
  double true_rel(const double* b, double bnorm, cudaStream_t s);
  double mbytes(int pa) const;
  void prof_begin(cudaStream_t s);
  void prof_end(cudaStream_t s, const char* name, double bytes);
  void halo(void* ext, int prec, cudaStream_t s) {
    if (!ex_) return;
    ++n_halo_;
    ex_->halo(ext, prec, s);
  }
  void allgather(cudaStream_t s) {
    ++n_reduce_;
    ex_->allgather(ex_->loc_buf(), ex_->all_buf(), s);
  }
  // row-block partition: the device's Richardson call counter before the next L2
  // invocation -> upd_from_ (first call position in it that can be an update call)
  void plan_update_calls(cudaStream_t s);
  // P == 1: launch(DistH{}) once. P > 1: rank-local launch, allgather, tail launch.
  template <class F>
  void reduce(cudaStream_t s, F&& launch);
  void enqueue_richardson(int l, int j, void* v_ext, const double* sj, void* z_own, cudaStream_t s);
  // one Richardson call of level l with the block-Jacobi M (launch sequence,
  // richardson.cuh k_richm_phase + the trsv.cuh sweeps); v at precision pv
  void enqueue_richardson_m(int l, int pv, const void* v, const double* sj, void* out, cudaStream_t s);
  bool has_m() const { return M_ && !M_->identity(); }
  size_t own(int p) const { return off_ * (p == 0 ? 2 : p == 1 ? 4 : 8); }  // byte offset of the owned rows

  Spec spec_;
  std::string id_;
  std::shared_ptr<DeviceMatrix> a_;
  std::vector<std::unique_ptr<Level>> lv_;
  uint64_t n_ = 0;    // rows of this rank (all rows on one rank)
  uint64_t ld_ = 0;   // vector stride of a basis (ext layout; = n_ on one rank)
  uint64_t off_ = 0;  // owned rows start here in an ext-layout vector
  Exchange* ex_ = nullptr;
  DevBuf dead_, cnt_, partials_, dpartials_, counter_, bar_, info_, io_, norm_, xbuf_, rbuf_, zbuf_, mbuf_;
  std::shared_ptr<const DevicePrecond> M_;
  std::unique_ptr<SweepWork> work_;
  StepInfo* info_host_ = nullptr;
  IoSlot* io_host_ = nullptr;
  double* stage_host_ = nullptr;
  double* reset_host_ = nullptr;  // pinned initial Richardson states, per level
  cudaStream_t own_stream_ = nullptr;
  cudaGraphExec_t inner_exec_ = nullptr;
  bool has_inner_graph_ = false;
  // Row-block partition: a Richardson call carries its update-call phases (halos,
  // allgathers) only from position upd_from_ of the L2 invocation on; rich_pos_
  // counts the calls enqueued in the current invocation. One captured graph per
  // upd_from_ value.
  int rich_pos_ = 0;
  int upd_from_ = 1;
  std::map<int, cudaGraphExec_t> part_exec_;
  unsigned long long n_halo_ = 0, n_reduce_ = 0;
  bool profile_ = false;
  bool profiling_now_ = false;
  bool reverse_off_ = false;  // F3RG_NO_REVERSE=1: no reversed tile walks (A/B tests)
  struct ProfRec;
  std::vector<std::unique_ptr<ProfRec>> prof_;
};

// ---- fp64 competitor solvers (reference src/cg.cpp:22-171), M = identity or block-Jacobi ----
class KrylovSolver {
 public:
  // m: the preconditioner (null = IdentityPrecond)
  explicit KrylovSolver(std::shared_ptr<DeviceMatrix> a, std::shared_ptr<const DevicePrecond> m = nullptr);
  ~KrylovSolver();
  KrylovSolver(const KrylovSolver&) = delete;
  KrylovSolver& operator=(const KrylovSolver&) = delete;
  // which: 0 = cg_solve, 1 = bicgstab_solve. b, x: device fp64 vectors (x may be
  // null); stream 0 = own stream. Throws Error(ERR_SOLVER) where the reference
  // throws SolverError (CG on an indefinite operator).
  Report solve(int which, const double* b, double* x, double tol, unsigned long long max_precond,
               cudaStream_t stream);

 private:
  double true_rel(const double* b, double bnorm, cudaStream_t s);
  std::shared_ptr<DeviceMatrix> a_;
  uint64_t n_ = 0;
  DevBuf x_, r_, p_, q_, s_, t_, rhat_, tmp_, hist_, state_, partials_, counter_, norm_, z_, shat_;
  std::shared_ptr<const DevicePrecond> M_;
  std::unique_ptr<SweepWork> work_;
  bool has_m() const { return M_ && !M_->identity(); }
  double* stage_host_ = nullptr;
  cudaStream_t own_ = nullptr;
};

}  // namespace f3rg
