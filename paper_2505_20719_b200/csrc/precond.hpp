// precond.hpp -- the block-Jacobi ILU(0)/IC(0) primary preconditioner on the device
// (reference include/f3r/ilu.hpp:44-84, src/ilu.cpp:38-263).
//
// The factorisation runs once on the host at fp64, exactly as the reference's
// (setup; the reference times it apart from the solve, src/bench.cpp:202-207). The
// factors are then laid out for the device as two SWEEPS, each a schedule of
// "level-sets":
//   * level(i) = 1 + max level of the rows row i reads (0 if none), so rows of one
//     level are independent;
//   * rows are grouped level by level into warp slices of 32 (a level's last slice
//     is padded), and each slice stores its rows' entries interleaved (entry e of
//     lane l at [(slice_base + e) * 32 + l]) in exactly the order the reference
//     accumulates them, so every row's dot is bit-identical to the sequential one.
// ILU: forward = strict lower row (unit diagonal); backward = upper row after its
// diagonal, then / u_ii. IC: forward = lower row without its diagonal, then / l_ii;
// backward = COLUMN i of L below the diagonal in descending row order -- the
// reference's column-oriented scatter (src/ilu.cpp:237-244) subtracts the later
// rows' contributions from work[i] from the last row upwards, then / l_ii.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "launch.hpp"

namespace f3rg {

struct IluConfig {  // reference IluConfig, include/f3r/ilu.hpp:44-49
  uint64_t nblocks = 1;
  double alpha = 1.0;
  bool symmetric = false;
  int prec = 2;  // apply precision tag
};

// host factors (values exactly representable at cfg.prec, held in doubles)
struct HostFactors {
  uint64_t n = 0;
  IluConfig cfg;
  std::vector<uint32_t> block_ranges;  // nblocks + 1
  std::vector<uint32_t> lp, li;        // lower (IC: diagonal last)
  std::vector<double> lv;
  std::vector<uint32_t> up, ui;  // upper, diagonal first (ILU only)
  std::vector<double> uv;
};

// BlockJacobiIlu0::factorize (src/ilu.cpp:38-185); throws Error(ERR_FACTORIZATION)
// with the reference's messages. Blocks are factorised on parallel host threads.
HostFactors factorize_host(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals,
                           const IluConfig& cfg);

// device view of one sweep (kernels in trsv.cuh)
struct SweepDev {
  uint32_t nslices = 0;
  uint32_t nlevels = 0;
  const uint32_t* rows = nullptr;  // nslices*32, 0xffffffff = padding lane
  const uint32_t* cnt = nullptr;   // nslices*32 entries per lane
  const uint32_t* soff = nullptr;  // nslices+1, offsets in 32-entry groups
  const uint32_t* col = nullptr;   // groups*32 dependency rows
  const void* val = nullptr;       // groups*32 factor values (apply precision)
  const void* dg = nullptr;        // nslices*32 divisor per lane, or null (ILU forward)
  const uint32_t* lvl = nullptr;   // nslices: level of each slice
  const uint32_t* lvl_ns = nullptr;  // nlevels: slices per level
  uint64_t n = 0;                    // rows
  uint32_t sleep_ns = 512;           // sleep per level behind the frontier (F3RG_SWEEP_SLEEP)
  uint32_t ahead = 4;                // poll rows from this many levels behind (F3RG_SWEEP_AHEAD)
  uint32_t poll = 0;                 // dependency polling strategy (F3RG_SWEEP_POLL, trsv.cuh)
};

// cross-launch control of one sweep direction (trsv.cuh)
struct SweepCtl {
  unsigned epoch;     // epoch tag of the last completed launch (trsv.cuh next_epoch)
  unsigned done;      // CTAs finished in the running launch
  unsigned frontier;  // levels completed in the running launch (a hint for sleeping)
  unsigned launches;  // launches completed (mod 2^32): level_done[L] = launches * slices(L)
};

// per-user sweep state: the two sweeps' row cells (n x 12 bytes each, enough for
// every compute precision), per-level completion counters and the epochs. One per
// solver (and one inside DevicePrecond for its direct apply()), so solvers sharing
// one M can run concurrently, as the reference allows (include/f3r/nesting.hpp:51-54).
class SweepWork {
 public:
  SweepWork(uint64_t n, uint32_t nlev_fwd, uint32_t nlev_bwd);
  ~SweepWork();
  SweepWork(const SweepWork&) = delete;
  SweepWork& operator=(const SweepWork&) = delete;
  // lay the cells out for compute precision c: cleared (stream-ordered) when c
  // changes, so a stale word of another layout can never read as current
  void prepare(int c, cudaStream_t s);
  void* cells[2] = {nullptr, nullptr};
  unsigned* level_done[2] = {nullptr, nullptr};  // monotone slice counts per level (frontier hint)
  SweepCtl* ctl = nullptr;                       // [2], one per direction

 private:
  uint64_t n_ = 0;
  int last_c_ = -1;
};

class DevicePrecond {
 public:
  // identity (n rows) or a factorised block-Jacobi ILU(0)/IC(0)
  explicit DevicePrecond(uint64_t n);
  DevicePrecond(uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* vals, const IluConfig& cfg);
  ~DevicePrecond();
  DevicePrecond(const DevicePrecond&) = delete;
  DevicePrecond& operator=(const DevicePrecond&) = delete;

  bool identity() const { return identity_; }
  uint64_t rows() const { return n_; }
  const IluConfig& config() const { return cfg_; }
  const std::vector<uint32_t>& block_ranges() const { return block_ranges_; }
  int compute_prec(int pr) const { return identity_ ? pr : (cfg_.prec > pr ? cfg_.prec : pr); }

  // Preconditioner::apply: z = M r (r at pr, z at pz; device pointers), on the
  // internal workspace (one caller at a time)
  void apply(const void* r, int pr, void* z, int pz, cudaStream_t s) const;
  // the two sweeps of z = M r on a caller's workspace; gate_dead/gate_n: the
  // engine's early-stop gate; re: fused Richardson update of the backward sweep
  void enqueue(SweepWork& w, const void* r, int pr, void* z, int pz, cudaStream_t s, const int* gate_dead,
               int gate_n, const RichEpiH* re) const;

  SweepDev sweep(int k) const;  // 0 forward, 1 backward
  uint32_t nlevels(int k) const { return nlev_[k]; }
  uint32_t nslices(int k) const { return nslices_[k]; }
  std::unique_ptr<SweepWork> make_work() const;

 private:
  void build_sweep(int k, const HostFactors& f);
  bool identity_ = true;
  uint64_t n_ = 0;
  IluConfig cfg_;
  std::vector<uint32_t> block_ranges_;
  // per sweep: rows, cnt, soff, col, val, dg, lvl, lvl_ns (device allocations)
  void* buf_[2][8] = {{nullptr}};
  uint32_t nslices_[2] = {0, 0}, nlev_[2] = {0, 0};
  std::unique_ptr<SweepWork> own_;
};

}  // namespace f3rg
