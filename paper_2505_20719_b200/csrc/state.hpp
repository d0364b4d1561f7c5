// state.hpp -- plain structs shared by host (C++) and device (CUDA) code: the
// device-resident CSR view, tile table, per-level FGMRES state, Richardson state,
// step summary and the I/O indirection slot. No device code here.
#pragma once

#include <cstdint>

namespace f3rg {

struct CsrDev {
  uint64_t n = 0, nnz = 0;
  const uint32_t* rp = nullptr;  // n+1 (+pad)
  const uint32_t* ci = nullptr;  // nnz (+pad)
  const void* val[3] = {nullptr, nullptr, nullptr};
  // "D16" column stream (same columns, fewer bytes): first[i] = column of row i's
  // first entry, dcol[k] = col[k] - col[k-1] - 1 inside a row (dcol[rp[i]] unused;
  // in-row gaps are >= 1, so a gap of 65,536 -- config 4's plane stride -- fits).
  // Present only when every in-row gap fits 16 bits; kernels then stream 2-byte
  // deltas instead of 4-byte indices.
  const uint16_t* dcol = nullptr;   // nnz (+pad)
  const uint32_t* first = nullptr;  // n (+pad)
  // "P16" stream of the fp16 replica: pk[k] = fp16 bits of val16[k] | dcol[k] << 16,
  // one 4-byte word per entry (one shared-memory load per entry instead of two);
  // present with the D16 stream
  const uint32_t* pk = nullptr;     // nnz (+pad)
};

// windowed SELL layout constants (wsell.cuh; built by engine.cpp build_wsell)
constexpr uint32_t kWsSortRows = 2048;      // rows per sort window
constexpr uint32_t kWsPadIdx = 0xffffffffu;  // padding slot / padding lane
// Ring class cl = 0 / 1 / 2: gathers whose ring element has 2 / 4 / 8 bytes. The ring
// is 128 KB: RN elements; a kernel window has TW rows; the band half-width is
// W = (RN - 2 TW) / 2 (the ring holds x[B - W, B + 2 TW + W) while the window at row
// B runs).
constexpr int ws_rn(int cl) { return 65536 >> cl; }
constexpr int ws_tw(int cl) { return 8192 >> cl; }
constexpr int ws_w(int cl) { return (ws_rn(cl) - 2 * ws_tw(cl)) / 2; }  // 24576, 12288, 6144 rows
// encoded column stream (per ring class): byte offset of the ring slot (in band),
// kWsZeroOffset (padding), or kWsFarBit | column (anything else)
constexpr uint32_t kWsZeroOffset = 128u * 1024u + 64u * 1024u + 32u;
constexpr uint32_t kWsFarBit = 0x80000000u;

// Packed windowed layout (wsell_pk.cuh / wsell_pk_layout.hpp): fp16 matrix, 2-byte ring.
// Window geometry on a global grid of kPkTW rows; ring of kPkRing slots (slot = row mod
// kPkRing, the last one reserved: it holds zero), band half-width kPkW = (kPkRing - 2 kPkTW) / 2.
// A slot's 16-bit code: < kPkLimit a ring slot, kPkPad the zero slot, >= kPkEsc the
// high part of a far column (the low 16 bits are the next slot's code).
constexpr int kPkTW = 8192, kPkRing = 49152, kPkW = (kPkRing - 2 * kPkTW) / 2;
constexpr uint32_t kPkLimit = kPkRing - 1, kPkPad = kPkRing - 1, kPkEsc = kPkRing;
// The same slot codes for 4-byte rings (class 1: any replica, fp32 operand -- the L2
// and L1 spmv_dots, fp16 A times fp32 x): 32,768 slots, 4096-row windows, band half-width 12,288; there the
// codes and the values are two streams (2 + 2, 4 or 8 bytes per slot). Class 0 is the packed
// fp16 stream above.
constexpr int pk_ring(int cl) { return cl == 0 ? kPkRing : 32768; }
constexpr int pk_tw(int cl) { return cl == 0 ? kPkTW : 4096; }
constexpr int pk_w(int cl) { return (pk_ring(cl) - 2 * pk_tw(cl)) / 2; }
constexpr uint32_t pk_pad(int cl) { return (uint32_t)pk_ring(cl) - 1u; }  // = the first unusable slot
constexpr uint32_t pk_esc(int cl) { return (uint32_t)pk_ring(cl); }

struct TilesDev {
  const uint32_t* r0 = nullptr;  // ntiles+1 row starts
  const uint32_t* k0 = nullptr;  // ntiles+1 nnz starts (= rp[r0])
  uint32_t ntiles = 0;
  // walk the tiles last-to-first: a pass that follows another pass over the same
  // replica then starts on the part the L2 still holds (set per launch site, so
  // every solve is still bitwise reproducible)
  uint32_t reverse = 0;
  // tile shape the tiles were cut for: 0 regular, 1 short rows, 2 gather-bound
  // (spmv.cuh TileCfg)
  uint32_t shape = 0;
  // L2 eviction priorities (common.cuh l2_policy): 1 = matrix stream evict-first,
  // gathered vector evict-last; 0 = the default policy (F3RG_L2HINT=0)
  uint32_t l2hint = 0;
  // sorted-row tiles (irregular row lengths): tile row q is matrix row perm[q]; the
  // CsrDev handed with these tiles stores the rows in that order. Null = identity
  const uint32_t* perm = nullptr;
  // windowed SELL layout (shape 3, wsell.cuh): slice entry offsets (slices+1), slice
  // lane -> matrix row (slices*32), chunk-major encoded columns (per ring class) and
  // values at this replica's precision, and the split of the sort windows over ws_G CTAs (ws_G+1)
  const uint32_t* ws_soff = nullptr;
  const uint32_t* ws_row = nullptr;
  const uint32_t* ws_enc[3] = {nullptr, nullptr, nullptr};  // encoded columns per ring class
  const void* ws_val = nullptr;
  const uint32_t* ws_cwin = nullptr;
  uint32_t ws_G = 0;
  // packed layout of the fp16 replica for 2-byte rings (null: none): slice slot offsets,
  // slice lane -> row, the packed words (code | fp16 value << 16), the CTA split
  const uint32_t* pk_soff = nullptr;
  const uint32_t* pk_row = nullptr;
  const uint32_t* pk_words = nullptr;
  const uint32_t* pk_cwin = nullptr;
  // the class-1 layout (4-byte rings) of this replica: slice tables, the 16-bit
  // code stream and the value stream at this replica's precision (null: none)
  const uint32_t* pk1_soff = nullptr;
  const uint32_t* pk1_row = nullptr;
  const uint32_t* pk1_cwin = nullptr;
  const uint16_t* pk1_code = nullptr;
  const void* pk1_val = nullptr;
};

// Device-resident state of one FGMRES level. H is column-major: column j holds
// h(0..j+1, j) at H[j*(m+1) + i]. All scalars are values of precision W held in
// doubles (exact).
struct LevelState {
  int m;
  int k;  // Arnoldi steps completed in the current invocation
  int happy, diverged, div_step, tol_hit;
  double beta, bnorm, estimate, tol;
  double* H;
  double* cs;
  double* sn;
  double* g;
  double* y;
  double* scale;
};

// counters layout (unsigned long long): [0..15] level invocations, [16..31] level
// iterations, [32] primary-preconditioner applications
enum { CNT_INV = 0, CNT_IT = 16, CNT_PRECOND = 32, CNT_N = 40 };

// Pointers of the outermost inner invocation, read by the captured graph at run
// time so one graph instance serves every outer Arnoldi step.
struct IoSlot {
  void* src;
  const double* src_scale;
  void* dst;
};

// Host-visible summary of one outer step (copied to pinned memory).
struct StepInfo {
  double estimate;
  int k, happy, diverged, div_step, tol_hit, pad;
};

struct RichState {
  int m;
  unsigned long long cycle;
  double* omegas;             // [m] persistent weights (binary64, as the reference)
  double* wused;              // [m] weight applied at each step of the current call
  int* wupd;                  // [m] 1 if step k computed a fresh w'
  unsigned long long* calls;  // [0] call_count (starts at 1), [1] update_count, [2] degenerate events
  void* R;                    // scratch vectors at the working precision
  void* Za;
  void* Zb;
};

// Scalar state of the fp64 CG / BiCGStab solvers (krylov.cuh), device-resident
enum { KS_RUN = 0, KS_TOL = 1, KS_CAPPED = 2, KS_INDEFINITE = 3, KS_BREAKDOWN = 4 };
struct KState {
  double bnorm, tol;
  double rz, alpha, beta, rho, omega, rr;
  unsigned long long it, precond, max_precond, hist_cap;
  double* hist;  // residual history, hist[0] = 1
  int stop;
};

}  // namespace f3rg
