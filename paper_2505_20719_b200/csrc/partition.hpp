// partition.hpp -- row-block partition of the solve over P ranks.
//
// Rows are split into contiguous blocks with the reference's own rule
// (src/ilu.cpp:47-54: base = n/P, the remainder spread over the leading blocks).
// Rank r owns rows [r0, r1) of A and of every Krylov vector. Its SpMV input vectors
// use the "ext" layout
//
//     [ pad | lo halo | owned rows r0..r1-1 | hi halo ]
//
// (pad < 8 entries, so the owned part starts 16-byte aligned at every precision)
// where the halos hold the remote columns referenced by the owned rows, ascending
// by global index (hence grouped by owner rank, lower ranks in the lo part). The
// ext layout is the sorted union of owned and referenced columns, so remapping
// the local CSR's columns into it keeps every row's columns strictly increasing
// (stored order unchanged: SpMV results stay bit-identical to the global SpMV) and
// never widens an in-row gap (the D16 column stream stays valid).
#pragma once

#include <cstdint>
#include <vector>

namespace f3rg {

// reference split rule; starts has P+1 entries
std::vector<uint64_t> partition_rows(uint64_t n, int P);

struct PartPlan {
  int P = 1, rank = 0;
  uint64_t n = 0;              // global rows
  uint64_t r0 = 0, r1 = 0;     // owned rows
  uint64_t n_lo = 0, n_hi = 0; // halo sizes
  uint64_t pad = 0;            // leading pad of the ext layout (P > 1 only)
  std::vector<uint32_t> halo;  // n_lo + n_hi global columns, ascending
  // receive side: entries from rank q land at ext offset recv_off[q] (count recv_cnt[q])
  std::vector<uint64_t> recv_off, recv_cnt;
  // send side: send_idx[q] = owned-local indices (0-based) rank q needs from us,
  // in q's halo order
  std::vector<std::vector<uint32_t>> send_idx;
  // local CSR: owned rows, columns remapped into the ext layout
  std::vector<uint32_t> rp, ci;
  uint64_t nnz_begin = 0;      // global position of the first local nonzero (values slice)

  uint64_t n_own() const { return r1 - r0; }
  uint64_t off() const { return pad + n_lo; }
  uint64_t n_ext() const { return off() + n_own() + n_hi; }
  // stride between vectors of one basis (multiple of 8 entries when P > 1)
  uint64_t ld() const { return P > 1 ? (n_ext() + 7) / 8 * 8 : n_ext(); }
};

// Builds rank `rank`'s plan from the global CSR (every rank holds the global
// pattern, so the plans of all ranks are computed without any exchange).
PartPlan make_plan(uint64_t n, const uint32_t* rp, const uint32_t* ci, int P, int rank);

}  // namespace f3rg
