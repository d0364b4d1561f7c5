// partition.cpp -- row-block partition plans (see partition.hpp).
#include "partition.hpp"

#include <algorithm>

#include "engine.hpp"

namespace f3rg {

std::vector<uint64_t> partition_rows(uint64_t n, int P) {
  if (P < 1 || (uint64_t)P > std::max<uint64_t>(n, 1))
    throw Error(ERR_DIMENSION, "partition: need 1 <= P <= n");
  // src/ilu.cpp:47-54
  const uint64_t base = n / (uint64_t)P, rem = n % (uint64_t)P;
  std::vector<uint64_t> s((size_t)P + 1, 0);
  for (int b = 0; b < P; ++b) s[b + 1] = s[b] + base + ((uint64_t)b < rem ? 1 : 0);
  return s;
}

PartPlan make_plan(uint64_t n, const uint32_t* rp, const uint32_t* ci, int P, int rank) {
  if (rank < 0 || rank >= P) throw Error(ERR_DIMENSION, "partition: rank out of range");
  const auto st = partition_rows(n, P);
  PartPlan p;
  p.P = P;
  p.rank = rank;
  p.n = n;
  p.r0 = st[rank];
  p.r1 = st[rank + 1];
  auto owner = [&](uint32_t c) { return (int)(std::upper_bound(st.begin(), st.end(), (uint64_t)c) - st.begin()) - 1; };

  // halo: remote columns of the owned rows, ascending and unique
  {
    std::vector<uint32_t> cols;
    for (uint64_t i = p.r0; i < p.r1; ++i)
      for (uint32_t k = rp[i]; k < rp[i + 1]; ++k)
        if (ci[k] < p.r0 || ci[k] >= p.r1) cols.push_back(ci[k]);
    std::sort(cols.begin(), cols.end());
    cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
    p.halo = std::move(cols);
  }
  p.n_lo = (uint64_t)(std::lower_bound(p.halo.begin(), p.halo.end(), (uint32_t)p.r0) - p.halo.begin());
  p.n_hi = p.halo.size() - p.n_lo;
  p.pad = P > 1 ? (8 - p.n_lo % 8) % 8 : 0;

  // receive layout: one contiguous run per owner rank
  p.recv_off.assign((size_t)P, 0);
  p.recv_cnt.assign((size_t)P, 0);
  for (uint64_t h = 0; h < p.halo.size(); ++h) {
    const int q = owner(p.halo[h]);
    const uint64_t ext = h < p.n_lo ? p.pad + h : p.off() + p.n_own() + (h - p.n_lo);
    if (p.recv_cnt[q] == 0) p.recv_off[q] = ext;
    p.recv_cnt[q] += 1;
  }

  // send lists: what every other rank's rows reference among ours, ascending
  p.send_idx.assign((size_t)P, {});
  {
    std::vector<uint8_t> mark(p.n_own(), 0);
    for (int q = 0; q < P; ++q) {
      if (q == rank) continue;
      std::fill(mark.begin(), mark.end(), 0);
      bool any = false;
      for (uint64_t i = st[q]; i < st[q + 1]; ++i)
        for (uint32_t k = rp[i]; k < rp[i + 1]; ++k)
          if (ci[k] >= p.r0 && ci[k] < p.r1) mark[ci[k] - p.r0] = 1, any = true;
      if (!any) continue;
      for (uint64_t i = 0; i < p.n_own(); ++i)
        if (mark[i]) p.send_idx[q].push_back((uint32_t)i);
    }
  }

  // local CSR with ext columns
  p.nnz_begin = rp[p.r0];
  const uint64_t lnnz = (uint64_t)rp[p.r1] - rp[p.r0];
  p.rp.resize(p.n_own() + 1);
  p.ci.resize(lnnz);
  const auto lo_end = p.halo.begin() + (std::ptrdiff_t)p.n_lo;
  for (uint64_t i = p.r0; i < p.r1; ++i) {
    p.rp[i - p.r0] = (uint32_t)(rp[i] - rp[p.r0]);
    for (uint32_t k = rp[i]; k < rp[i + 1]; ++k) {
      const uint32_t c = ci[k];
      uint64_t e;
      if (c < p.r0) e = p.pad + (uint64_t)(std::lower_bound(p.halo.begin(), lo_end, c) - p.halo.begin());
      else if (c < p.r1) e = p.off() + (c - p.r0);
      else e = p.off() + p.n_own() + (uint64_t)(std::lower_bound(lo_end, p.halo.end(), c) - lo_end);
      p.ci[k - rp[p.r0]] = (uint32_t)e;
    }
  }
  p.rp[p.n_own()] = (uint32_t)lnnz;
  return p;
}

}  // namespace f3rg
