// problem_gen.cpp -- standalone writer of the binary CSR cache of a BASELINE
// configuration (§8(f)-2 "binary CSR cache").
//
//     f3rg_gen <kind> <g0> <g1> <g2> <param> <seed> <rhs_mode> <rhs_seed> <out.csr>
//
// Built by buildlib.py as lib/f3rg_gen from this file + problems.cpp (host code
// only: no CUDA, no solver). It exists so a process can obtain the scaled system
// without mapping libf3rg.so -- bench.py's reference arm runs the unmodified
// reference on these bytes -- and so configs 4-5 (10^8-10^9 entries) are
// generated once per host instead of once per process.
//
// File layout (little endian), read by paper_2505_20719_b200/csr_cache.py:
//   char magic[8] = "F3RGCSR1"; uint64 n; uint64 nnz;
//   uint32 row_ptr[n+1]; uint32 col_idx[nnz]; double values[nnz]; double b[n]
// The file is written to <out>.tmp and renamed, so a reader never sees a partial one.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "../../include/f3rg_problems.h"

static bool put(std::FILE* f, const void* p, size_t bytes) { return bytes == 0 || std::fwrite(p, 1, bytes, f) == bytes; }

int main(int argc, char** argv) {
  if (argc != 10) {
    std::fprintf(stderr, "usage: %s kind g0 g1 g2 param seed rhs_mode rhs_seed out.csr\n", argv[0]);
    return 2;
  }
  const int kind = std::atoi(argv[1]);
  const uint64_t grid[3] = {std::strtoull(argv[2], nullptr, 10), std::strtoull(argv[3], nullptr, 10),
                            std::strtoull(argv[4], nullptr, 10)};
  const double param = std::strtod(argv[5], nullptr);
  const uint64_t seed = std::strtoull(argv[6], nullptr, 10);
  const int mode = std::atoi(argv[7]);
  const uint64_t rseed = std::strtoull(argv[8], nullptr, 10);
  const std::string out = argv[9];
  f3rg_problem* p = nullptr;
  int rc = f3rg_problem_generate(&p, kind, grid, param, seed);
  if (rc == 0) rc = f3rg_problem_finalize(p, mode, rseed);
  if (rc != 0) {
    std::fprintf(stderr, "generation failed (code %d)\n", rc);
    if (p) f3rg_problem_destroy(p);
    return 1;
  }
  uint64_t n = 0, nnz = 0;
  const uint32_t *rp = nullptr, *ci = nullptr;
  const double *val = nullptr, *b = nullptr, *d = nullptr;
  f3rg_problem_arrays(p, &n, &nnz, &rp, &ci, &val, &b, &d);
  const std::string tmp = out + ".tmp";
  std::FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) {
    std::perror(tmp.c_str());
    return 1;
  }
  const char magic[8] = {'F', '3', 'R', 'G', 'C', 'S', 'R', '1'};
  bool ok = put(f, magic, 8) && put(f, &n, 8) && put(f, &nnz, 8) && put(f, rp, (n + 1) * 4) && put(f, ci, nnz * 4) &&
            put(f, val, nnz * 8) && put(f, b, n * 8);
  ok = (std::fclose(f) == 0) && ok;
  f3rg_problem_destroy(p);
  if (!ok || std::rename(tmp.c_str(), out.c_str()) != 0) {
    std::perror(out.c_str());
    std::remove(tmp.c_str());
    return 1;
  }
  return 0;
}
