// mmio.cpp -- Matrix Market coordinate I/O for external matrices,
// restating reference src/matrix_market.cpp:33-127: matrix coordinate real /
// integer / pattern, general / symmetric; symmetric storage expanded, duplicates
// summed after the (row, col) sort, pattern entries 1.0; square only; the
// reference's ParseError messages. Host code: the result feeds f3rg_matrix_create /
// f3rg_matrix_create_scaled like any host CSR.
#include <algorithm>
#include <cctype>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "engine.hpp"

namespace f3rg {

struct HostCsr {
  uint64_t n = 0;
  std::vector<uint32_t> rp, ci;
  std::vector<double> v;
};

namespace {
std::string lower(std::string s) {
  for (auto& c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}
struct Triplet {
  uint32_t r, c;
  double v;
};
[[noreturn]] void fail(const std::string& m) { throw Error(ERR_PARSE, "matrix market: " + m); }
}  // namespace

HostCsr read_matrix_market(std::istream& in) {
  std::string line;
  if (!std::getline(in, line)) fail("empty stream");
  std::string banner, object, format, field, symmetry;
  {
    std::istringstream h(line);
    h >> banner >> object >> format >> field >> symmetry;
  }
  if (banner != "%%MatrixMarket") fail("missing %%MatrixMarket banner");
  object = lower(object), format = lower(format), field = lower(field), symmetry = lower(symmetry);
  if (object != "matrix" || format != "coordinate")
    fail("only 'matrix coordinate' is supported, got '" + object + " " + format + "'");
  if (field != "real" && field != "integer" && field != "pattern") fail("unsupported field '" + field + "'");
  if (symmetry != "general" && symmetry != "symmetric") fail("unsupported symmetry '" + symmetry + "'");
  const bool pattern = field == "pattern", sym = symmetry == "symmetric";

  std::size_t nr = 0, nc = 0, nz = 0;
  for (;;) {  // the size line follows any % comments
    if (!std::getline(in, line)) fail("missing size line");
    if (line.empty() || line[0] == '%') continue;
    std::istringstream s(line);
    if (!(s >> nr >> nc >> nz)) fail("malformed size line");
    break;
  }
  if (nr != nc) fail("non-square matrix (" + std::to_string(nr) + " x " + std::to_string(nc) + ")");

  std::vector<Triplet> t;
  t.reserve(sym ? 2 * nz : nz);
  for (std::size_t seen = 0; seen < nz;) {
    if (!std::getline(in, line)) fail("unexpected end of stream");
    if (line.empty() || line[0] == '%') continue;
    std::istringstream s(line);
    long long i = 0, j = 0;
    double v = 1.0;
    if (!(s >> i >> j)) fail("malformed entry '" + line + "'");
    if (!pattern && !(s >> v)) fail("missing value in '" + line + "'");
    if (i < 1 || j < 1 || (std::size_t)i > nr || (std::size_t)j > nc)
      fail("index out of bounds at entry (" + std::to_string(i) + ", " + std::to_string(j) + ")");
    t.push_back({(uint32_t)(i - 1), (uint32_t)(j - 1), v});
    if (sym && i != j) t.push_back({(uint32_t)(j - 1), (uint32_t)(i - 1), v});
    ++seen;
  }
  // same comparison sort as the reference, so equal (row, col) keys meet in the same
  // order and their sums round identically
  std::sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) { return std::tie(a.r, a.c) < std::tie(b.r, b.c); });
  HostCsr m;
  m.n = nr;
  m.rp.assign(nr + 1, 0);
  m.ci.reserve(t.size());
  m.v.reserve(t.size());
  for (std::size_t k = 0; k < t.size(); ++k) {
    if (k > 0 && t[k].r == t[k - 1].r && t[k].c == t[k - 1].c) {
      m.v.back() += t[k].v;
      continue;
    }
    m.ci.push_back(t[k].c);
    m.v.push_back(t[k].v);
    ++m.rp[t[k].r + 1];
  }
  for (std::size_t i = 0; i < nr; ++i) m.rp[i + 1] += m.rp[i];
  return m;
}

void write_matrix_market(std::ostream& out, uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* v) {
  out << "%%MatrixMarket matrix coordinate real general\n" << n << " " << n << " " << rp[n] << "\n";
  char buf[64];
  for (uint64_t i = 0; i < n; ++i)
    for (uint32_t k = rp[i]; k < rp[i + 1]; ++k) {
      std::snprintf(buf, sizeof buf, "%.17g", v[k]);
      out << (i + 1) << " " << (ci[k] + 1) << " " << buf << "\n";
    }
}

}  // namespace f3rg

// ---- C ABI (include/f3rg.h) ------------------------------------------------------------
#include "../../include/f3rg.h"

struct f3rg_host_csr {
  f3rg::HostCsr m;
};

// error plumbing shared with capi.cpp
namespace f3rg {
void set_last_error(const std::string& m);
}

extern "C" int f3rg_read_matrix_market(const char* path, f3rg_host_csr** out) {
  try {
    if (!path || !out) throw f3rg::Error(f3rg::ERR_DIMENSION, "null argument");
    std::ifstream in(path);
    if (!in) throw f3rg::Error(f3rg::ERR_PARSE, std::string("matrix market: cannot open '") + path + "'");
    auto h = new f3rg_host_csr{f3rg::read_matrix_market(in)};
    *out = h;
    return F3RG_OK;
  } catch (const f3rg::Error& e) {
    f3rg::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    f3rg::set_last_error(e.what());
    return F3RG_EINTERNAL;
  }
}

extern "C" int f3rg_host_csr_view(const f3rg_host_csr* h, f3rg_csr* view) {
  if (!h || !view) return F3RG_EDIMENSION;
  view->n = h->m.n;
  view->row_ptr = h->m.rp.data();
  view->col_idx = h->m.ci.data();
  view->values = h->m.v.data();
  return F3RG_OK;
}

extern "C" uint64_t f3rg_host_csr_nnz(const f3rg_host_csr* h) { return h ? h->m.ci.size() : 0; }

extern "C" void f3rg_host_csr_destroy(f3rg_host_csr* h) { delete h; }

extern "C" int f3rg_write_matrix_market(const char* path, const f3rg_csr* a) {
  try {
    if (!path || !a) throw f3rg::Error(f3rg::ERR_DIMENSION, "null argument");
    f3rg::validate_csr(a->n, a->row_ptr, a->col_idx);
    std::ofstream out(path);
    if (!out) throw f3rg::Error(f3rg::ERR_DIMENSION, std::string("cannot write '") + path + "'");
    f3rg::write_matrix_market(out, a->n, a->row_ptr, a->col_idx, a->values);
    return F3RG_OK;
  } catch (const f3rg::Error& e) {
    f3rg::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    f3rg::set_last_error(e.what());
    return F3RG_EINTERNAL;
  }
}
