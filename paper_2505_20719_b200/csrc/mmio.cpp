// mmio.cpp -- Matrix Market exchange files: the NIST "matrix
// coordinate" format, written from the format's definition. A file is
//   %%MatrixMarket matrix coordinate <field> <symmetry>     banner (case-insensitive)
//   % ...                                                   comments / blank lines
//   <rows> <cols> <entries>                                 size line
//   <i> <j> [<value>]                                       1-based entries
// with field real | integer | pattern (value 1) and symmetry general | symmetric
// (only one triangle stored; the mirror entry is implied).
// Reader contract (pinned to the reference reader's outputs and messages,
// tests/golden/reference_mm.npz): square matrices only; duplicates are summed in
// the order a (row, col) comparison sort of the entry list -- mirrors appended
// right after their entry -- puts them (std::sort: the same comparator on the same
// sequence visits equal keys in the same order, so the rounded sums agree); errors
// are ParseError "matrix market: ...". The result feeds f3rg_matrix_create /
// f3rg_matrix_create_scaled like any host CSR.
#include <algorithm>
#include <cctype>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <numeric>
#include <sstream>
#include <string>
#include <vector>

#include "engine.hpp"

namespace f3rg {

struct HostCsr {
  uint64_t n = 0;
  std::vector<uint32_t> rp, ci;
  std::vector<double> v;
};

namespace {

[[noreturn]] void parse_error(const std::string& what) { throw Error(ERR_PARSE, "matrix market: " + what); }

// the file as a sequence of '\n'-terminated lines (the terminator dropped)
class Lines {
 public:
  explicit Lines(std::string text) : text_(std::move(text)) {}
  bool next(std::string& out) {
    if (pos_ >= text_.size()) return false;
    const size_t e = text_.find('\n', pos_);
    const size_t stop = e == std::string::npos ? text_.size() : e;
    out.assign(text_, pos_, stop - pos_);
    pos_ = e == std::string::npos ? text_.size() : e + 1;
    return true;
  }
  // the next line that carries data (comments and empty lines skipped)
  bool next_data(std::string& out) {
    while (next(out))
      if (!out.empty() && out[0] != '%') return true;
    return false;
  }

 private:
  std::string text_;
  size_t pos_ = 0;
};

enum class Field { Real, Integer, Pattern };

struct Banner {
  Field field = Field::Real;
  bool symmetric = false;
};

Banner read_banner(const std::string& line) {
  std::istringstream words(line);
  std::string tok[5];
  for (auto& t : tok) words >> t;
  if (tok[0] != "%%MatrixMarket") parse_error("missing %%MatrixMarket banner");
  for (int k = 1; k < 5; ++k)
    std::transform(tok[k].begin(), tok[k].end(), tok[k].begin(), [](unsigned char c) { return (char)std::tolower(c); });
  if (tok[1] != "matrix" || tok[2] != "coordinate")
    parse_error("only 'matrix coordinate' is supported, got '" + tok[1] + " " + tok[2] + "'");
  Banner b;
  static const std::pair<const char*, Field> fields[] = {{"real", Field::Real}, {"integer", Field::Integer},
                                                         {"pattern", Field::Pattern}};
  const auto f = std::find_if(std::begin(fields), std::end(fields), [&](const auto& e) { return tok[3] == e.first; });
  if (f == std::end(fields)) parse_error("unsupported field '" + tok[3] + "'");
  b.field = f->second;
  if (tok[4] == "symmetric") b.symmetric = true;
  else if (tok[4] != "general") parse_error("unsupported symmetry '" + tok[4] + "'");
  return b;
}

struct Coo {
  uint32_t row, col;
  double val;
  bool operator<(const Coo& o) const { return row != o.row ? row < o.row : col < o.col; }
};

// sorted triplets -> CSR, equal (row, col) runs summed left to right
HostCsr compress(uint64_t n, std::vector<Coo>& coo) {
  std::sort(coo.begin(), coo.end());
  HostCsr m;
  m.n = n;
  m.rp.assign(n + 1, 0);
  size_t k = 0;
  while (k < coo.size()) {
    const Coo head = coo[k];
    double sum = head.val;
    for (++k; k < coo.size() && coo[k].row == head.row && coo[k].col == head.col; ++k) sum += coo[k].val;
    m.ci.push_back(head.col);
    m.v.push_back(sum);
    m.rp[head.row + 1] += 1;
  }
  std::partial_sum(m.rp.begin(), m.rp.end(), m.rp.begin());
  return m;
}

}  // namespace

HostCsr read_matrix_market(std::istream& in) {
  Lines lines{std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>())};
  std::string line;
  if (!lines.next(line)) parse_error("empty stream");
  const Banner banner = read_banner(line);

  if (!lines.next_data(line)) parse_error("missing size line");
  std::size_t rows = 0, cols = 0, entries = 0;
  if (!(std::istringstream(line) >> rows >> cols >> entries)) parse_error("malformed size line");
  if (rows != cols) parse_error("non-square matrix (" + std::to_string(rows) + " x " + std::to_string(cols) + ")");

  std::vector<Coo> coo;
  coo.reserve(banner.symmetric ? 2 * entries : entries);
  for (std::size_t e = 0; e < entries; ++e) {
    if (!lines.next_data(line)) parse_error("unexpected end of stream");
    std::istringstream fields(line);
    long long i = 0, j = 0;
    double value = 1.0;  // pattern entries
    if (!(fields >> i >> j)) parse_error("malformed entry '" + line + "'");
    if (banner.field != Field::Pattern && !(fields >> value)) parse_error("missing value in '" + line + "'");
    const bool inside = i >= 1 && j >= 1 && (std::size_t)i <= rows && (std::size_t)j <= cols;
    if (!inside) parse_error("index out of bounds at entry (" + std::to_string(i) + ", " + std::to_string(j) + ")");
    coo.push_back({(uint32_t)(i - 1), (uint32_t)(j - 1), value});
    if (banner.symmetric && i != j) coo.push_back({(uint32_t)(j - 1), (uint32_t)(i - 1), value});
  }
  return compress(rows, coo);
}

void write_matrix_market(std::ostream& out, uint64_t n, const uint32_t* rp, const uint32_t* ci, const double* v) {
  out << "%%MatrixMarket matrix coordinate real general\n" << n << " " << n << " " << rp[n] << "\n";
  char num[40];
  for (uint64_t i = 0; i < n; ++i)
    for (uint32_t k = rp[i]; k < rp[i + 1]; ++k) {
      std::snprintf(num, sizeof num, "%.17g", v[k]);  // round-trips every binary64
      out << (i + 1) << ' ' << (ci[k] + 1) << ' ' << num << '\n';
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
