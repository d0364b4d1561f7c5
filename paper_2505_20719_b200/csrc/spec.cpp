// spec.cpp -- the reference's nesting grammar (include/f3r/solver_spec.hpp:9-15):
//
//   F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > ilu0(blocks=8,alpha=1.0,prec=f16)
//
// Same accepted language, error class (ParseError -> ERR_PARSE) and canonical
// printing as src/solver_spec.cpp:147-212, written independently.
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <sstream>

#include "engine.hpp"

namespace f3rg {

namespace {

std::string trim(const std::string& s) {
  size_t b = 0, e = s.size();
  while (b < e && (s[b] == ' ' || s[b] == '\t')) ++b;
  while (e > b && (s[e - 1] == ' ' || s[e - 1] == '\t')) --e;
  return s.substr(b, e - b);
}

std::vector<std::string> split_trim(const std::string& s, char sep) {
  std::vector<std::string> out;
  size_t start = 0;
  for (;;) {
    const size_t pos = s.find(sep, start);
    out.push_back(trim(s.substr(start, pos == std::string::npos ? std::string::npos : pos - start)));
    if (pos == std::string::npos) return out;
    start = pos + 1;
  }
}

[[noreturn]] void bad(const std::string& token, const std::string& why) {
  throw Error(ERR_PARSE, "solver spec: bad token '" + token + "': " + why);
}

int prec_of(const std::string& tok, const std::string& ctx) {
  if (tok == "f64") return 2;
  if (tok == "f32") return 1;
  if (tok == "f16") return 0;
  bad(ctx, "unknown precision '" + tok + "' (expected f64|f32|f16)");
}

// non-negative int consuming the whole token (std::from_chars semantics)
long long int_of(const std::string& tok, const std::string& ctx) {
  if (tok.empty()) bad(ctx, "expected a non-negative integer");
  size_t i = 0;
  bool neg = false;
  if (tok[0] == '-') neg = true, i = 1;
  if (i >= tok.size()) bad(ctx, "expected a non-negative integer");
  long long v = 0;
  for (; i < tok.size(); ++i) {
    if (tok[i] < '0' || tok[i] > '9') bad(ctx, "expected a non-negative integer");
    v = v * 10 + (tok[i] - '0');
    if (v > 2147483647LL) bad(ctx, "expected a non-negative integer");
  }
  if (neg && v != 0) bad(ctx, "expected a non-negative integer");
  return v;
}

double dbl_of(const std::string& tok, const std::string& ctx) {
  if (tok.empty()) bad(ctx, "expected a number");
  errno = 0;
  char* end = nullptr;
  const double v = std::strtod(tok.c_str(), &end);
  // std::stod skips leading whitespace and must consume the rest
  if (end == tok.c_str() || *end != '\0' || errno == ERANGE) bad(ctx, "expected a number");
  return v;
}

LevelSpec level_of(const std::string& token) {
  const char kind = token[0];
  const size_t colon = token.find(':');
  if (colon == std::string::npos) bad(token, "missing ':<precision>' part");
  const long long m = int_of(token.substr(1, colon - 1), token);
  if (m < 1) bad(token, "iteration count must be >= 1");
  const std::string rest = token.substr(colon + 1);
  LevelSpec L;
  L.m = (int)m;
  if (kind == 'F') {
    const size_t slash = rest.find('/');
    if (slash == std::string::npos) bad(token, "FGMRES level needs '<matrix>/<vector>' precisions");
    L.kind = LK_FGMRES;
    L.pa = prec_of(trim(rest.substr(0, slash)), token);
    L.pv = prec_of(trim(rest.substr(slash + 1)), token);
    return L;
  }
  L.kind = LK_RICHARDSON;
  const auto parts = split_trim(rest, ',');
  L.pa = L.pv = prec_of(parts[0], token);
  for (size_t i = 1; i < parts.size(); ++i) {
    const size_t eq = parts[i].find('=');
    if (eq == std::string::npos) bad(token, "expected key=value after the precision");
    const std::string key = trim(parts[i].substr(0, eq)), val = trim(parts[i].substr(eq + 1));
    if (key == "c") {
      L.cycle = (unsigned long long)int_of(val, token);
    } else if (key == "omega") {
      L.has_omega = true;
      L.omega = dbl_of(val, token);
    } else {
      bad(token, "unknown Richardson parameter '" + key + "'");
    }
  }
  return L;
}

PrecondSpec precond_of(const std::string& token) {
  PrecondSpec p;
  if (token == "identity") {
    p.has_kind = true;
    p.kind = PK_IDENTITY;
    return p;
  }
  std::string head;
  if (token.rfind("ilu0", 0) == 0) {
    p.has_kind = true, p.kind = PK_ILU0;
    head = token.substr(4);
  } else if (token.rfind("ic0", 0) == 0) {
    p.has_kind = true, p.kind = PK_IC0;
    head = token.substr(3);
  } else {
    bad(token, "expected a level (F<m>:... | R<m>:...) or terminal (ilu0(...) | ic0(...) | identity)");
  }
  head = trim(head);
  if (head.empty()) return p;
  if (head.front() != '(' || head.back() != ')') bad(token, "expected '(...)' parameter list");
  const std::string body = trim(head.substr(1, head.size() - 2));
  if (body.empty()) return p;
  for (const auto& part : split_trim(body, ',')) {
    const size_t eq = part.find('=');
    if (eq == std::string::npos) bad(token, "expected key=value in the parameter list");
    const std::string key = trim(part.substr(0, eq)), val = trim(part.substr(eq + 1));
    if (key == "blocks") {
      p.has_blocks = true, p.blocks = (unsigned long long)int_of(val, token);
    } else if (key == "alpha") {
      p.has_alpha = true, p.alpha = dbl_of(val, token);
    } else if (key == "prec") {
      p.has_prec = true, p.prec = prec_of(val, token);
    } else {
      bad(token, "unknown preconditioner parameter '" + key + "'");
    }
  }
  return p;
}

std::string fmt_g(double v) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "%g", v);
  return buf;
}

}  // namespace

const char* precision_name(int p) { return p == 0 ? "f16" : p == 1 ? "f32" : "f64"; }

Spec parse_spec(const std::string& text) {
  Spec spec;
  const auto tokens = split_trim(text, '>');
  for (size_t i = 0; i < tokens.size(); ++i) {
    const std::string& t = tokens[i];
    if (t.empty()) bad(text, "empty nesting level");
    if (t[0] == 'F' || t[0] == 'R') {
      if (spec.has_precond) bad(t, "levels may not follow the terminal preconditioner");
      spec.levels.push_back(level_of(t));
    } else {
      if (i + 1 != tokens.size()) bad(t, "the preconditioner must be the last element");
      spec.has_precond = true;
      spec.precond = precond_of(t);
    }
  }
  if (spec.levels.empty()) bad(text, "at least one solver level is required");
  return spec;
}

std::string Spec::to_string() const {
  std::ostringstream out;
  bool first = true;
  for (const auto& L : levels) {
    if (!first) out << " > ";
    first = false;
    if (L.kind == LK_FGMRES) {
      out << "F" << L.m << ":" << precision_name(L.pa) << "/" << precision_name(L.pv);
    } else {
      out << "R" << L.m << ":" << precision_name(L.pa) << ",c=" << L.cycle;
      if (L.has_omega) out << ",omega=" << fmt_g(L.omega);
    }
  }
  if (has_precond) {
    out << " > ";
    const int kind = precond.has_kind ? precond.kind : PK_ILU0;
    out << (kind == PK_IDENTITY ? "identity" : kind == PK_IC0 ? "ic0" : "ilu0");
    if (kind != PK_IDENTITY) {
      out << "(";
      bool comma = false;
      if (precond.has_blocks) out << "blocks=" << precond.blocks, comma = true;
      if (precond.has_alpha) out << (comma ? "," : "") << "alpha=" << fmt_g(precond.alpha), comma = true;
      if (precond.has_prec) out << (comma ? "," : "") << "prec=" << precision_name(precond.prec);
      out << ")";
    }
  }
  return out.str();
}

// ---- tiles --------------------------------------------------------------------------
// (tile_max_rows / tile_max_nnz are defined next to TileCfg, launch_level.cu)

void build_tiles(uint64_t n, const uint32_t* rp, uint32_t max_rows, uint32_t max_nnz, std::vector<uint32_t>& r0,
                 std::vector<uint32_t>& k0) {
  r0.clear();
  k0.clear();
  uint64_t i = 0;
  while (i < n) {
    r0.push_back((uint32_t)i);
    k0.push_back(rp[i]);
    const uint32_t start = rp[i];
    if (rp[i + 1] - rp[i] > max_nnz) {  // long row: alone
      ++i;
      continue;
    }
    uint64_t j = i;
    while (j < n && j - i < max_rows && rp[j + 1] - start <= max_nnz) ++j;
    i = j;
  }
  r0.push_back((uint32_t)n);
  k0.push_back(rp[n]);
}

}  // namespace f3rg
