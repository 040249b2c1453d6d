// Matrix Market coordinate I/O: the wire format for exchanging matrices
// with the reference (msbench gen, IFISS exports).  Behaviour follows
// proj/src/matrix_market.cpp:20-142:
//  * banner "%%MatrixMarket matrix coordinate real|integer general|
//    symmetric|skew-symmetric" (case-insensitive words after the banner);
//  * '%' comment lines and blank lines skipped anywhere after the banner;
//  * entries 1-based, off-diagonal symmetric entries mirrored (negated for
//    skew), then assembled like SparseMatrix::from_triplets (sort by
//    (row, col), duplicates summed from 0.0, exact zeros dropped);
//  * IoError messages carry " (line N)" exactly as the reference's;
//  * writer: "general" banner, one entry per line, %.17g values.
#include <algorithm>
#include <cctype>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "host/setup.hpp"

namespace mscg::host {

namespace {

std::string io_msg(const std::string& what, int line) {
  return line >= 0 ? what + " (line " + std::to_string(line) + ")" : what;
}

[[noreturn]] void io_fail(const std::string& what, int line = -1) {
  throw IoError(io_msg(what, line));
}

std::string to_lower(std::string s) {
  for (char& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  return s;
}

bool skippable(const std::string& line) {
  return (!line.empty() && line[0] == '%') ||
         line.find_first_not_of(" \t\r\n") == std::string::npos;
}

struct Entry {
  int row, col;
  double value;
};

// Assembly with the reference's from_triplets order (sparse_matrix.cpp:15-50):
// std::sort by (row, col) — the same libstdc++ algorithm, so duplicates are
// summed in the same order — then per (row, col) run sum = 0.0 + ...
Csr csr_from_entries(int nrows, int ncols, std::vector<Entry>& e) {
  std::sort(e.begin(), e.end(), [](const Entry& x, const Entry& y) {
    return x.row != y.row ? x.row < y.row : x.col < y.col;
  });
  Csr a(nrows, ncols);
  a.ci.reserve(e.size());
  a.v.reserve(e.size());
  size_t k = 0;
  for (int r = 0; r < nrows; ++r) {
    while (k < e.size() && e[k].row == r) {
      const int c = e[k].col;
      double sum = 0.0;
      for (; k < e.size() && e[k].row == r && e[k].col == c; ++k) sum += e[k].value;
      if (sum != 0.0) {
        a.ci.push_back(c);
        a.v.push_back(sum);
      }
    }
    a.rp[r + 1] = static_cast<int>(a.ci.size());
  }
  return a;
}

}  // namespace

Csr load_matrix_market(const std::string& path) {
  std::ifstream f(path);
  if (!f) io_fail("cannot open " + path);
  std::string line;
  int ln = 0;
  if (!std::getline(f, line)) io_fail("empty file " + path, 1);
  ln = 1;
  std::string w[5];
  {
    std::istringstream hs(line);
    for (auto& s : w) hs >> s;
  }
  if (w[0] != "%%MatrixMarket" || to_lower(w[1]) != "matrix")
    io_fail("not a MatrixMarket matrix file: " + path, ln);
  if (to_lower(w[2]) != "coordinate")
    io_fail("unsupported format '" + w[2] + "' (coordinate only)", ln);
  const std::string field = to_lower(w[3]);
  if (field != "real" && field != "integer")
    io_fail("unsupported field '" + w[3] + "' (real only)", ln);
  const std::string sym = to_lower(w[4]);
  const bool mirror = sym == "symmetric" || sym == "skew-symmetric";
  const double mirror_sign = sym == "skew-symmetric" ? -1.0 : 1.0;
  if (!mirror && sym != "general") io_fail("unsupported symmetry '" + w[4] + "'", ln);

  int nrows = -1, ncols = -1;
  long long declared = -1;
  while (std::getline(f, line)) {
    ++ln;
    if (skippable(line)) continue;
    std::istringstream ds(line);
    if (!(ds >> nrows >> ncols >> declared) || nrows < 0 || ncols < 0 || declared < 0)
      io_fail("malformed dimension line", ln);
    break;
  }
  if (nrows < 0) io_fail("missing dimension line", ln);

  std::vector<Entry> e;
  e.reserve(static_cast<size_t>(declared) * (mirror ? 2 : 1));
  long long found = 0;
  while (std::getline(f, line)) {
    ++ln;
    if (skippable(line)) continue;
    std::istringstream es(line);
    int i = 0, j = 0;
    double v = 0.0;
    if (!(es >> i >> j >> v)) io_fail("malformed entry", ln);
    if (i < 1 || i > nrows || j < 1 || j > ncols) io_fail("entry indices out of range", ln);
    e.push_back({i - 1, j - 1, v});
    if (mirror && i != j) e.push_back({j - 1, i - 1, mirror_sign * v});
    ++found;
  }
  if (found != declared)
    io_fail("expected " + std::to_string(declared) + " entries, found " + std::to_string(found),
            ln);
  return csr_from_entries(nrows, ncols, e);
}

void write_matrix_market(const std::string& path, const Csr& a) {
  std::ofstream f(path);
  if (!f) io_fail("cannot write " + path);
  f << "%%MatrixMarket matrix coordinate real general\n"
    << a.nrows << ' ' << a.ncols << ' ' << a.nnz() << '\n';
  f.precision(17);
  for (int r = 0; r < a.nrows; ++r)
    for (int k = a.rp[r]; k < a.rp[r + 1]; ++k) f << r + 1 << ' ' << a.ci[k] + 1 << ' ' << a.v[k] << '\n';
  if (!f) io_fail("write failed for " + path);
}

std::vector<double> load_vector_market(const std::string& path) {
  const Csr m = load_matrix_market(path);
  if (m.ncols != 1) io_fail("expected an n x 1 vector in " + path);
  std::vector<double> out(m.nrows, 0.0);
  for (int r = 0; r < m.nrows; ++r)
    if (m.rp[r + 1] > m.rp[r]) out[r] = m.v[m.rp[r]];
  return out;
}

void write_vector_market(const std::string& path, const double* v, int n) {
  Csr m(n, 1);
  for (int r = 0; r < n; ++r) {
    if (v[r] != 0.0) {
      m.ci.push_back(0);
      m.v.push_back(v[r]);
    }
    m.rp[r + 1] = static_cast<int>(m.ci.size());
  }
  write_matrix_market(path, m);
}

}  // namespace mscg::host
