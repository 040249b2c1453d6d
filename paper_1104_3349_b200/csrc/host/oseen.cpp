// Host problem layer, part 1: the Oseen saddle-point system on a MAC grid,
// assembled directly in CSR, plus row equilibration.
//
// Produces bit-for-bit the matrix the reference builds with
// generate_oseen(grid_n, nu, Uniform|Stretched, Recirculating, stretch)
// (proj/src/oseen.cpp:373-441, assembly :108-192, pin :196-202) followed by
// scale_rows (proj/src/row_scaling.cpp:8-31).  The reference collects
// triplets and sorts them (sparse_matrix.cpp:15-50); here each row is built
// in place from its at most 7 stencil entries.  Every floating-point
// expression keeps the reference's operation order (compiled with
// -ffp-contract=off) so no value differs in any bit; duplicate (row, col)
// contributions are summed as from_triplets does (0.0 + a + b).
#include <algorithm>
#include <array>
#include <cmath>

#include "setup.hpp"

namespace mscg::host {

namespace {

struct Grid {
  int n = 0;
  std::vector<double> x, y, xc, yc;
  int nu_per_comp() const { return n * (n - 1); }
  int velocity_count() const { return 2 * nu_per_comp(); }
  int pressure_count() const { return n * n; }
  int iu(int i, int j) const { return (i - 1) + j * (n - 1); }
  int iv(int i, int j) const { return nu_per_comp() + i + (j - 1) * n; }
  int ip(int i, int j) const { return i + j * n; }
};

// oseen.cpp:19-33 (cell widths) and :57-71 (cell boundaries / centres).
Grid make_grid(int n, bool stretched, double factor) {
  std::vector<double> w(n, 1.0 / n);
  if (stretched) {
    const int half = n / 2;
    for (int k = 0; k < half; ++k) {
      w[k] = std::pow(factor, static_cast<double>(k));
      w[n - 1 - k] = w[k];
    }
    if (n % 2 == 1) w[half] = std::pow(factor, static_cast<double>(half));
    double total = 0.0;
    for (double wi : w) total += wi;
    for (double& wi : w) wi /= total;
  }
  Grid g;
  g.n = n;
  g.x.assign(1, 0.0);
  for (int i = 0; i < n; ++i) g.x.push_back(g.x.back() + w[i]);
  g.x.back() = 1.0;
  g.y = g.x;
  for (int i = 0; i < n; ++i) {
    g.xc.push_back(0.5 * (g.x[i] + g.x[i + 1]));
    g.yc.push_back(0.5 * (g.y[i] + g.y[i + 1]));
  }
  return g;
}

// Recirculating wind mapped onto [0,1]^2 (oseen.cpp:386-390).
inline std::array<double, 2> wind(double x, double y) {
  const double xh = 2.0 * x - 1.0;
  const double yh = 2.0 * y - 1.0;
  return {2.0 * yh * (1.0 - xh * xh), -2.0 * xh * (1.0 - yh * yh)};
}

struct Nb {
  int col;       // unknown index or -1 for a boundary value
  double value;  // boundary value
  double dist, face;
};

// Row under construction: <= 5 D entries (+ duplicates) and 2 E entries.
struct RowBuf {
  int c[16];
  double v[16];
  int m = 0;
  void push(int col, double val) { c[m] = col; v[m] = val; ++m; }
};

struct MomentumRow {
  RowBuf buf;
  double rhs = 0.0;
  double diag = 0.0;
};

// add_diffusion / add_convection, oseen.cpp:84-106.
inline void diffusion(MomentumRow& r, double nu, const Nb& nb) {
  const double t = nu * nb.face / nb.dist;
  r.diag += t;
  if (nb.col >= 0) r.buf.push(nb.col, -t);
  else r.rhs += t * nb.value;
}
inline void convection(MomentumRow& r, double speed, double vol, const Nb& up,
                       bool upstream_is_low) {
  if (speed == 0.0) return;
  const bool use_low = speed > 0.0;
  if (use_low != upstream_is_low) return;
  const double c = std::abs(speed) * vol / up.dist;
  r.diag += c;
  if (up.col >= 0) r.buf.push(up.col, -c);
  else r.rhs += c * up.value;
}

// Sort a row's entries by column and sum duplicates the way from_triplets
// does (sum = 0.0; sum += each), pruning exact zeros.
void flush_row(Csr& a, RowBuf& b) {
  // insertion sort: <= 16 entries
  for (int i = 1; i < b.m; ++i) {
    const int c = b.c[i];
    const double v = b.v[i];
    int j = i - 1;
    while (j >= 0 && b.c[j] > c) {
      b.c[j + 1] = b.c[j];
      b.v[j + 1] = b.v[j];
      --j;
    }
    b.c[j + 1] = c;
    b.v[j + 1] = v;
  }
  int k = 0;
  while (k < b.m) {
    const int c = b.c[k];
    double sum = 0.0;
    while (k < b.m && b.c[k] == c) sum += b.v[k++];
    if (sum != 0.0) {
      a.ci.push_back(c);
      a.v.push_back(sum);
    }
  }
}

}  // namespace

void check_oseen_args(int grid_n, double nu, bool stretched, double stretch) {
  if (grid_n < 8) throw std::invalid_argument("generate_oseen: grid_n must be >= 8");
  if (!(nu > 0.0)) throw std::invalid_argument("generate_oseen: viscosity must be positive");
  if (stretched && !(stretch > 1.0))
    throw std::invalid_argument("generate_oseen: stretch factor must exceed 1");
}

void oseen_grid(int grid_n, bool stretched, double stretch, std::vector<double>& x,
                std::vector<double>& y, std::vector<double>& xc, std::vector<double>& yc) {
  Grid g = make_grid(grid_n, stretched, stretch);
  x = std::move(g.x);
  y = std::move(g.y);
  xc = std::move(g.xc);
  yc = std::move(g.yc);
}

OseenSystem generate_oseen(int grid_n, double nu, bool stretched, double stretch) {
  check_oseen_args(grid_n, nu, stretched, stretch);
  const Grid g = make_grid(grid_n, stretched, stretch);
  const int n = g.n;
  const int p = g.velocity_count();
  const int np = g.pressure_count();
  const int pin = np - 1;  // pin_pressure, oseen.cpp:196-202

  OseenSystem out;
  out.p = p;
  Csr& a = out.C;
  a = Csr(p + np, p + np);
  a.ci.reserve(static_cast<size_t>(p) * 7 + static_cast<size_t>(np) * 4);
  a.v.reserve(a.ci.capacity());
  out.rhs.assign(p + np, 0.0);

  int row = 0;
  // u-momentum rows (oseen.cpp:115-149).
  for (int j = 0; j < n; ++j) {
    for (int i = 1; i <= n - 1; ++i, ++row) {
      const double wx = g.xc[i] - g.xc[i - 1];
      const double hy = g.y[j + 1] - g.y[j];
      const double vol = wx * hy;
      const auto [w1, w2] = wind(g.x[i], g.yc[j]);
      Nb west{i - 1 >= 1 ? g.iu(i - 1, j) : -1, 0.0, g.x[i] - g.x[i - 1], hy};
      Nb east{i + 1 <= n - 1 ? g.iu(i + 1, j) : -1, 0.0, g.x[i + 1] - g.x[i], hy};
      Nb south{j - 1 >= 0 ? g.iu(i, j - 1) : -1, 0.0,
               j - 1 >= 0 ? g.yc[j] - g.yc[j - 1] : g.yc[j], wx};
      Nb north{j + 1 <= n - 1 ? g.iu(i, j + 1) : -1, 1.0,
               j + 1 <= n - 1 ? g.yc[j + 1] - g.yc[j] : 1.0 - g.yc[n - 1], wx};
      MomentumRow r;
      diffusion(r, nu, west);
      diffusion(r, nu, east);
      diffusion(r, nu, south);
      diffusion(r, nu, north);
      convection(r, w1, vol, west, true);
      convection(r, w1, vol, east, false);
      convection(r, w2, vol, south, true);
      convection(r, w2, vol, north, false);
      r.buf.push(row, r.diag);
      if (g.ip(i, j) != pin) r.buf.push(p + g.ip(i, j), hy);
      if (g.ip(i - 1, j) != pin) r.buf.push(p + g.ip(i - 1, j), -hy);
      flush_row(a, r.buf);
      a.rp[row + 1] = static_cast<int>(a.ci.size());
      out.rhs[row] = r.rhs;
    }
  }
  // v-momentum rows (oseen.cpp:151-181).
  for (int j = 1; j <= n - 1; ++j) {
    for (int i = 0; i < n; ++i, ++row) {
      const double wx = g.x[i + 1] - g.x[i];
      const double hy = g.yc[j] - g.yc[j - 1];
      const double vol = wx * hy;
      const auto [w1, w2] = wind(g.xc[i], g.y[j]);
      Nb west{i - 1 >= 0 ? g.iv(i - 1, j) : -1, 0.0,
              i - 1 >= 0 ? g.xc[i] - g.xc[i - 1] : g.xc[0], hy};
      Nb east{i + 1 <= n - 1 ? g.iv(i + 1, j) : -1, 0.0,
              i + 1 <= n - 1 ? g.xc[i + 1] - g.xc[i] : 1.0 - g.xc[n - 1], hy};
      Nb south{j - 1 >= 1 ? g.iv(i, j - 1) : -1, 0.0, g.y[j] - g.y[j - 1], wx};
      Nb north{j + 1 <= n - 1 ? g.iv(i, j + 1) : -1, 0.0, g.y[j + 1] - g.y[j], wx};
      MomentumRow r;
      diffusion(r, nu, west);
      diffusion(r, nu, east);
      diffusion(r, nu, south);
      diffusion(r, nu, north);
      convection(r, w1, vol, west, true);
      convection(r, w1, vol, east, false);
      convection(r, w2, vol, south, true);
      convection(r, w2, vol, north, false);
      r.buf.push(row, r.diag);
      if (g.ip(i, j) != pin) r.buf.push(p + g.ip(i, j), wx);
      if (g.ip(i, j - 1) != pin) r.buf.push(p + g.ip(i, j - 1), -wx);
      flush_row(a, r.buf);
      a.rp[row + 1] = static_cast<int>(a.ci.size());
      out.rhs[row] = r.rhs;
    }
  }
  // Continuity rows in flux form (oseen.cpp:183-193), pinned last pressure.
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < n; ++i, ++row) {
      const int q = g.ip(i, j);
      RowBuf b;
      if (q == pin) {
        b.push(p + pin, 1.0);
      } else {
        const double dx = g.x[i + 1] - g.x[i];
        const double dy = g.y[j + 1] - g.y[j];
        if (i + 1 <= n - 1) b.push(g.iu(i + 1, j), dy);
        if (i >= 1) b.push(g.iu(i, j), -dy);
        if (j + 1 <= n - 1) b.push(g.iv(i, j + 1), dx);
        if (j >= 1) b.push(g.iv(i, j), -dx);
      }
      flush_row(a, b);
      a.rp[row + 1] = static_cast<int>(a.ci.size());
    }
  }
  return out;
}

// Row equilibration (row_scaling.cpp:8-31): divide each row and its rhs by
// the signed entry of largest magnitude, first maximum wins ties.
void scale_rows(Csr& a, std::vector<double>& rhs) {
  if (static_cast<int>(rhs.size()) != a.nrows)
    throw std::invalid_argument("scale_rows: rhs length mismatch");
  for (int i = 0; i < a.nrows; ++i) {
    const int b = a.rp[i], e = a.rp[i + 1];
    if (b == e)
      throw std::invalid_argument("scale_rows: row " + std::to_string(i) +
                                  " is identically zero");
    double pivot = a.v[b];
    for (int k = b; k < e; ++k)
      if (std::abs(a.v[k]) > std::abs(pivot)) pivot = a.v[k];
    for (int k = b; k < e; ++k) a.v[k] /= pivot;
    rhs[i] /= pivot;
  }
}

}  // namespace mscg::host
