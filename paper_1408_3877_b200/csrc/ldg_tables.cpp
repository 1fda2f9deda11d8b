// Host-side reference-element math (see ldg_tables.hpp).
#include "ldg_tables.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

namespace ldgb {

namespace {

// The orthonormal modal basis of the reference (basis.hpp:42-85) written as
// scale * polynomial with integer monomial coefficients.  Row i lists the
// coefficient of x1^a x2^b for total degree d = 0..4, a = d..0, b = d - a.
struct BasisRow {
  double mult;
  double root;  // scale = mult * sqrt(root)
  int c[15];
};
constexpr BasisRow kBasis[15] = {
    {1, 2, {1}},
    {1, 1, {2, -6}},
    {2, 3, {1, -1, -2}},
    {1, 6, {1, -8, 0, 10}},
    {1, 3, {-1, -4, 12, 5, 0, -15}},
    {3, 5, {1, -4, -4, 3, 8, 3}},
    {2, 2, {-1, 15, 0, -45, 0, 0, 35}},
    {2, 6, {-1, 13, 2, -33, -24, 0, 21, 42}},
    {2, 10, {-1, 9, 6, -15, -48, -6, 7, 42, 42}},
    {2, 14, {-1, 3, 12, -3, -24, -30, 1, 12, 30, 20}},
    {1, 10, {1, -24, 0, 126, 0, 0, -224, 0, 0, 0, 126}},
    {1, 30, {1, -22, -2, 105, 42, 0, -168, -168, 0, 0, 84, 168}},
    {5, 2, {1, -18, -6, 69, 102, 6, -88, -312, -96, 0, 36, 216, 216}},
    {1, 70, {1, -12, -12, 30, 132, 30, -28, -228, -300, -20, 9, 108, 270, 180}},
    {3, 10, {1, -4, -20, 6, 60, 90, -4, -60, -180, -140, 1, 20, 90, 140, 70}},
};
constexpr int kMonoA[15] = {0, 1, 0, 2, 1, 0, 3, 2, 1, 0, 4, 3, 2, 1, 0};
constexpr int kMonoB[15] = {0, 0, 1, 0, 1, 2, 0, 1, 2, 3, 0, 1, 2, 3, 4};

// Evaluates sum_{a,b} c_ab d^(da)_{x1} d^(db)_{x2} x1^a x2^b by Horner in x1
// for each power of x2, then Horner in x2.
double poly_eval(const int* c, int da, int db, double x1, double x2) {
  double coef[5][5] = {};
  for (int m = 0; m < 15; ++m) {
    int a = kMonoA[m], b = kMonoB[m];
    if (a < da || b < db || c[m] == 0) continue;
    double f = c[m];
    for (int t = 0; t < da; ++t) f *= (a - t);
    for (int t = 0; t < db; ++t) f *= (b - t);
    coef[b - db][a - da] += f;
  }
  double acc = 0.0;
  for (int b = 4; b >= 0; --b) {
    double row = 0.0;
    for (int a = 4; a >= 0; --a) row = row * x1 + coef[b][a];
    acc = acc * x2 + row;
  }
  return acc;
}

double scale_of(int i) { return kBasis[i].mult * std::sqrt(kBasis[i].root); }

}  // namespace

double basis_value(int i, double x1, double x2) {
  if (i < 0 || i >= 15) throw std::out_of_range("basis index must be in 0..14");
  return scale_of(i) * poly_eval(kBasis[i].c, 0, 0, x1, x2);
}

void basis_gradient(int i, double x1, double x2, double* g1, double* g2) {
  if (i < 0 || i >= 15) throw std::out_of_range("basis index must be in 0..14");
  *g1 = scale_of(i) * poly_eval(kBasis[i].c, 1, 0, x1, x2);
  *g2 = scale_of(i) * poly_eval(kBasis[i].c, 0, 1, x1, x2);
}

Rule1D gauss_unit(int npts) {
  // Legendre P_n by the three-term recurrence; Newton from the Tricomi-type
  // initial guess cos(pi (i + 3/4) / (n + 1/2)).  Nodes ascend on (0,1).
  Rule1D r;
  r.s.assign(npts, 0.0);
  r.w.assign(npts, 0.0);
  auto legendre = [npts](double x, double* pn, double* dpn) {
    double p_prev = 1.0, p = x;
    for (int j = 2; j <= npts; ++j) {
      const double next = ((2.0 * j - 1.0) * x * p - (j - 1.0) * p_prev) / j;
      p_prev = p;
      p = next;
    }
    *pn = p;
    *dpn = npts * (x * p - p_prev) / (x * x - 1.0);
  };
  for (int i = 0; i < npts; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (npts + 0.5));
    double pn, dpn;
    for (int it = 0; it < 100; ++it) {
      legendre(x, &pn, &dpn);
      const double step = pn / dpn;
      x -= step;
      if (std::fabs(step) < 1e-16) break;
    }
    legendre(x, &pn, &dpn);
    r.s[npts - 1 - i] = 0.5 * (x + 1.0);
    r.w[npts - 1 - i] = 1.0 / ((1.0 - x * x) * dpn * dpn);
  }
  return r;
}

Rule1D rule_1d(int order) {
  if (order < 0 || order > 17)
    throw std::invalid_argument("1D quadrature order out of supported range 0..17: " + std::to_string(order));
  return gauss_unit(std::max(order, 1) / 2 + 1);
}

Rule2D rule_2d(int order) {
  Rule2D r;
  const int o = std::max(order, 1);
  auto add = [&r](double a, double b, double w) {
    r.x1.push_back(a);
    r.x2.push_back(b);
    r.w.push_back(w);
  };
  if (o == 1) {
    add(1.0 / 3.0, 1.0 / 3.0, 0.5);
  } else if (o == 2) {
    add(1.0 / 6.0, 1.0 / 6.0, 1.0 / 6.0);
    add(2.0 / 3.0, 1.0 / 6.0, 1.0 / 6.0);
    add(1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0);
  } else if (o <= 4) {
    // The reference's 6-point rule with its 15-digit constants (used for
    // orders 3 and 4); projection integrands are not polynomial, so the
    // very same nodes are needed for parity.
    const double a = 0.445948490915965, b = 0.108103018168070;
    const double c = 0.091576213509771, d = 0.816847572980458;
    const double wa = 0.111690794839005, wc = 0.054975871827661;
    add(a, b, wa);
    add(b, a, wa);
    add(a, a, wa);
    add(c, d, wc);
    add(d, c, wc);
    add(c, c, wc);
  } else if (o == 5) {
    const double s15 = std::sqrt(15.0);
    const double a1 = (6.0 - s15) / 21.0, a2 = (6.0 + s15) / 21.0;
    const double w1 = (155.0 - s15) / 2400.0, w2 = (155.0 + s15) / 2400.0;
    add(1.0 / 3.0, 1.0 / 3.0, 9.0 / 80.0);
    add(a1, 1.0 - 2.0 * a1, w1);
    add(1.0 - 2.0 * a1, a1, w1);
    add(a1, a1, w1);
    add(a2, 1.0 - 2.0 * a2, w2);
    add(1.0 - 2.0 * a2, a2, w2);
    add(a2, a2, w2);
  } else {
    // Collapsed (Duffy) product: x1 = u, x2 = v (1 - u), Jacobian (1 - u).
    const int n = (o + 3) / 2;
    const Rule1D g = gauss_unit(n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) add(g.s[i], g.s[j] * (1.0 - g.s[i]), g.w[i] * g.w[j] * (1.0 - g.s[i]));
  }
  return r;
}

void edge_point(int n, double s, double* x1, double* x2) {
  // Local edge n (0-based) is opposite vertex n, oriented counter-clockwise.
  switch (n) {
    case 0: *x1 = 1.0 - s; *x2 = s; return;
    case 1: *x1 = 0.0; *x2 = 1.0 - s; return;
    case 2: *x1 = s; *x2 = 0.0; return;
    default: throw std::out_of_range("local edge index must be 0..2");
  }
}

void edge_to_edge(int nm, int np, double x1, double x2, double* y1, double* y2) {
  // A point of edge nm seen from the neighbour whose edge np is the same
  // physical edge, traversed in the opposite direction.
  double s;  // parameter of the point on edge nm
  switch (nm) {
    case 0: s = x2; break;
    case 1: s = 1.0 - x2; break;
    case 2: s = x1; break;
    default: throw std::out_of_range("local edge index must be 0..2");
  }
  switch (np) {
    case 0: *y1 = s; *y2 = 1.0 - s; return;    // gamma_0(1 - s)
    case 1: *y1 = 0.0; *y2 = s; return;        // gamma_1(1 - s)
    case 2: *y1 = 1.0 - s; *y2 = 0.0; return;  // gamma_2(1 - s)
    default: throw std::out_of_range("local edge index must be 0..2");
  }
}

RefTensors reference_tensors(int n) {
  int p = -1;
  for (int q = 0; q <= kMaxP; ++q)
    if (dofs_of(q) == n) p = q;
  if (p < 0) throw std::invalid_argument("unsupported number of local basis functions: " + std::to_string(n));
  RefTensors t;
  t.n = n;
  t.m.assign(n * n, 0.0);
  t.h.assign(n * n * 2, 0.0);
  t.g.assign(static_cast<size_t>(n) * n * n * 2, 0.0);
  t.sd.assign(n * n * 3, 0.0);
  t.so.assign(n * n * 9, 0.0);
  t.rd.assign(static_cast<size_t>(n) * n * n * 3, 0.0);
  t.ro.assign(static_cast<size_t>(n) * n * n * 9, 0.0);
  std::vector<double> phi(n), d1(n), d2(n), pe(n);

  // element pair tensors, order max(2p,1)
  Rule2D r2 = rule_2d(std::max(2 * p, 1));
  for (size_t q = 0; q < r2.w.size(); ++q) {
    for (int i = 0; i < n; ++i) {
      phi[i] = basis_value(i, r2.x1[q], r2.x2[q]);
      basis_gradient(i, r2.x1[q], r2.x2[q], &d1[i], &d2[i]);
    }
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        t.m[i * n + j] += r2.w[q] * phi[i] * phi[j];
        t.h[(i * n + j) * 2 + 0] += r2.w[q] * d1[i] * phi[j];
        t.h[(i * n + j) * 2 + 1] += r2.w[q] * d2[i] * phi[j];
      }
  }
  // element triple tensor, order max(3p,1)
  Rule2D r3 = rule_2d(std::max(3 * p, 1));
  for (size_t q = 0; q < r3.w.size(); ++q) {
    for (int i = 0; i < n; ++i) {
      phi[i] = basis_value(i, r3.x1[q], r3.x2[q]);
      basis_gradient(i, r3.x1[q], r3.x2[q], &d1[i], &d2[i]);
    }
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int l = 0; l < n; ++l) {
          const size_t at = ((static_cast<size_t>(i) * n + j) * n + l) * 2;
          const double wl = r3.w[q] * phi[l] * phi[j];
          t.g[at] += wl * d1[i];
          t.g[at + 1] += wl * d2[i];
        }
  }
  // edge pair tensors, order 2p+1; edge triple tensors, order min(3p+1,17)
  for (int pass = 0; pass < 2; ++pass) {
    Rule1D r1 = rule_1d(pass == 0 ? 2 * p + 1 : std::min(3 * p + 1, 17));
    for (size_t q = 0; q < r1.w.size(); ++q)
      for (int nm = 0; nm < 3; ++nm) {
        double x1, x2;
        edge_point(nm, r1.s[q], &x1, &x2);
        for (int i = 0; i < n; ++i) phi[i] = basis_value(i, x1, x2);
        if (pass == 0) {
          for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) t.sd[(i * n + j) * 3 + nm] += r1.w[q] * phi[i] * phi[j];
        } else {
          for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
              for (int l = 0; l < n; ++l)
                t.rd[((static_cast<size_t>(i) * n + j) * n + l) * 3 + nm] += r1.w[q] * phi[i] * phi[l] * phi[j];
        }
        for (int np = 0; np < 3; ++np) {
          double y1, y2;
          edge_to_edge(nm, np, x1, x2, &y1, &y2);
          for (int j = 0; j < n; ++j) pe[j] = basis_value(j, y1, y2);
          if (pass == 0) {
            for (int i = 0; i < n; ++i)
              for (int j = 0; j < n; ++j) t.so[((i * n + j) * 3 + nm) * 3 + np] += r1.w[q] * phi[i] * pe[j];
          } else {
            for (int i = 0; i < n; ++i)
              for (int j = 0; j < n; ++j)
                for (int l = 0; l < n; ++l)
                  t.ro[(((static_cast<size_t>(i) * n + j) * n + l) * 3 + nm) * 3 + np] +=
                      r1.w[q] * phi[i] * pe[l] * pe[j];
          }
        }
      }
  }
  return t;
}

namespace {

// Gauss-Jordan inverse with partial pivoting of a small dense matrix.
std::vector<double> invert(std::vector<double> a, int n) {
  std::vector<double> inv(n * n, 0.0);
  for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(a[r * n + c]) > std::fabs(a[piv * n + c])) piv = r;
    if (a[piv * n + c] == 0.0) throw std::runtime_error("singular reference mass matrix");
    if (piv != c)
      for (int k = 0; k < n; ++k) {
        std::swap(a[c * n + k], a[piv * n + k]);
        std::swap(inv[c * n + k], inv[piv * n + k]);
      }
    const double d = a[c * n + c];
    for (int k = 0; k < n; ++k) {
      a[c * n + k] /= d;
      inv[c * n + k] /= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == c || a[r * n + c] == 0.0) continue;
      const double f = a[r * n + c];
      for (int k = 0; k < n; ++k) {
        a[r * n + k] -= f * a[c * n + k];
        inv[r * n + k] -= f * inv[c * n + k];
      }
    }
  }
  return inv;
}

}  // namespace

HostTables build_tables(int p, const RefTensors* caller_rt) {
  if (p < 0 || p > kMaxP) throw std::invalid_argument("polynomial order must be zero to four");
  HostTables ht;
  TableLayout& L = ht.lay;
  const int N = dofs_of(p);
  L.p = p;
  L.N = N;
  const Rule2D proj = rule_2d(std::max(2 * p, 1));            // system.hpp:188
  const Rule1D exact = gauss_unit((3 * p + 2) / 2);            // exact for degree 3p
  const Rule1D bnd = rule_1d(2 * p + 1);                       // quadrature.hpp:204
  L.R = static_cast<int>(proj.w.size());
  L.Qe = static_cast<int>(exact.w.size());
  L.Qb = static_cast<int>(bnd.w.size());
  const RefTensors rt = caller_rt ? *caller_rt : reference_tensors(N);
  if (rt.n != N) throw std::invalid_argument("reference tensor size mismatch");

  long off = 0;
  auto take = [&off](long n) {
    const long at = off;
    off += (n + 1) & ~1L;  // keep 16-byte alignment for vector loads
    return at;
  };
  L.proj_phi = take(L.R * N);
  L.proj_w = take(L.R);
  L.proj_x = take(L.R * 2);
  L.mhat = take(N * N);
  L.minv = take(N * N);
  L.ghat = take(2L * N * N * N);
  L.hhat = take(2L * N * N);
  L.sdiag = take(3L * N * N);
  L.soff = take(9L * N * N);
  L.pe = take(3L * L.Qe * N);
  L.pth = take(9L * L.Qe * N);
  L.we = take(L.Qe);
  L.pb = take(3L * L.Qb * N);
  L.sb = take(L.Qb);
  L.wb = take(L.Qb);
  L.mono = take(15L * N);
  L.NP = (N % 2) ? N + 1 : N;
  L.tH = take(2L * N * L.NP);
  L.tSd = take(3L * N * L.NP);
  L.tSo = take(9L * N * L.NP);
  L.tM = take(1L * N * L.NP);
  L.tMinv = take(1L * N * L.NP);
  L.tmH = take(2L * N * L.NP);
  L.tmSd = take(3L * N * L.NP);
  L.tmSo = take(9L * N * L.NP);
  L.QP = (L.Qe + 1) & ~1;
  L.rkR = take(3L * L.Qe * L.NP);
  L.rkRm = take(3L * L.Qe * L.NP);
  L.rkT = take(3L * N * L.QP);
  L.rkV = take(9L * N * L.QP);
  L.rkW = take(L.QP);
  L.rkEnd = off;
  L.bjG2 = take(9L * L.Qe * N);
  L.total = off;
  ht.data.assign(off, 0.0);
  double* d = ht.data.data();

  for (int r = 0; r < L.R; ++r) {
    for (int j = 0; j < N; ++j) d[L.proj_phi + r * N + j] = basis_value(j, proj.x1[r], proj.x2[r]);
    d[L.proj_w + r] = proj.w[r];
    d[L.proj_x + 2 * r] = proj.x1[r];
    d[L.proj_x + 2 * r + 1] = proj.x2[r];
  }
  std::copy(rt.m.begin(), rt.m.end(), d + L.mhat);
  const std::vector<double> minv = invert(rt.m, N);
  std::copy(minv.begin(), minv.end(), d + L.minv);
  std::copy(rt.g.begin(), rt.g.end(), d + L.ghat);
  std::copy(rt.h.begin(), rt.h.end(), d + L.hhat);
  std::copy(rt.sd.begin(), rt.sd.end(), d + L.sdiag);
  std::copy(rt.so.begin(), rt.so.end(), d + L.soff);
  for (int n = 0; n < 3; ++n)
    for (int q = 0; q < L.Qe; ++q) {
      double x1, x2;
      edge_point(n, exact.s[q], &x1, &x2);
      for (int i = 0; i < N; ++i) d[L.pe + (n * L.Qe + q) * N + i] = basis_value(i, x1, x2);
      for (int np = 0; np < 3; ++np) {
        double y1, y2;
        edge_to_edge(n, np, x1, x2, &y1, &y2);
        for (int j = 0; j < N; ++j) d[L.pth + ((n * 3 + np) * L.Qe + q) * N + j] = basis_value(j, y1, y2);
      }
    }
  for (int q = 0; q < L.Qe; ++q) d[L.we + q] = exact.w[q];
  for (int n = 0; n < 3; ++n)
    for (int q = 0; q < L.Qb; ++q) {
      double x1, x2;
      edge_point(n, bnd.s[q], &x1, &x2);
      for (int i = 0; i < N; ++i) d[L.pb + (n * L.Qb + q) * N + i] = basis_value(i, x1, x2);
    }
  for (int q = 0; q < L.Qb; ++q) {
    d[L.sb + q] = bnd.s[q];
    d[L.wb + q] = bnd.w[q];
  }
  // phi_i = sum_m mono[i][m] x1^a_m x2^b_m (monomial order of kMonoA/kMonoB)
  for (int i = 0; i < N; ++i)
    for (int m = 0; m < 15; ++m) d[L.mono + i * 15 + m] = scale_of(i) * kBasis[i].c[m];
  const int NP = L.NP;
  auto put_t = [&](long at, auto value) {  // at[j*NP + i] = value(i, j)
    for (int j = 0; j < N; ++j)
      for (int i = 0; i < N; ++i) d[at + j * NP + i] = value(i, j);
  };
  for (int m = 0; m < 2; ++m) put_t(L.tH + m * N * NP, [&](int i, int j) { return rt.h[(i * N + j) * 2 + m]; });
  for (int n = 0; n < 3; ++n) put_t(L.tSd + n * N * NP, [&](int i, int j) { return rt.sd[(i * N + j) * 3 + n]; });
  for (int nm = 0; nm < 3; ++nm)
    for (int np = 0; np < 3; ++np)
      put_t(L.tSo + (nm * 3 + np) * N * NP, [&](int i, int j) { return rt.so[((i * N + j) * 3 + nm) * 3 + np]; });
  put_t(L.tM, [&](int i, int j) { return rt.m[i * N + j]; });
  put_t(L.tMinv, [&](int i, int j) { return minv[i * N + j]; });
  // (m_hat^-1 T)[i][j] = sum_a minv[i][a] T[a][j]
  auto minv_times = [&](long at, auto value) {
    put_t(at, [&](int i, int j) {
      double s = 0.0;
      for (int a = 0; a < N; ++a) s += minv[i * N + a] * value(a, j);
      return s;
    });
  };
  for (int m = 0; m < 2; ++m) minv_times(L.tmH + m * N * NP, [&](int a, int j) { return rt.h[(a * N + j) * 2 + m]; });
  for (int n = 0; n < 3; ++n)
    minv_times(L.tmSd + n * N * NP, [&](int a, int j) { return rt.sd[(a * N + j) * 3 + n]; });
  for (int nm = 0; nm < 3; ++nm)
    for (int np = 0; np < 3; ++np)
      minv_times(L.tmSo + (nm * 3 + np) * N * NP,
                 [&](int a, int j) { return rt.so[((a * N + j) * 3 + nm) * 3 + np]; });
  // rank-Qe edge block
  for (int n = 0; n < 3; ++n)
    for (int q = 0; q < L.Qe; ++q)
      for (int i = 0; i < N; ++i) {
        const double v = d[L.pe + (n * L.Qe + q) * N + i];
        d[L.rkR + (n * L.Qe + q) * NP + i] = v;
        d[L.rkT + (n * N + i) * L.QP + q] = v;
        double s = 0.0;
        for (int a = 0; a < N; ++a) s += minv[i * N + a] * d[L.pe + (n * L.Qe + q) * N + a];
        d[L.rkRm + (n * L.Qe + q) * NP + i] = s;
      }
  for (int e = 0; e < 9; ++e)
    for (int q = 0; q < L.Qe; ++q)
      for (int j = 0; j < N; ++j) d[L.rkV + (e * N + j) * L.QP + q] = d[L.pth + (e * L.Qe + q) * N + j];
  for (int q = 0; q < L.Qe; ++q) d[L.rkW + q] = exact.w[q];
  for (int n = 0; n < 3; ++n)
    for (int np = 0; np < 3; ++np)
      for (int q = 0; q < L.Qe; ++q)
        for (int j = 0; j < N; ++j) {
          double s = 0.0;
          for (int i = 0; i < N; ++i)  // (m_hat^-1 s_off(np, n))[i][j] = stored transpose at tmSo[(np, n)][j*NP + i]
            s += d[L.pth + ((n * 3 + np) * L.Qe + q) * N + i] * d[L.tmSo + (np * 3 + n) * N * NP + j * NP + i];
          d[L.bjG2 + ((n * 3 + np) * L.Qe + q) * N + j] = s;
        }
  // do the caller's tensors have the structure the rank form assumes?
  {
    double dev = 0.0, ref = 0.0;
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        for (int n = 0; n < 3; ++n) {
          double sd = 0.0;
          for (int q = 0; q < L.Qe; ++q)
            sd += exact.w[q] * d[L.pe + (n * L.Qe + q) * N + i] * d[L.pe + (n * L.Qe + q) * N + j];
          dev = std::max(dev, std::fabs(sd - rt.sd[(i * N + j) * 3 + n]));
          ref = std::max(ref, std::fabs(sd));
          for (int np = 0; np < 3; ++np) {
            double so = 0.0;
            for (int q = 0; q < L.Qe; ++q)
              so += exact.w[q] * d[L.pe + (n * L.Qe + q) * N + i] * d[L.pth + ((n * 3 + np) * L.Qe + q) * N + j];
            dev = std::max(dev, std::fabs(so - rt.so[((i * N + j) * 3 + n) * 3 + np]));
          }
        }
        // h_hat[i][j][m] = 0 unless deg(phi_i) > deg(phi_j)
        int dj = 0;
        while ((dj + 1) * (dj + 2) / 2 <= j) ++dj;
        if (i < (dj + 1) * (dj + 2) / 2)
          for (int m = 0; m < 2; ++m) {
            double s = 0.0;  // entry of m_hat^-1 h_hat, as staged
            for (int a = 0; a < N; ++a) s += minv[i * N + a] * rt.h[(a * N + j) * 2 + m];
            dev = std::max(dev, std::max(std::fabs(s), std::fabs(rt.h[(i * N + j) * 2 + m])));
          }
      }
    L.rank_ok = dev <= 1e-13 * std::max(ref, 1.0);
  }
  return ht;
}

FTables build_f32_tables(const HostTables& ht) {
  const TableLayout& L = ht.lay;
  const int N = L.N, NP = L.NP;
  FTables f;
  f.NF = (N + 3) / 4 * 4;
  const long tab = static_cast<long>(N) * f.NF;
  f.fmH = 0;
  f.fmSd = f.fmH + 2 * tab;
  f.fmSo = f.fmSd + 3 * tab;
  f.fM = f.fmSo + 9 * tab;
  f.fSd = f.fM + tab;
  f.fSo = f.fSd + 3 * tab;
  const long qn = static_cast<long>(L.Qe) * N;
  f.fpe = f.fSo + 9 * tab;
  f.fpth = f.fpe + 3 * qn;
  f.fwe = f.fpth + 9 * qn;
  f.QF = (L.Qe + 3) / 4 * 4;
  f.fR = (f.fwe + L.Qe + 3) / 4 * 4;
  f.fpeT = f.fR + 3L * L.Qe * f.NF;
  f.fpthT = f.fpeT + 3L * N * f.QF;
  f.fweR = f.fpthT + 9L * N * f.QF;
  f.fRend = f.fweR + f.QF;
  f.total = f.fRend;
  f.data.assign(f.total, 0.0f);
  for (int n = 0; n < 3; ++n)
    for (int q = 0; q < L.Qe; ++q)
      for (int i = 0; i < N; ++i) {
        const float v = static_cast<float>(ht.data[L.pe + (n * L.Qe + q) * N + i]);
        f.data[f.fR + (n * L.Qe + q) * f.NF + i] = v;
        f.data[f.fpeT + (n * N + i) * f.QF + q] = v;
      }
  for (int e = 0; e < 9; ++e)
    for (int q = 0; q < L.Qe; ++q)
      for (int j = 0; j < N; ++j)
        f.data[f.fpthT + (e * N + j) * f.QF + q] = static_cast<float>(ht.data[L.pth + (e * L.Qe + q) * N + j]);
  for (int q = 0; q < L.Qe; ++q) f.data[f.fweR + q] = static_cast<float>(ht.data[L.we + q]);
  for (long t = 0; t < 3 * qn; ++t) f.data[f.fpe + t] = static_cast<float>(ht.data[L.pe + t]);
  for (long t = 0; t < 9 * qn; ++t) f.data[f.fpth + t] = static_cast<float>(ht.data[L.pth + t]);
  for (int q = 0; q < L.Qe; ++q) f.data[f.fwe + q] = static_cast<float>(ht.data[L.we + q]);
  auto copy = [&](long dst, long src, int count) {  // count tables, NP -> NF row padding
    for (int t = 0; t < count; ++t)
      for (int j = 0; j < N; ++j)
        for (int i = 0; i < N; ++i)
          f.data[dst + t * tab + j * f.NF + i] = static_cast<float>(ht.data[src + (static_cast<long>(t) * N + j) * NP + i]);
  };
  copy(f.fmH, L.tmH, 2);
  copy(f.fmSd, L.tmSd, 3);
  copy(f.fmSo, L.tmSo, 9);
  copy(f.fM, L.tM, 1);
  copy(f.fSd, L.tSd, 3);
  copy(f.fSo, L.tSo, 9);
  return f;
}

}  // namespace ldgb
