// Host reference element of the library.  Independent implementation (Newton
// iterations on three-term recurrences, barycentric Lagrange, Gauss-Jordan);
// shares nothing with oracle/.
#include "refelem.h"

#include <cmath>
#include <stdexcept>

namespace sem {

static const double kPi = 3.14159265358979323846;

void jacobi(int n, double a, double b, double x, double* P, double* dP) {
  // three-term recurrence for P_k^{(a,b)}; derivative via (k+a+b+1)/2 P_{k-1}^{(a+1,b+1)}
  auto val = [](int n, double a, double b, double x) {
    if (n == 0) return 1.0;
    double p0 = 1.0, p1 = 0.5 * (a - b + (a + b + 2.0) * x);
    for (int k = 2; k <= n; ++k) {
      double c = 2.0 * k + a + b;
      double a1 = 2.0 * k * (k + a + b) * (c - 2.0);
      double a2 = (c - 1.0) * (a * a - b * b);
      double a3 = (c - 2.0) * (c - 1.0) * c;
      double a4 = 2.0 * (k + a - 1.0) * (k + b - 1.0) * c;
      double p2 = ((a2 + a3 * x) * p1 - a4 * p0) / a1;
      p0 = p1;
      p1 = p2;
    }
    return p1;
  };
  if (P) *P = val(n, a, b, x);
  if (dP) *dP = (n == 0) ? 0.0 : 0.5 * (n + a + b + 1.0) * val(n - 1, a + 1.0, b + 1.0, x);
}

Rule1D lgl_rule(int p) {
  // Newton on x P_p - P_{p-1} (proportional to (1-x^2) P_p'), whose derivative
  // is (p+1) P_p; seeds at Chebyshev-Gauss-Lobatto points.
  Rule1D r;
  r.x.resize(p + 1);
  r.w.resize(p + 1);
  for (int i = 0; i <= p; ++i) {
    double x = -std::cos(kPi * i / p);
    for (int it = 0; it < 100; ++it) {
      double P, Pm1;
      jacobi(p, 0, 0, x, &P, nullptr);
      jacobi(p - 1, 0, 0, x, &Pm1, nullptr);
      double dx = (x * P - Pm1) / ((p + 1) * P);
      x -= dx;
      if (std::fabs(dx) < 1e-16) break;
    }
    r.x[i] = x;
  }
  r.x[0] = -1.0;
  r.x[p] = 1.0;
  for (int i = 0; i <= p / 2; ++i) {  // exact symmetry
    double m = 0.5 * (r.x[p - i] - r.x[i]);
    r.x[i] = -m;
    r.x[p - i] = m;
  }
  if (p % 2 == 0) r.x[p / 2] = 0.0;
  for (int i = 0; i <= p; ++i) {
    double P;
    jacobi(p, 0, 0, r.x[i], &P, nullptr);
    r.w[i] = 2.0 / (p * (p + 1.0) * P * P);
  }
  return r;
}

static Rule1D gauss_jacobi_rule(int n, double a, double b) {
  // Newton with deflation from Chebyshev seeds (roots of P_n^{(a,b)}), weights
  // from the Christoffel formula.
  Rule1D r;
  r.x.resize(n);
  r.w.resize(n);
  for (int k = 0; k < n; ++k) {
    double x = -std::cos((2.0 * k + 1.0) * kPi / (2.0 * n));
    if (k > 0) x = 0.5 * (x + r.x[k - 1]);
    for (int it = 0; it < 200; ++it) {
      double P, dP;
      jacobi(n, a, b, x, &P, &dP);
      double s = 0.0;
      for (int j = 0; j < k; ++j) s += 1.0 / (x - r.x[j]);
      double dx = -P / (dP - s * P);
      x += dx;
      if (std::fabs(dx) < 1e-16) break;
    }
    r.x[k] = x;
  }
  // gamma factor: 2^{a+b+1} G(n+a+1) G(n+b+1) / (G(n+a+b+1) n!)
  double lg = (a + b + 1.0) * std::log(2.0) + std::lgamma(n + a + 1.0) + std::lgamma(n + b + 1.0) -
              std::lgamma(n + a + b + 1.0) - std::lgamma(n + 1.0);
  double C = std::exp(lg);
  for (int k = 0; k < n; ++k) {
    double dP;
    jacobi(n, a, b, r.x[k], nullptr, &dP);
    r.w[k] = C / ((1.0 - r.x[k] * r.x[k]) * dP * dP);
  }
  return r;
}

Rule1D gauss_legendre_rule(int n) { return gauss_jacobi_rule(n, 0.0, 0.0); }
Rule1D gauss_jacobi10_rule(int n) { return gauss_jacobi_rule(n, 1.0, 0.0); }

Lagrange1D::Lagrange1D(const std::vector<double>& nd) : nodes(nd), bw(nd.size()) {
  int n = (int)nd.size();
  for (int j = 0; j < n; ++j) {
    double prod = 1.0;
    for (int k = 0; k < n; ++k)
      if (k != j) prod *= (nd[j] - nd[k]);
    bw[j] = 1.0 / prod;
  }
}

void Lagrange1D::eval(double x, double* h, double* dh) const {
  int n = (int)nodes.size();
  for (int j = 0; j < n; ++j) {
    if (x == nodes[j]) {
      // at a node: h = delta; derivative from the differentiation matrix row
      for (int k = 0; k < n; ++k) h[k] = (k == j) ? 1.0 : 0.0;
      if (dh) {
        double djj = 0.0;
        for (int k = 0; k < n; ++k) {
          if (k == j) continue;
          dh[k] = (bw[k] / bw[j]) / (nodes[j] - nodes[k]);
          djj -= dh[k];
        }
        dh[j] = djj;
      }
      return;
    }
  }
  // l(x) = prod (x - x_k); h_j = l(x) bw_j / (x - x_j)
  double l = 1.0;
  for (int k = 0; k < n; ++k) l *= (x - nodes[k]);
  double s = 0.0;
  for (int k = 0; k < n; ++k) s += 1.0 / (x - nodes[k]);
  for (int j = 0; j < n; ++j) {
    h[j] = l * bw[j] / (x - nodes[j]);
    if (dh) dh[j] = h[j] * (s - 1.0 / (x - nodes[j]));
  }
}

// ---------------------------------------------------------------- triangle
static void dubiner_eval(int p, double r, double s, double* psi, double* pr, double* ps) {
  bool top = std::fabs(1.0 - s) < 1e-14;
  double a = top ? -1.0 : 2.0 * (1.0 + r) / (1.0 - s) - 1.0;
  double b = s;
  int idx = 0;
  for (int i = 0; i <= p; ++i) {
    for (int j = 0; j <= p - i; ++j) {
      double Pi, dPi, Qj, dQj;
      jacobi(i, 0, 0, a, &Pi, &dPi);
      jacobi(j, 2.0 * i + 1.0, 0, b, &Qj, &dQj);
      double om = 1.0 - b;
      double omi = std::pow(om, i);
      double omim1 = (i >= 1) ? std::pow(om, i - 1) : 0.0;
      psi[idx] = Pi * Qj * omi;
      if (pr) pr[idx] = 2.0 * dPi * Qj * omim1;
      if (ps) ps[idx] = dPi * Qj * omim1 * (1.0 + a) + Pi * (dQj * omi - i * Qj * omim1);
      ++idx;
    }
  }
}

static void invert(std::vector<double>& A, int n) {
  // Gauss-Jordan with partial pivoting, in place, row-major
  std::vector<double> I(n * n, 0.0);
  for (int i = 0; i < n; ++i) I[i * n + i] = 1.0;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(A[r * n + c]) > std::fabs(A[piv * n + c])) piv = r;
    if (piv != c)
      for (int k = 0; k < n; ++k) {
        std::swap(A[c * n + k], A[piv * n + k]);
        std::swap(I[c * n + k], I[piv * n + k]);
      }
    double d = A[c * n + c];
    if (d == 0.0) throw std::runtime_error("singular Vandermonde");
    for (int k = 0; k < n; ++k) {
      A[c * n + k] /= d;
      I[c * n + k] /= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      double f = A[r * n + c];
      if (f == 0.0) continue;
      for (int k = 0; k < n; ++k) {
        A[r * n + k] -= f * A[c * n + k];
        I[r * n + k] -= f * I[c * n + k];
      }
    }
  }
  A.swap(I);
}

TriBasis::TriBasis(int p_) : p(p_), nt(n_tri(p_)) {
  Rule1D g = lgl_rule(p);
  std::vector<double> v(p + 1);
  for (int i = 0; i <= p; ++i) v[i] = 0.5 * (1.0 + g.x[i]);
  for (int j = 0; j <= p; ++j)
    for (int i = 0; i <= p - j; ++i) {
      int k = p - i - j;
      double l1 = (1.0 + 2.0 * v[i] - v[j] - v[k]) / 3.0;
      double l2 = (1.0 + 2.0 * v[j] - v[i] - v[k]) / 3.0;
      r.push_back(2.0 * l1 - 1.0);
      s.push_back(2.0 * l2 - 1.0);
      li.push_back(i);
      lj.push_back(j);
    }
  // V[node][mode]; Lagrange L_m(x) = sum_k psi_k(x) Vinv[k][m]
  std::vector<double> V(nt * nt);
  std::vector<double> row(nt);
  for (int n = 0; n < nt; ++n) {
    dubiner_eval(p, r[n], s[n], row.data(), nullptr, nullptr);
    for (int k = 0; k < nt; ++k) V[n * nt + k] = row[k];
  }
  invert(V, nt);
  vinv = V;
}

void TriBasis::eval(double rr, double ss, double* L, double* Lr, double* Ls) const {
  std::vector<double> psi(nt), pr(nt), ps(nt);
  dubiner_eval(p, rr, ss, psi.data(), pr.data(), ps.data());
  for (int m = 0; m < nt; ++m) {
    double a = 0, b = 0, c = 0;
    for (int k = 0; k < nt; ++k) {
      double vi = vinv[k * nt + m];
      a += psi[k] * vi;
      b += pr[k] * vi;
      c += ps[k] * vi;
    }
    if (L) L[m] = a;
    if (Lr) Lr[m] = b;
    if (Ls) Ls[m] = c;
  }
}

// ---------------------------------------------------------------- prism
struct TriCub {
  std::vector<double> r, s, w;
};
static TriCub tri_cubature(int p) {
  Rule1D a = gauss_legendre_rule(p + 1), b = gauss_jacobi10_rule(p + 1);
  TriCub c;
  for (int jb = 0; jb <= p; ++jb)
    for (int ia = 0; ia <= p; ++ia) {
      c.r.push_back(0.5 * (1.0 + a.x[ia]) * (1.0 - b.x[jb]) - 1.0);
      c.s.push_back(b.x[jb]);
      c.w.push_back(0.5 * a.w[ia] * b.w[jb]);
    }
  return c;
}

LevelRef make_level_ref(int p, int qz) {
  // P_p(triangle) x P_q(t): horizontal order p, vertical order q (q = p isotropic)
  const int qo = qz < 0 ? p : qz;
  LevelRef L;
  L.p = p;
  L.q = qo;
  L.n1 = qo + 1;
  L.nt = n_tri(p);
  L.N = L.nt * L.n1;
  L.qt = (p + 1) * (p + 1);
  L.qv = qo + 1;
  L.Q = L.qt * L.qv;
  TriBasis tb(p);
  TriCub tc = tri_cubature(p);
  Rule1D gv = gauss_legendre_rule(qo + 1);
  Lagrange1D h(lgl_rule(qo).x);
  L.B0.resize(L.qt * L.nt);
  L.Br.resize(L.qt * L.nt);
  L.Bs.resize(L.qt * L.nt);
  for (int a = 0; a < L.qt; ++a) tb.eval(tc.r[a], tc.s[a], &L.B0[a * L.nt], &L.Br[a * L.nt], &L.Bs[a * L.nt]);
  L.Bt.resize(L.qv * L.n1);
  L.Dt.resize(L.qv * L.n1);
  for (int q = 0; q < L.qv; ++q) h.eval(gv.x[q], &L.Bt[q * L.n1], &L.Dt[q * L.n1]);
  L.wq.resize(L.Q);
  for (int q = 0; q < L.qv; ++q)
    for (int a = 0; a < L.qt; ++a) L.wq[a + L.qt * q] = tc.w[a] * gv.w[q];
  L.Dfull.assign(3 * (size_t)L.Q * L.N, 0.0);
  for (int q = 0; q < L.qv; ++q)
    for (int a = 0; a < L.qt; ++a)
      for (int l = 0; l < L.n1; ++l)
        for (int m = 0; m < L.nt; ++m) {
          size_t qq = a + (size_t)L.qt * q, n = m + (size_t)L.nt * l;
          L.Dfull[(0 * L.Q + qq) * L.N + n] = L.Br[a * L.nt + m] * L.Bt[q * L.n1 + l];
          L.Dfull[(1 * L.Q + qq) * L.N + n] = L.Bs[a * L.nt + m] * L.Bt[q * L.n1 + l];
          L.Dfull[(2 * L.Q + qq) * L.N + n] = L.B0[a * L.nt + m] * L.Dt[q * L.n1 + l];
        }
  for (int l = 0; l < L.n1; ++l)
    for (int m = 0; m < L.nt; ++m) {
      L.li.push_back(tb.li[m]);
      L.lj.push_back(tb.lj[m]);
      L.ll.push_back(l);
    }
  return L;
}

std::vector<double> geometry_matrix(int pg, int p, int qg, int q) {
  // d/dr, d/ds, d/dt of the order-(pg, qg) nodal basis at the order-(p, q) cubature
  if (qg < 0) qg = pg;
  if (q < 0) q = p;
  TriBasis tb(pg);
  TriCub tc = tri_cubature(p);
  Rule1D gv = gauss_legendre_rule(q + 1);
  Lagrange1D h(lgl_rule(qg).x);
  int ntg = n_tri(pg), n1g = qg + 1, Ng = ntg * n1g, qt = (p + 1) * (p + 1), qv = q + 1, Q = qt * qv;
  std::vector<double> out(3 * (size_t)Ng * Q);
  std::vector<double> L(ntg), Lr(ntg), Ls(ntg), hv(n1g), dh(n1g);
  for (int a = 0; a < qt; ++a) {
    tb.eval(tc.r[a], tc.s[a], L.data(), Lr.data(), Ls.data());
    for (int q = 0; q < qv; ++q) {
      h.eval(gv.x[q], hv.data(), dh.data());
      size_t qq = a + (size_t)qt * q;
      for (int l = 0; l < n1g; ++l)
        for (int m = 0; m < ntg; ++m) {
          size_t n = m + (size_t)ntg * l;
          out[(n * 3 + 0) * Q + qq] = Lr[m] * hv[l];
          out[(n * 3 + 1) * Q + qq] = Ls[m] * hv[l];
          out[(n * 3 + 2) * Q + qq] = L[m] * dh[l];
        }
    }
  }
  return out;
}

void transfer_matrices(int pf, int pc, std::vector<double>& Itri, std::vector<double>& I1, int qf, int qc) {
  if (qf < 0) qf = pf;
  if (qc < 0) qc = pc;
  TriBasis tf(pf), tc(pc);
  int ntf = n_tri(pf), ntc = n_tri(pc);
  Itri.assign((size_t)ntf * ntc, 0.0);
  for (int m = 0; m < ntf; ++m) tc.eval(tf.r[m], tf.s[m], &Itri[(size_t)m * ntc], nullptr, nullptr);
  Rule1D gf = lgl_rule(qf);
  Lagrange1D hc(lgl_rule(qc).x);
  I1.assign((size_t)(qf + 1) * (qc + 1), 0.0);
  for (int l = 0; l <= qf; ++l) hc.eval(gf.x[l], &I1[(size_t)l * (qc + 1)], nullptr);
}

std::vector<double> reference_nodes(int p, int q) {
  if (q < 0) q = p;
  TriBasis tb(p);
  Rule1D g = lgl_rule(q);
  int nt = n_tri(p);
  std::vector<double> rst(3 * (size_t)nt * (q + 1));
  for (int l = 0; l <= q; ++l)
    for (int m = 0; m < nt; ++m) {
      size_t n = m + (size_t)nt * l;
      rst[3 * n + 0] = tb.r[m];
      rst[3 * n + 1] = tb.s[m];
      rst[3 * n + 2] = g.x[l];
    }
  return rst;
}

}  // namespace sem
