// Host-side reference element of the library (independent of oracle/).
// P:209 (LGL), reading O1 (Blyth-Pozrikidis triangle nodes), O2 (prism space
// P_p(tri) x P_p(t)), O6 (collapsed GL x GJ(1,0) x GL cubature).
#pragma once
#include <vector>

namespace sem {

struct Rule1D {
  std::vector<double> x, w;
};

Rule1D lgl_rule(int p);            // p+1 Legendre-Gauss-Lobatto points
Rule1D gauss_legendre_rule(int n);  // n points
Rule1D gauss_jacobi10_rule(int n);  // weight (1-x)

// Jacobi polynomial P_n^{(a,b)}(x) and its derivative.
void jacobi(int n, double a, double b, double x, double* P, double* dP);

// 1D Lagrange cardinal basis on given nodes (barycentric form).
struct Lagrange1D {
  std::vector<double> nodes, bw;
  explicit Lagrange1D(const std::vector<double>& nd);
  void eval(double x, double* h, double* dh) const;  // h[n], dh[n]
};

// Triangle cardinal basis of order p on Blyth-Pozrikidis nodes.
struct TriBasis {
  int p = 0, nt = 0;
  std::vector<double> r, s;      // nodes [nt]
  std::vector<int> li, lj;       // lattice (i toward v1, j toward v2)
  std::vector<double> vinv;      // inverse Vandermonde [nt][nt] (row = modal index)
  explicit TriBasis(int p);
  void eval(double r, double s, double* L, double* Lr, double* Ls) const;
};

inline int n_tri(int p) { return (p + 1) * (p + 2) / 2; }
inline int n_prism(int p, int q = -1) { return n_tri(p) * ((q < 0 ? p : q) + 1); }

// Reference data of one multigrid level of order p.
struct LevelRef {
  int p, q, n1, nt, N, qt, qv, Q;   // q: vertical order (n1 = qv = q + 1); q = p isotropic
  std::vector<double> B0, Br, Bs;   // [qt][nt]
  std::vector<double> Bt, Dt;       // [qv][n1]
  std::vector<double> wq;           // [Q] cubature weights, q = a + qt*qv
  std::vector<double> Dfull;        // [3][Q][N] full reference gradients (setup only)
  std::vector<int> li, lj, ll;      // lattice coords of local nodes [N]
};
// P_p(triangle) x P_q(t) (the paper's (P_xy, P_z)); q < 0: q = p
LevelRef make_level_ref(int p, int q = -1);

// Derivatives of the order-(pg, qg) nodal basis at the cubature of order (p, q):
// layout [n][c][Q] (n = geometry node, c = r,s,t) for the geometry kernel.
std::vector<double> geometry_matrix(int pg, int p, int qg = -1, int q = -1);

// Transfer (prolongation) factors from order (pc, qc) to order (pf, qf):
// Itri[mf][mc] = L^c_mc(node mf of pf), I1[lf][lc] = h^c_lc(t_lf).
void transfer_matrices(int pf, int pc, std::vector<double>& Itri, std::vector<double>& I1, int qf = -1,
                       int qc = -1);

// Reference node coordinates [N][3] in the documented local order.
std::vector<double> reference_nodes(int p, int q = -1);

}  // namespace sem
