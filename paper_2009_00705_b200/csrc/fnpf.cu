// FNPF time stage on the device (eq 2.1a-b and 2.2).
//
// The state is the free-surface elevation eta and surface potential phi~ at the
// free-surface nodes.  One stage (fnpf_rhs):
//   1. geometry (reading O37): every node of the finest nodal map keeps its sigma on
//      the vertical line of its free-surface node, z = z_b + sigma (eta - z_b)
//      (the sigma map of eq 3.3); only z moves, x and y are fixed, so the update is
//      one kernel over the nodal map and G is recomputed on the device from it
//      (k_geometry) -- the finest level (strategy 1 = the paper's strategy I:
//      smoothers and coarse operators from t = 0) or every level's operator
//      (strategy 2: the smoothers and the coarse inverse stay those of t = 0);
//   2. the Laplace solve eq 2.2 with phi = phi~ on the free surface, warm-started
//      from the previous stage's solution (laplace_solve_guess);
//   3. w~ = dphi/dz at the free surface (reading O38) and the horizontal gradients of
//      eta and phi~ along the surface (reading O39): per top element and top-face
//      node, the isoparametric gradient of the element interpolant, averaged over
//      the elements holding the node;
//   4. the rates of eq 2.1a-b (linear = 1: the small-amplitude version on the t = 0
//      geometry, d eta/dt = w~, d phi~/dt = -g eta).
// fnpf_erk4_step: classical four-stage RK4 (reading O40), one solve per stage.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <vector>

#include "internal.h"
#include "setup_util.h"

namespace sem {

int do_solve(sem_ctx* c, const double* rhs, const double* phiD, double tol, double* phi, sem_report* rep, int guess,
             int cond);

struct Fnpf {
  int64_t ns = 0;                 // free-surface nodes
  int ntop = 0, Nt = 0, Nf = 0, strategy = 1;
  double* X = nullptr;            // [E][Nf][3] current finest nodal map
  double* X0 = nullptr;           // [E][Nf][3] nodal map of t = 0
  int32_t* gline = nullptr;       // [n0] surface index of every finest-level node
  double* gsig = nullptr;         // [n0] sigma of every finest-level node
  double* zb = nullptr;           // [ns] bottom z of every vertical line
  int32_t* snode = nullptr;       // [ns] library node id of every surface node
  int32_t* top = nullptr;         // [ntop] top elements (top face on the free surface)
  double* icnt = nullptr;         // [ns] 1 / (top elements holding the node)
  double *Dtop = nullptr, *Dr2 = nullptr, *Ds2 = nullptr;   // [3][Nt][Nf], [Nt][Nt] x2
  std::vector<double*> gm, wq;    // geometry matrices / cubature weights per level
  double *phiD = nullptr, *phi = nullptr, *acc = nullptr;   // [n0], [n0], [ns][5]
  double *ea = nullptr, *pa = nullptr, *ke = nullptr, *kp = nullptr;   // RK4 stage buffers [ns], [4 ns]
  std::vector<int32_t> snode_host;
  int warm = 0;                   // 1: phi holds the previous stage's solution
  int geom_t0 = 1;                // 1: the device geometry is that of t = 0
};

static int fgrid(int64_t n, int t) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + t - 1) / t, 148 * 64)); }

// z of every finest nodal-map point from eta (reading O37)
__global__ void k_fnpf_z(int64_t EN, const int32_t* __restrict__ conn, const int32_t* __restrict__ gline,
                         const double* __restrict__ gsig, const double* __restrict__ zb,
                         const double* __restrict__ eta, double* __restrict__ X) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < EN; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t g = conn[i];
    if (g < 0) g = ~g;
    const int32_t s = gline[g];
    X[3 * i + 2] = zb[s] + gsig[g] * (eta[s] - zb[s]);
  }
}

// phiD[snode[s]] = phis[s]
__global__ void k_fnpf_scatter(int64_t ns, const int32_t* __restrict__ snode, const double* __restrict__ phis,
                               double* __restrict__ phiD) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < ns; s += (int64_t)gridDim.x * blockDim.x)
    phiD[snode[s]] = phis[s];
}

// per (top element, top-face node m): w~ = (J^-T grad_ref phi)_z and the surface gradients of eta, phi~
// (readings O38, O39); acc[s][0..4] += w, eta_x, eta_y, phi~_x, phi~_y
__global__ void k_fnpf_recover(int ntop, int Nt, int Nf, int p, const int32_t* __restrict__ top,
                               const int32_t* __restrict__ conn, const int32_t* __restrict__ gline,
                               const double* __restrict__ X, const double* __restrict__ Dtop,
                               const double* __restrict__ Dr2, const double* __restrict__ Ds2,
                               const double* __restrict__ phi, const double* __restrict__ eta,
                               const double* __restrict__ phis, double* __restrict__ acc) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)ntop * Nt) return;
  const int j = (int)(idx / Nt), m = (int)(idx % Nt);
  const int64_t e = top[j];
  const double* Xe = X + e * Nf * 3;
  const int32_t* ce = conn + e * Nf;
  double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, gr[3] = {0, 0, 0};
  for (int n = 0; n < Nf; ++n) {
    int32_t g = ce[n];
    if (g < 0) g = ~g;
    const double f = phi[g];
    const double d[3] = {Dtop[(0 * Nt + m) * Nf + n], Dtop[(1 * Nt + m) * Nf + n], Dtop[(2 * Nt + m) * Nf + n]};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      gr[c] = fma(f, d[c], gr[c]);
#pragma unroll
      for (int i = 0; i < 3; ++i) J[i][c] = fma(Xe[3 * n + i], d[c], J[i][c]);
    }
  }
  // grad = J^-T gr: solve J^T x = gr by Cramer's rule
  const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                     J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
  // inverse of J (row i of J^-1 = d xi_i / d x); grad_x = sum_c (J^-1)[c][x] gr[c]
  const double i02 = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
  const double i12 = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
  const double i22 = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
  const double w = i02 * gr[0] + i12 * gr[1] + i22 * gr[2];
  // surface gradients on the top face (x, y affine): J2 = [[x_r, x_s], [y_r, y_s]]
  const int off = Nt * p;
  double xr = 0, xs = 0, yr = 0, ys = 0, er = 0, es = 0, pr = 0, ps = 0;
  for (int k = 0; k < Nt; ++k) {
    const double dr = Dr2[m * Nt + k], ds = Ds2[m * Nt + k];
    const double x = Xe[3 * (off + k)], y = Xe[3 * (off + k) + 1];
    int32_t g = ce[off + k];
    if (g < 0) g = ~g;
    const int32_t s = gline[g];
    const double fe = eta[s], fp = phis[s];
    xr = fma(dr, x, xr);
    xs = fma(ds, x, xs);
    yr = fma(dr, y, yr);
    ys = fma(ds, y, ys);
    er = fma(dr, fe, er);
    es = fma(ds, fe, es);
    pr = fma(dr, fp, pr);
    ps = fma(ds, fp, ps);
  }
  // J2^T [fx, fy] = [fr, fs]:  fx = ( y_s fr - y_r fs) / D,  fy = (-x_s fr + x_r fs) / D
  const double D2 = xr * ys - xs * yr;
  int32_t gm_ = ce[off + m];
  if (gm_ < 0) gm_ = ~gm_;
  double* a = acc + 5 * (int64_t)gline[gm_];
  atomicAdd(a + 0, w);
  atomicAdd(a + 1, (ys * er - yr * es) / D2);
  atomicAdd(a + 2, (-xs * er + xr * es) / D2);
  atomicAdd(a + 3, (ys * pr - yr * ps) / D2);
  atomicAdd(a + 4, (-xs * pr + xr * ps) / D2);
}

// eq 2.1a-b at every surface node
__global__ void k_fnpf_rates(int64_t ns, const double* __restrict__ acc, const double* __restrict__ icnt,
                             const double* __restrict__ eta, double* __restrict__ deta, double* __restrict__ dphis,
                             double* __restrict__ wout, int linear, double g) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < ns; s += (int64_t)gridDim.x * blockDim.x) {
    const double ic = icnt[s];
    const double w = acc[5 * s] * ic;
    if (wout) wout[s] = w;
    if (linear) {
      deta[s] = w;
      dphis[s] = -g * eta[s];
      continue;
    }
    const double ex = acc[5 * s + 1] * ic, ey = acc[5 * s + 2] * ic, px = acc[5 * s + 3] * ic, py = acc[5 * s + 4] * ic;
    const double ge2 = ex * ex + ey * ey;
    deta[s] = -(ex * px + ey * py) + w * (1.0 + ge2);
    dphis[s] = -g * eta[s] - 0.5 * ((px * px + py * py) - w * w * (1.0 + ge2));
  }
}

// y = x + a k
__global__ void k_fnpf_axpy(int64_t n, const double* __restrict__ x, double a, const double* __restrict__ k,
                            double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(a, k[i], x[i]);
}

// x += dt/6 (k1 + 2 k2 + 2 k3 + k4)
__global__ void k_fnpf_rk4(int64_t n, double* __restrict__ x, const double* __restrict__ k, double dt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] += dt / 6.0 * (k[i] + 2.0 * k[n + i] + 2.0 * k[2 * n + i] + k[3 * n + i]);
}

// ---------------------------------------------------------------- setup
void fnpf_init(sem_ctx* c, const double* node_xyz, int strategy) {
  if (c->dist) throw SemError(SEM_EUNSUPPORTED, "FNPF stages: single-domain ctx only");
  if (c->PZ != c->P) throw SemError(SEM_EUNSUPPORTED, "FNPF stages: isotropic orders only");
  if (strategy < 1 || strategy > 4) throw SemError(SEM_EINVAL, "strategy must be 1..4");
  if (strategy >= 3 && c->L.size() > 1 && !c->L[0].fdm)
    throw SemError(SEM_EUNSUPPORTED, "strategies II / III re-form the smoothers every stage: local_solve = 1 (FDM)");
  if (strategy == 4 && c->L.size() > 1 && !c->C.iterative)
    throw SemError(SEM_EUNSUPPORTED, "strategy III re-forms the coarse operator every stage: coarse_solver = 1");
  if (!c->fnpf) c->fnpf = new Fnpf();
  Fnpf& F = *c->fnpf;
  F.strategy = strategy;
  DeviceLevel& L0 = c->L[0];
  const int p = c->P, Nf = n_prism(p), Nt = n_tri(p), E = c->E;
  F.Nf = Nf;
  F.Nt = Nt;
  if (L0.p != p) throw SemError(SEM_EINVAL, "finest level order mismatch");
  // vertical lines: every finest node below a free-surface (Dirichlet) node with the same (x, y)
  const int64_t n0 = L0.n;
  const std::vector<double>& xyz = L0.xyz;
  std::map<std::pair<long long, long long>, int32_t> at;
  double ext = 1.0;
  for (int64_t i = 0; i < n0; ++i) ext = std::max({ext, std::fabs(xyz[3 * i]), std::fabs(xyz[3 * i + 1])});
  const double q = 1e-9 * ext;
  auto key = [&](int64_t i) {
    return std::make_pair((long long)std::llround(xyz[3 * i] / q), (long long)std::llround(xyz[3 * i + 1] / q));
  };
  F.snode_host.clear();
  for (int64_t i = 0; i < n0; ++i)
    if (L0.dir_host[i]) {
      if (!at.emplace(key(i), (int32_t)F.snode_host.size()).second)
        throw SemError(SEM_EUNSUPPORTED, "FNPF: two free-surface nodes on one vertical line");
      F.snode_host.push_back((int32_t)i);
    }
  F.ns = (int64_t)F.snode_host.size();
  std::vector<int32_t> gline(n0);
  std::vector<double> zb(F.ns, INFINITY), gsig(n0);
  for (int64_t i = 0; i < n0; ++i) {
    auto it = at.find(key(i));
    if (it == at.end())
      throw SemError(SEM_EUNSUPPORTED, "FNPF: a node is not below a free-surface node (needs a sigma-layered mesh)");
    gline[i] = it->second;
    zb[it->second] = std::min(zb[it->second], xyz[3 * i + 2]);
  }
  for (int64_t i = 0; i < n0; ++i) {
    const double zs = xyz[3 * (int64_t)F.snode_host[gline[i]] + 2], z0 = zb[gline[i]];
    gsig[i] = (xyz[3 * i + 2] - z0) / (zs - z0);
  }
  // top elements and averaging counts
  std::vector<int32_t> top;
  std::vector<double> cnt(F.ns, 0.0);
  const std::vector<int32_t>& conn = L0.conn_host;
  for (int e = 0; e < E; ++e) {
    const int32_t gtop = conn[(size_t)e * Nf + Nt * p];   // top-face node m = 0
    if (!L0.dir_host[gtop]) continue;
    bool all = true;
    for (int m = 0; m < Nt; ++m) all &= L0.dir_host[conn[(size_t)e * Nf + Nt * p + m]] != 0;
    if (!all) continue;
    top.push_back(e);
    for (int m = 0; m < Nt; ++m) cnt[gline[conn[(size_t)e * Nf + Nt * p + m]]] += 1.0;
  }
  for (double& v : cnt) {
    if (v == 0.0) throw SemError(SEM_EUNSUPPORTED, "FNPF: a free-surface node lies on no element's top face");
    v = 1.0 / v;
  }
  F.ntop = (int)top.size();
  // reference derivatives at the top-face nodes (prism basis) and at the triangle nodes (2D)
  TriBasis tb(p);
  Lagrange1D lt(lgl_rule(p).x);
  std::vector<double> h(p + 1), dh(p + 1);
  lt.eval(1.0, h.data(), dh.data());
  std::vector<double> Dtop((size_t)3 * Nt * Nf), Dr2((size_t)Nt * Nt), Ds2((size_t)Nt * Nt), Lv(Nt), Lr(Nt), Ls(Nt);
  for (int m = 0; m < Nt; ++m) {
    tb.eval(tb.r[m], tb.s[m], Lv.data(), Lr.data(), Ls.data());
    for (int k = 0; k < Nt; ++k) {
      Dr2[(size_t)m * Nt + k] = Lr[k];
      Ds2[(size_t)m * Nt + k] = Ls[k];
    }
    for (int l = 0; l <= p; ++l)
      for (int k = 0; k < Nt; ++k) {
        const int n = k + Nt * l;
        Dtop[((size_t)0 * Nt + m) * Nf + n] = Lr[k] * h[l];
        Dtop[((size_t)1 * Nt + m) * Nf + n] = Ls[k] * h[l];
        Dtop[((size_t)2 * Nt + m) * Nf + n] = Lv[k] * dh[l];
      }
  }
  std::vector<double> X(node_xyz, node_xyz + (size_t)E * Nf * 3);
  F.X = upload(c, X);
  F.X0 = upload(c, X);
  F.gline = upload(c, gline);
  F.gsig = upload(c, gsig);
  F.zb = upload(c, zb);
  F.snode = upload(c, F.snode_host);
  F.top = upload(c, top);
  F.icnt = upload(c, cnt);
  F.Dtop = upload(c, Dtop);
  F.Dr2 = upload(c, Dr2);
  F.Ds2 = upload(c, Ds2);
  F.gm.clear();
  F.wq.clear();
  for (size_t li = 0; li < c->L.size(); ++li) {
    F.gm.push_back(upload(c, geometry_matrix(p, c->L[li].p)));
    F.wq.push_back(upload(c, c->L[li].ref.wq));
  }
  F.phiD = dalloc<double>(c, n0);
  F.phi = dalloc<double>(c, n0);
  F.acc = dalloc<double>(c, 5 * F.ns);
  F.ea = dalloc<double>(c, F.ns);
  F.pa = dalloc<double>(c, F.ns);
  F.ke = dalloc<double>(c, 4 * F.ns);
  F.kp = dalloc<double>(c, 4 * F.ns);
  CUDA_CHECK(cudaMemset(F.phiD, 0, n0 * 8));
  CUDA_CHECK(cudaMemset(F.phi, 0, n0 * 8));
  F.warm = 0;
  F.geom_t0 = 1;
  if (strategy == 3 && c->L.size() > 1) {
    // strategy II (reading O41): the coarse levels' "LIN" operators and smoothers are those of the
    // still-water geometry (eta = 0), formed once here
    double* Xf = dalloc<double>(c, X.size());
    CUDA_CHECK(cudaMemcpy(Xf, F.X0, X.size() * 8, cudaMemcpyDeviceToDevice));
    double* zero = dalloc<double>(c, F.ns);
    CUDA_CHECK(cudaMemset(zero, 0, F.ns * 8));
    const int64_t EN = (int64_t)E * Nf;
    k_fnpf_z<<<fgrid(EN, 256), 256, 0, c->stream>>>(EN, c->L[0].conn, F.gline, F.gsig, F.zb, zero, Xf);
    CUDA_CHECK(cudaGetLastError());
    const int nl = (int)c->L.size();
    for (int li = 1; li < nl; ++li) refresh_level_operator(c, li, Xf, F.gm[li], F.wq[li]);
    for (int li = 1; li + 1 < nl; ++li) fdm_refresh_vertical(c, li, Xf);
    if (c->C.iterative) coarse_refresh_lines(c);
    else coarse_rebuild_dense(c);
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
  }
}

// operators (and, strategies 3 / 4, smoothers) of the levels that follow the free surface (stage.cu)
static void fnpf_geometry(sem_ctx* c, const double* X) {
  Fnpf& F = *c->fnpf;
  const int nl = (int)c->L.size(), st = F.strategy;
  const int nop = (st == 1 || st == 3) ? 1 : nl;
  for (int li = 0; li < nop; ++li) refresh_level_operator(c, li, X, F.gm[li], F.wq[li]);
  if (st == 3 && nl > 1) fdm_refresh_vertical(c, 0, X);
  if (st == 4) {
    for (int li = 0; li + 1 < nl; ++li) fdm_refresh_vertical(c, li, X);
    if (nl > 1) coarse_refresh_lines(c);
  }
}

void fnpf_stage(sem_ctx* c, const double* eta, const double* phis, double* deta, double* dphis, double* w,
                double tol, int linear, sem_report* rep) {
  Fnpf& F = *c->fnpf;
  const int64_t EN = (int64_t)c->E * F.Nf;
  if (!linear) {
    k_fnpf_z<<<fgrid(EN, 256), 256, 0, c->stream>>>(EN, c->L[0].conn, F.gline, F.gsig, F.zb, eta, F.X);
    CUDA_CHECK(cudaGetLastError());
    c->launches++;
    fnpf_geometry(c, F.X);
    F.geom_t0 = 0;
  } else if (!F.geom_t0) {  // back to the still-water operators
    fnpf_geometry(c, F.X0);
    F.geom_t0 = 1;
  }
  k_fnpf_scatter<<<fgrid(F.ns, 256), 256, 0, c->stream>>>(F.ns, F.snode, phis, F.phiD);
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
  int st = do_solve(c, nullptr, F.phiD, tol, F.phi, rep, F.warm, 0);
  if (st != SEM_OK && st != SEM_ENOTCONV) throw SemError(st, "FNPF stage solve failed");
  F.warm = 1;
  CUDA_CHECK(cudaMemsetAsync(F.acc, 0, 5 * F.ns * sizeof(double), c->stream));
  const int64_t nt = (int64_t)F.ntop * F.Nt;
  k_fnpf_recover<<<(int)((nt + 127) / 128), 128, 0, c->stream>>>(F.ntop, F.Nt, F.Nf, c->P, F.top, c->L[0].conn,
                                                                F.gline, linear ? F.X0 : F.X, F.Dtop, F.Dr2, F.Ds2,
                                                                F.phi, eta, phis, F.acc);
  CUDA_CHECK(cudaGetLastError());
  k_fnpf_rates<<<fgrid(F.ns, 256), 256, 0, c->stream>>>(F.ns, F.acc, F.icnt, eta, deta, dphis, w, linear, 9.81);
  CUDA_CHECK(cudaGetLastError());
  c->launches += 2;
}

void fnpf_erk4(sem_ctx* c, double* eta, double* phis, double dt, double tol, int linear, int* iters) {
  Fnpf& F = *c->fnpf;
  const int64_t ns = F.ns;
  const int gs = fgrid(ns, 256);
  int it = 0;
  sem_report R;
  for (int k = 0; k < 4; ++k) {
    const double* e_in = eta;
    const double* p_in = phis;
    if (k > 0) {  // stage state: x + c_k dt k_{k-1}, c = (1/2, 1/2, 1)
      const double a = (k == 3) ? dt : 0.5 * dt;
      k_fnpf_axpy<<<gs, 256, 0, c->stream>>>(ns, eta, a, F.ke + (k - 1) * ns, F.ea);
      k_fnpf_axpy<<<gs, 256, 0, c->stream>>>(ns, phis, a, F.kp + (k - 1) * ns, F.pa);
      CUDA_CHECK(cudaGetLastError());
      c->launches += 2;
      e_in = F.ea;
      p_in = F.pa;
    }
    fnpf_stage(c, e_in, p_in, F.ke + k * ns, F.kp + k * ns, nullptr, tol, linear, &R);
    it += R.iters;
  }
  k_fnpf_rk4<<<gs, 256, 0, c->stream>>>(ns, eta, F.ke, dt);
  k_fnpf_rk4<<<gs, 256, 0, c->stream>>>(ns, phis, F.kp, dt);
  CUDA_CHECK(cudaGetLastError());
  c->launches += 2;
  if (iters) *iters = it;
}

int64_t fnpf_surface(const sem_ctx* c, int32_t* ids) {
  if (!c->fnpf) return -1;
  if (ids) std::copy(c->fnpf->snode_host.begin(), c->fnpf->snode_host.end(), ids);
  return c->fnpf->ns;
}

void fnpf_destroy(sem_ctx* c) {
  delete c->fnpf;
  c->fnpf = nullptr;
}

}  // namespace sem
