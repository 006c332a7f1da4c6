// Per-stage re-formation of the operators and smoothers (the
// strategies of P:350-356, Fig 5.1; readings O41, O42 in DESIGN.md):
//
//   strategy 1 (I)   the finest operator follows the free surface; smoothers and
//                    coarse operators from t = 0 ("pre-compute ... and re-use");
//   strategy 2       every level's operator follows it, smoothers / coarse inverse
//                    from t = 0 ("operators only", not one of the paper's strategies);
//   strategy 3 (II)  the finest operator AND its smoother follow the free surface;
//                    the coarse levels use the still-water (eta = 0) "LIN" operators
//                    and smoothers, formed once (FNPF only: needs the sigma structure);
//   strategy 4 (III) every level's operator and smoother follow it, the P=1 coarse
//                    solve's preconditioner too (iterative coarse solver).
//
// Smoother re-formation is built for the FDM local solves (reading O33): the
// horizontal factors depend on x, y only, which do not move, so only the vertical
// 1D operators K_v, M_v of every element's box change with the layer thicknesses;
// their generalised eigenproblems K_v S = M_v S L (n_v <= 32) are solved here on the
// device, one thread per element (Cholesky of M_v, cyclic Jacobi on L^-1 K_v L^-T),
// with no library call on the per-stage path.  The exact dense inverses (eq 4.4)
// would need a batched factorisation of every R_k A R_k^T per stage (cuSOLVER at
// setup), which is the "by a large margin more expensive" assembly of P:343:
// strategies 3 and 4 need local_solve = 1 (SEM_EUNSUPPORTED otherwise).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"
#include "setup_util.h"

namespace sem {

// one element's vertical box: K_v, M_v from the column's layer thicknesses (mean of the 3 vertical
// edges of the finest nodal map), generalised eigenpairs, written as S_v [i][a] (S^T M S = I), l_v [a]
template <int NV>
__global__ void __launch_bounds__(64) k_fdm_vertical(int E, int p, int Ntg, int pg, const double* __restrict__ X,
                                                     const int32_t* __restrict__ col,
                                                     const int64_t* __restrict__ cfirst,
                                                     const int32_t* __restrict__ colel, const int32_t* __restrict__ z0,
                                                     const int32_t* __restrict__ nvv, const int64_t* __restrict__ voff,
                                                     const int64_t* __restrict__ lvoff,
                                                     const double* __restrict__ kmref, double* __restrict__ Sv,
                                                     double* __restrict__ lv, int* bad) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int n1 = p + 1, c = col[e], lo = z0[e], n = nvv[e];
  const int64_t cb = cfirst[c], nl = cfirst[c + 1] - cb;
  const int Ng = Ntg * (pg + 1);
  const int corner[3] = {0, pg, Ntg - 1};
  double K[NV][NV], M[NV][NV], V[NV][NV];
  for (int i = 0; i < NV; ++i)
    for (int j = 0; j < NV; ++j) K[i][j] = M[i][j] = V[i][j] = 0.0;
  for (int64_t jj = 0; jj < nl; ++jj) {
    const int zb = (int)jj * p;
    if (zb + p < lo || zb > lo + n - 1) continue;
    const int64_t x = colel[cb + jj];
    double d = 0.0;
    for (int v = 0; v < 3; ++v)
      d += X[(x * Ng + corner[v] + Ntg * pg) * 3 + 2] - X[(x * Ng + corner[v]) * 3 + 2];
    d /= 3.0;
    for (int a = 0; a < n1; ++a)
      for (int b = 0; b < n1; ++b) {
        const int za = zb + a - lo, zc = zb + b - lo;
        if (za < 0 || za >= n || zc < 0 || zc >= n) continue;
        K[za][zc] += (2.0 / d) * kmref[a * n1 + b];
        M[za][zc] += (d / 2.0) * kmref[n1 * n1 + a * n1 + b];
      }
  }
  // Cholesky M = L L^T (L in the lower triangle of M)
  for (int j = 0; j < n; ++j) {
    double s = M[j][j];
    for (int k = 0; k < j; ++k) s -= M[j][k] * M[j][k];
    if (!(s > 0.0)) {
      atomicExch(bad, 1);
      return;
    }
    const double ljj = sqrt(s);
    M[j][j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double t = M[i][j];
      for (int k = 0; k < j; ++k) t -= M[i][k] * M[j][k];
      M[i][j] = t / ljj;
    }
  }
  // C = L^-1 K L^-T: K <- L^-1 K (columns), then K <- K L^-T (rows)
  for (int col2 = 0; col2 < n; ++col2)
    for (int i = 0; i < n; ++i) {
      double t = K[i][col2];
      for (int k = 0; k < i; ++k) t -= M[i][k] * K[k][col2];
      K[i][col2] = t / M[i][i];
    }
  for (int row = 0; row < n; ++row)
    for (int i = 0; i < n; ++i) {
      double t = K[row][i];
      for (int k = 0; k < i; ++k) t -= K[row][k] * M[i][k];
      K[row][i] = t / M[i][i];
    }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) K[i][j] = K[j][i] = 0.5 * (K[i][j] + K[j][i]);
  // cyclic Jacobi: K = V diag(l) V^T
  for (int i = 0; i < n; ++i) V[i][i] = 1.0;
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, dia = 0.0;
    for (int i = 0; i < n; ++i) {
      dia += K[i][i] * K[i][i];
      for (int j = i + 1; j < n; ++j) off += K[i][j] * K[i][j];
    }
    if (off <= 1e-32 * dia) break;
    for (int i = 0; i < n - 1; ++i)
      for (int j = i + 1; j < n; ++j) {
        const double kij = K[i][j];
        if (kij == 0.0) continue;
        const double th = (K[j][j] - K[i][i]) / (2.0 * kij);
        const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
        const double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
        for (int k = 0; k < n; ++k) {  // columns i, j
          const double a = K[k][i], b = K[k][j];
          K[k][i] = cs * a - sn * b;
          K[k][j] = sn * a + cs * b;
        }
        for (int k = 0; k < n; ++k) {  // rows i, j
          const double a = K[i][k], b = K[j][k];
          K[i][k] = cs * a - sn * b;
          K[j][k] = sn * a + cs * b;
        }
        for (int k = 0; k < n; ++k) {
          const double a = V[k][i], b = V[k][j];
          V[k][i] = cs * a - sn * b;
          V[k][j] = sn * a + cs * b;
        }
      }
  }
  // S = L^-T V (back substitution per column), written row-major S[i][a]
  double* S = Sv + voff[e];
  for (int a = 0; a < n; ++a) {
    double y[NV];
    for (int i = n - 1; i >= 0; --i) {
      double t = V[i][a];
      for (int k = i + 1; k < n; ++k) t -= M[k][i] * y[k];
      y[i] = t / M[i][i];
    }
    for (int i = 0; i < n; ++i) S[i * n + a] = y[i];
    lv[lvoff[e] + a] = K[a][a];
  }
}

// Thomas factors of every coarse line from the assembled diagonal and vertical off-diagonals
__global__ void k_line_factor(int nlines, const int64_t* __restrict__ loff, const int32_t* __restrict__ lnode,
                              const double* __restrict__ diag, const double* __restrict__ off,
                              double* __restrict__ ta, double* __restrict__ tinv, double* __restrict__ tc, int* bad) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nlines) return;
  const int64_t b = loff[l], e = loff[l + 1];
  double cprev = 0.0;
  for (int64_t t = b; t < e; ++t) {
    const int32_t g = lnode[t];
    const double a = t > b ? off[lnode[t - 1]] : 0.0;
    const double den = diag[g] - a * cprev;
    if (!(den > 0.0)) atomicExch(bad, 1);
    const double cg = t + 1 < e ? off[g] : 0.0;
    ta[t] = a;
    tinv[t] = 1.0 / den;
    tc[t] = cg / den;
    cprev = cg / den;
  }
}

void k_pad_vertical_launch(sem_ctx* c, int li);

// FDM vertical factors of level li from the finest nodal map X (device)
void fdm_refresh_vertical(sem_ctx* c, int li, const double* X) {
  DeviceLevel& L = c->L[li];
  if (!L.fdm) throw SemError(SEM_EUNSUPPORTED, "smoother re-formation needs FDM local solves (local_solve = 1)");
  const int E = c->E, pg = c->P, Ntg = n_tri(pg);
  int* bad = nullptr;
  CUDA_CHECK(cudaMalloc(&bad, sizeof(int)));
  CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
  const int g = (E + 63) / 64;
  if (L.f_nv_max <= 8)
    k_fdm_vertical<8><<<g, 64, 0, c->stream>>>(E, L.p, Ntg, pg, X, L.f_col, L.f_cfirst, L.f_colel, L.f_z0, L.f_nv,
                                                L.f_voff, L.f_lvoff, L.f_kmref, L.f_Sv, L.f_lv, bad);
  else if (L.f_nv_max <= 16)
    k_fdm_vertical<16><<<g, 64, 0, c->stream>>>(E, L.p, Ntg, pg, X, L.f_col, L.f_cfirst, L.f_colel, L.f_z0, L.f_nv,
                                                 L.f_voff, L.f_lvoff, L.f_kmref, L.f_Sv, L.f_lv, bad);
  else if (L.f_nv_max <= 32)
    k_fdm_vertical<32><<<g, 64, 0, c->stream>>>(E, L.p, Ntg, pg, X, L.f_col, L.f_cfirst, L.f_colel, L.f_z0, L.f_nv,
                                                 L.f_voff, L.f_lvoff, L.f_kmref, L.f_Sv, L.f_lv, bad);
  else
    throw SemError(SEM_EUNSUPPORTED, "vertical FDM box larger than 32 nodes");
  CUDA_CHECK(cudaGetLastError());
  k_pad_vertical_launch(c, li);
  int hb = 0;
  CUDA_CHECK(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
  cudaFree(bad);
  c->launches += 2;
  if (hb) throw SemError(SEM_ESINGULAR, "FDM vertical mass matrix not SPD");
}

// The iterative coarse solve's line-Jacobi preconditioner from the coarsest level's current G
void coarse_refresh_lines(sem_ctx* c) {
  Coarse& C = c->C;
  if (!C.iterative) throw SemError(SEM_EUNSUPPORTED, "re-forming the coarse operator every stage needs the "
                                                     "iterative coarse solver (coarse_solver = 1)");
  const int li = (int)c->L.size() - 1;
  DeviceLevel& L = c->L[li];
  Scratch sc;
  double* diag = sc.get<double>((size_t)L.n);
  double* off = sc.get<double>((size_t)L.n);
  double* d_D = sc.put(L.ref.Dfull);
  CUDA_CHECK(cudaMemsetAsync(diag, 0, sizeof(double) * L.n, c->stream));
  CUDA_CHECK(cudaMemsetAsync(off, 0, sizeof(double) * L.n, c->stream));
  const int E = c->E;
  const int64_t chunk = std::min<int64_t>(E, 1 << 20);
  double* Ae = sc.get<double>((size_t)chunk * L.N * L.N);
  for (int64_t e0 = 0; e0 < E; e0 += chunk) {
    const int ne = (int)std::min<int64_t>(chunk, E - e0);
    launch_elem_matrices(c, li, d_D, Ae, (int)e0, ne);
    launch_diag_accum_range(c, L.conn + (size_t)e0 * L.N, L.N, ne, Ae, diag);
    launch_offdiag_accum(c, L.conn + (size_t)e0 * L.N, ne, Ae, off);
  }
  int* bad = sc.get<int>(1);
  CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
  k_line_factor<<<(C.nlines + 127) / 128, 128, 0, c->stream>>>(C.nlines, C.loff, C.lnode, diag, off, C.ta, C.tinv,
                                                               C.tc, bad);
  CUDA_CHECK(cudaGetLastError());
  int hb = 0;
  CUDA_CHECK(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
  if (hb) throw SemError(SEM_ESINGULAR, "coarse line block is not SPD");
}

// Operator of level li (G, the a-tile copy, the P <= 2 element matrices) from the finest nodal map X
void refresh_level_operator(sem_ctx* c, int li, const double* X, const double* d_gm, const double* d_w) {
  DeviceLevel& L = c->L[li];
  if (launch_geometry(c, li, X, d_gm, n_prism(c->P, c->PZ), d_w))
    throw SemError(SEM_EBADELEM, "detJ <= 0 at a cubature point");
  if (L.Gw) build_g_tiles(c, li);
  if (L.Ae1) {
    Scratch s2;
    build_p1_matrices(c, li, s2.put(L.ref.Dfull));
  }
}

}  // namespace sem
