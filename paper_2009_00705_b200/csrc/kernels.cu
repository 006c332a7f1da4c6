// Device kernels of the hot path (sm_100a, FP64).
//
//  k_apply<P>      a2/a3/a4: y (+/-)= sum_e Q_e^T D^T (G (.) D Q_e u), matrix-free
//                  sum-factorised prism operator (eq 3.8) with
//                  gather-scatter of shared nodes and Dirichlet mask.
//  k_schwarz       a5/a6: u += W sum_k R_k^T B_k^-1 R_k r (eq 4.4-4.6),
//                  packed-symmetric 16x16-tile GEMV per subdomain, HBM streaming.
//  k_restrict      a7: r_c = P^T r_f (eq 4.3), sum-factorised.
//  k_prolong       a9: u_f += P u_c, sum-factorised.
//  k_coarse_symv   a8: z = A_1^-1 r, packed lower tiles of the symmetric inverse.
//  vector kernels  a11: fused PCG updates and dot products (Alg 4.3).
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"

namespace sem {

// ============================================================== operator apply
template <int P>
struct AD {
  static constexpr int N1 = P + 1;
  static constexpr int NT = N1 * (N1 + 1) / 2;
  static constexpr int N = NT * N1;
  static constexpr int QT = N1 * N1;
  static constexpr int Q = QT * N1;
  static constexpr int NTP = NT | 1;  // odd row stride: conflict-free strided smem reads
  static constexpr int N1P = N1 | 1;
  static constexpr int T = 256;
  static constexpr int NE = (3 * QT >= T) ? 1 : T / (3 * QT);
  static constexpr int SM_MATS = 3 * QT * NTP + 2 * N1 * N1;
  static constexpr int SM_U = NE * N;
  static constexpr int SM_UU = NE * 3 * QT * N1P;
  static constexpr int SM_G = NE * 3 * Q;
  static constexpr int SMEM = (SM_MATS + SM_U + SM_UU + SM_G) * (int)sizeof(double);
  static constexpr int IT3 = (NE * Q + T - 1) / T;
};

template <int P>
__global__ void __launch_bounds__(256) k_apply(int E, const int32_t* __restrict__ conn,
                                               const double* __restrict__ G, const double* __restrict__ mats,
                                               const double* __restrict__ u, double* __restrict__ y, int flags,
                                               const int32_t* __restrict__ elist) {
  using D = AD<P>;
  extern __shared__ double sm[];
  double* sB0 = sm;
  double* sBr = sB0 + D::QT * D::NTP;
  double* sBs = sBr + D::QT * D::NTP;
  double* sBt = sBs + D::QT * D::NTP;
  double* sDt = sBt + D::N1 * D::N1;
  double* su = sm + D::SM_MATS;
  double* sU = su + D::SM_U;
  double* sg = sU + D::SM_UU;
  const int tid = threadIdx.x;
  const int e0 = blockIdx.x * D::NE;

  for (int i = tid; i < D::SM_MATS; i += D::T) sm[i] = __ldg(mats + i);
  // gather u_e = Q_e u (Dirichlet entries as 0 unless AP_GATHER_ALL)
  // slot e0 + j holds element elist[e0 + j] (deterministic colour batches) or e0 + j
  auto elem = [&](int slot) { return elist ? __ldg(elist + slot) : slot; };
  for (int i = tid; i < D::NE * D::N; i += D::T) {
    const int e = e0 + i / D::N;
    double v = 0.0;
    if (e < E) {
      const int c = __ldg(conn + (size_t)elem(e) * D::N + (i % D::N));
      if (c >= 0) v = u[c];
      else if (flags & AP_GATHER_ALL) v = u[~c];
    }
    su[i] = v;
  }
  // prefetch this thread's geometric factors (consumed in stage 3)
  double gv[D::IT3][6];
#pragma unroll
  for (int k = 0; k < D::IT3; ++k) {
    const int it = tid + k * D::T;
    const int e = it / D::Q, q = it % D::Q;
    if (it < D::NE * D::Q && e0 + e < E) {
      const double* g = G + (size_t)elem(e0 + e) * 6 * D::Q + q;
#pragma unroll
      for (int c = 0; c < 6; ++c) gv[k][c] = __ldg(g + c * D::Q);
    } else {
#pragma unroll
      for (int c = 0; c < 6; ++c) gv[k][c] = 0.0;
    }
  }
  __syncthreads();
  // stage 1: triangle contraction  U_c[a][l] = sum_m B_c[a][m] u[m][l]
  for (int it = tid; it < D::NE * 3 * D::QT; it += D::T) {
    const int e = it / (3 * D::QT), rem = it % (3 * D::QT), c = rem / D::QT, a = rem % D::QT;
    const double* B = (c == 0 ? sBr : (c == 1 ? sBs : sB0)) + a * D::NTP;
    const double* ue = su + e * D::N;
    double acc[D::N1];
#pragma unroll
    for (int l = 0; l < D::N1; ++l) acc[l] = 0.0;
#pragma unroll 4
    for (int m = 0; m < D::NT; ++m) {
      const double b = B[m];
#pragma unroll
      for (int l = 0; l < D::N1; ++l) acc[l] = fma(b, ue[m + D::NT * l], acc[l]);
    }
    double* o = sU + ((e * 3 + c) * D::QT + a) * D::N1P;
#pragma unroll
    for (int l = 0; l < D::N1; ++l) o[l] = acc[l];
  }
  __syncthreads();
  // stage 2: vertical  g_c[a][q] = sum_l M_c[q][l] U_c[a][l]   (M = Bt for r,s; Dt for t)
  for (int it = tid; it < D::NE * 3 * D::QT; it += D::T) {
    const int e = it / (3 * D::QT), rem = it % (3 * D::QT), c = rem / D::QT, a = rem % D::QT;
    const double* row = sU + ((e * 3 + c) * D::QT + a) * D::N1P;
    double v[D::N1];
#pragma unroll
    for (int l = 0; l < D::N1; ++l) v[l] = row[l];
    const double* M = (c < 2) ? sBt : sDt;
    double* o = sg + (e * 3 + c) * D::Q + a;
#pragma unroll
    for (int q = 0; q < D::N1; ++q) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < D::N1; ++l) s = fma(M[q * D::N1 + l], v[l], s);
      o[q * D::QT] = s;
    }
  }
  __syncthreads();
  // stage 3: w = G g at every cubature point
#pragma unroll
  for (int k = 0; k < D::IT3; ++k) {
    const int it = tid + k * D::T;
    if (it < D::NE * D::Q) {
      const int e = it / D::Q, q = it % D::Q;
      double* g = sg + e * 3 * D::Q + q;
      const double gr = g[0], gs = g[D::Q], gt = g[2 * D::Q];
      g[0] = gv[k][0] * gr + gv[k][1] * gs + gv[k][2] * gt;
      g[D::Q] = gv[k][1] * gr + gv[k][3] * gs + gv[k][4] * gt;
      g[2 * D::Q] = gv[k][2] * gr + gv[k][4] * gs + gv[k][5] * gt;
    }
  }
  __syncthreads();
  // stage 4: vertical transpose  V_c[a][l] = sum_q M_c[q][l] w_c[a][q]
  for (int it = tid; it < D::NE * 3 * D::QT; it += D::T) {
    const int e = it / (3 * D::QT), rem = it % (3 * D::QT), c = rem / D::QT, a = rem % D::QT;
    const double* src = sg + (e * 3 + c) * D::Q + a;
    double w[D::N1];
#pragma unroll
    for (int q = 0; q < D::N1; ++q) w[q] = src[q * D::QT];
    const double* M = (c < 2) ? sBt : sDt;
    double* o = sU + ((e * 3 + c) * D::QT + a) * D::N1P;
#pragma unroll
    for (int l = 0; l < D::N1; ++l) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < D::N1; ++q) s = fma(M[q * D::N1 + l], w[q], s);
      o[l] = s;
    }
  }
  __syncthreads();
  // stage 5: triangle transpose, one partial per gradient component c
  double* part = sg;  // [3][NE][N]
  for (int it = tid; it < D::NE * 3 * D::NT; it += D::T) {
    const int e = it / (3 * D::NT), rem = it % (3 * D::NT), c = rem / D::NT, m = rem % D::NT;
    const double* B = (c == 0 ? sBr : (c == 1 ? sBs : sB0)) + m;
    const double* V = sU + (e * 3 + c) * D::QT * D::N1P;
    double acc[D::N1];
#pragma unroll
    for (int l = 0; l < D::N1; ++l) acc[l] = 0.0;
#pragma unroll 4
    for (int a = 0; a < D::QT; ++a) {
      const double b = B[a * D::NTP];
#pragma unroll
      for (int l = 0; l < D::N1; ++l) acc[l] = fma(b, V[a * D::N1P + l], acc[l]);
    }
    double* o = part + (c * D::NE + e) * D::N + m;
#pragma unroll
    for (int l = 0; l < D::N1; ++l) o[D::NT * l] = acc[l];
  }
  __syncthreads();
  // stage 6: scatter-add y = Q_e^T y_e (gather-scatter of shared nodes)
  const double sgn = (flags & AP_NEGATE) ? -1.0 : 1.0;
  for (int it = tid; it < D::NE * D::N; it += D::T) {
    const int e = it / D::N, n = it % D::N;
    if (e0 + e >= E) continue;
    const double v = part[(0 * D::NE + e) * D::N + n] + part[(1 * D::NE + e) * D::N + n] +
                     part[(2 * D::NE + e) * D::N + n];
    const int c = __ldg(conn + (size_t)elem(e0 + e) * D::N + n);
    if (c >= 0) atomicAdd(y + c, sgn * v);
    else if (flags & AP_SCATTER_ALL) atomicAdd(y + ~c, sgn * v);
  }
}

template <int P>
static void apply_P(sem_ctx* c, const DeviceLevel& L, const double* u, double* y, int flags) {
  using D = AD<P>;
  static int attr[kMaxDev] = {0};
  smem_opt_in(k_apply<P>, D::SMEM, attr);
  if (c->E_own == 0) return;
  if (c->det.on) {  // deterministic: one launch per element colour (no two elements of a colour share a node)
    for (size_t k = 0; k + 1 < c->det.ecol_off.size(); ++k) {
      const int cnt = (int)(c->det.ecol_off[k + 1] - c->det.ecol_off[k]);
      k_apply<P><<<(cnt + D::NE - 1) / D::NE, D::T, D::SMEM, c->stream>>>(cnt, L.conn, L.G, L.mats, u, y, flags,
                                                                        c->det.ecol + c->det.ecol_off[k]);
    }
    CUDA_CHECK(cudaGetLastError());
    return;
  }
  const int grid = (c->E_own + D::NE - 1) / D::NE;
  k_apply<P><<<grid, D::T, D::SMEM, c->stream>>>(c->E_own, L.conn, L.G, L.mats, u, y, flags, nullptr);
  CUDA_CHECK(cudaGetLastError());
}

// Operator of an anisotropic level P_p(triangle) x P_q(t), any orders at run
// time: one CTA per element, the same sum factorisation as k_apply<P> (eq 3.8) with the vertical
// stages over q + 1 nodes / Gauss points.  Shared memory: the reference matrices, u_e, Ut/Udt,
// the three cubature-point fields and Vt/Vdt.  elist: deterministic colour batches.
__global__ void __launch_bounds__(128) k_apply_pq(int E, int nt, int n1, int qt, const int32_t* __restrict__ conn,
                                                  const double* __restrict__ G, const double* __restrict__ mats,
                                                  const double* __restrict__ u, double* __restrict__ y, int flags,
                                                  const int32_t* __restrict__ elist) {
  extern __shared__ double sm[];
  const int ntp = nt | 1, N = nt * n1, qv = n1, Q = qt * qv;
  const int e = elist ? elist[blockIdx.x] : blockIdx.x;
  if (blockIdx.x >= E) return;
  const double* B0 = mats;                 // [qt][ntp]
  const double* Br = B0 + qt * ntp;
  const double* Bs = Br + qt * ntp;
  const double* Bt = Bs + qt * ntp;        // [qv][n1]
  const double* Dt = Bt + n1 * n1;
  double* ue = sm;                         // [N]
  double* Ut = ue + N;                     // [nt][qv]
  double* Ud = Ut + nt * qv;
  double* g = Ud + nt * qv;                // [3][Q]
  double* Vt = g + 3 * Q;                  // [nt][qv]
  double* Vd = Vt + nt * qv;
  const int tid = threadIdx.x, T = blockDim.x;
  const int32_t* ce = conn + (size_t)e * N;
  for (int i = tid; i < N; i += T) {
    const int c = __ldg(ce + i);
    ue[i] = c >= 0 ? u[c] : ((flags & AP_GATHER_ALL) ? u[~c] : 0.0);
  }
  __syncthreads();
  // A: Ut[m][z] = sum_l u[m + nt l] Bt[z][l], Ud with Dt
  for (int i = tid; i < nt * qv; i += T) {
    const int m = i / qv, z = i % qv;
    double a = 0.0, b = 0.0;
    for (int l = 0; l < n1; ++l) {
      const double v = ue[m + nt * l];
      a = fma(v, __ldg(Bt + z * n1 + l), a);
      b = fma(v, __ldg(Dt + z * n1 + l), b);
    }
    Ut[i] = a;
    Ud[i] = b;
  }
  __syncthreads();
  // B and G: at every point (a, z): (g_r, g_s, g_0) = (Br Ut, Bs Ut, B0 Ud), w = G g
  for (int pt = tid; pt < Q; pt += T) {
    const int a = pt % qt, z = pt / qt;
    double gr = 0.0, gs = 0.0, g0 = 0.0;
    for (int m = 0; m < nt; ++m) {
      const double ut = Ut[m * qv + z], ud = Ud[m * qv + z];
      gr = fma(__ldg(Br + a * ntp + m), ut, gr);
      gs = fma(__ldg(Bs + a * ntp + m), ut, gs);
      g0 = fma(__ldg(B0 + a * ntp + m), ud, g0);
    }
    const double* Gp = G + (size_t)e * 6 * Q + pt;
    const double xx = __ldg(Gp), xy = __ldg(Gp + Q), xz = __ldg(Gp + 2 * Q), yy = __ldg(Gp + 3 * Q),
                 yz = __ldg(Gp + 4 * Q), zz = __ldg(Gp + 5 * Q);
    g[pt] = xx * gr + xy * gs + xz * g0;
    g[Q + pt] = xy * gr + yy * gs + yz * g0;
    g[2 * Q + pt] = xz * gr + yz * gs + zz * g0;
  }
  __syncthreads();
  // B^T: Vt[m][z] = sum_a Br[a][m] w_r + Bs[a][m] w_s, Vd[m][z] = sum_a B0[a][m] w_0
  for (int i = tid; i < nt * qv; i += T) {
    const int m = i / qv, z = i % qv;
    double a1 = 0.0, a2 = 0.0;
    for (int a = 0; a < qt; ++a) {
      const int pt = a + qt * z;
      a1 = fma(__ldg(Br + a * ntp + m), g[pt], fma(__ldg(Bs + a * ntp + m), g[Q + pt], a1));
      a2 = fma(__ldg(B0 + a * ntp + m), g[2 * Q + pt], a2);
    }
    Vt[i] = a1;
    Vd[i] = a2;
  }
  __syncthreads();
  // A^T + scatter: y[m + nt l] (+/-)= sum_z Vt[m][z] Bt[z][l] + Vd[m][z] Dt[z][l]
  const double sgn = (flags & AP_NEGATE) ? -1.0 : 1.0;
  for (int i = tid; i < N; i += T) {
    const int m = i % nt, l = i / nt;
    double acc = 0.0;
    for (int z = 0; z < qv; ++z)
      acc = fma(Vt[m * qv + z], __ldg(Bt + z * n1 + l), fma(Vd[m * qv + z], __ldg(Dt + z * n1 + l), acc));
    const int c = __ldg(ce + i);
    if (c >= 0) atomicAdd(y + c, sgn * acc);
    else if (flags & AP_SCATTER_ALL) atomicAdd(y + ~c, sgn * acc);
  }
}

static void apply_pq(sem_ctx* c, const DeviceLevel& L, const double* u, double* y, int flags) {
  const LevelRef& R = L.ref;
  const int smem = (R.N + 4 * R.nt * R.qv + 3 * R.Q) * (int)sizeof(double);
  static int attr[kMaxDev] = {0};
  if (smem > 48 * 1024) smem_opt_in(k_apply_pq, smem, attr);
  if (c->E_own == 0) return;
  if (c->det.on) {
    for (size_t k = 0; k + 1 < c->det.ecol_off.size(); ++k) {
      const int cnt = (int)(c->det.ecol_off[k + 1] - c->det.ecol_off[k]);
      k_apply_pq<<<cnt, 128, smem, c->stream>>>(cnt, R.nt, R.n1, R.qt, L.conn, L.G, L.mats, u, y, flags,
                                                c->det.ecol + c->det.ecol_off[k]);
    }
  } else {
    k_apply_pq<<<c->E_own, 128, smem, c->stream>>>(c->E_own, R.nt, R.n1, R.qt, L.conn, L.G, L.mats, u, y, flags,
                                                   nullptr);
  }
  CUDA_CHECK(cudaGetLastError());
}

// P <= 2 operators: one thread per element, y_e = A_e u_e with the element matrix
// precomputed at setup (N(N+1)/2 packed entries, structure-of-arrays for coalescing).
// P = 1: 168 B per element instead of G's 384 B; P = 2: 1368 B vs 1296 B, but no
// padded tensor-core tiles (N = 18 fills 8x8 fragments poorly).
template <int N>
__global__ void __launch_bounds__(128) k_apply_em(int E, int64_t ld, const int32_t* __restrict__ conn,
                                                  const double* __restrict__ Aem, const double* __restrict__ u,
                                                  double* __restrict__ y, int flags) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  int g[N];
  double x[N], acc[N];
#pragma unroll
  for (int i = 0; i < N; ++i) g[i] = __ldg(conn + (size_t)e * N + i);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    x[i] = (g[i] >= 0 || (flags & AP_GATHER_ALL)) ? __ldg(u + (g[i] >= 0 ? g[i] : ~g[i])) : 0.0;
    acc[i] = 0.0;
  }
  // packed lower triangle, row r: entries (r, 0..r); A symmetric
  int k = 0;
#pragma unroll
  for (int r = 0; r < N; ++r) {
#pragma unroll
    for (int q = 0; q <= r; ++q) {
      const double a = __ldg(Aem + (size_t)(k++) * ld + e);
      acc[r] = fma(a, x[q], acc[r]);
      if (q != r) acc[q] = fma(a, x[r], acc[q]);
    }
  }
  const double sgn = (flags & AP_NEGATE) ? -1.0 : 1.0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if (g[i] >= 0) atomicAdd(y + g[i], sgn * acc[i]);
    else if (flags & AP_SCATTER_ALL) atomicAdd(y + ~g[i], sgn * acc[i]);
  }
}

__global__ void k_pack_em(int N, int ne, int e0, int64_t ld, const double* __restrict__ Ae, double* __restrict__ Aem) {
  const int le = blockIdx.x * blockDim.x + threadIdx.x;
  if (le >= ne) return;
  int k = 0;
  for (int r = 0; r < N; ++r)
    for (int q = 0; q <= r; ++q) Aem[(size_t)(k++) * ld + e0 + le] = Ae[(size_t)le * N * N + r * N + q];
}

void build_p1_matrices(sem_ctx* c, int level, const double* d_D) {
  DeviceLevel& L = c->L[level];
  if (L.p > 2) return;
  const int E = c->E, N = L.N, NP = N * (N + 1) / 2;
  if (!L.Ae1) {  // refreshed in place by sem_update_geometry
    CUDA_CHECK(cudaMalloc(&L.Ae1, (size_t)NP * E * sizeof(double)));
    c->allocs.push_back(L.Ae1);
    c->device_bytes += (int64_t)NP * E * 8;
  }
  const int chunk = 1 << 18;
  double* Ae = nullptr;
  CUDA_CHECK(cudaMalloc(&Ae, (size_t)std::min(chunk, E) * N * N * sizeof(double)));
  for (int e0 = 0; e0 < E; e0 += chunk) {
    const int ne = std::min(chunk, E - e0);
    launch_elem_matrices(c, level, d_D, Ae, e0, ne);
    k_pack_em<<<(ne + 255) / 256, 256, 0, c->stream>>>(N, ne, e0, (int64_t)E, Ae, L.Ae1);
    CUDA_CHECK(cudaGetLastError());
  }
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
  CUDA_CHECK(cudaFree(Ae));
}

// operator over an element subset (partitioned overlap, dist.cu): the same kernel choice as
// launch_apply for the kernels that take element lists; false if none applies
bool launch_apply_subset(sem_ctx* c, int level, const double* u, double* y, int flags, const int32_t* elist, int ne) {
  if (c->det.on || !(c->opts.apply_kernel == 0 || c->opts.apply_kernel >= 3)) return false;
  if ((c->opts.apply_kernel == 4 || (c->opts.apply_kernel == 0 && c->L[level].p <= 5)) &&
      launch_apply_qs(c, level, u, y, flags, elist, ne))
    return true;
  return launch_apply_warp(c, level, u, y, flags, elist, ne);
}

void launch_apply(sem_ctx* c, int level, const double* u, double* y, int flags) {
  if (c->L[level].p != c->L[level].q) {  // anisotropic level
    if (!c->det.on && (c->opts.apply_kernel == 0 || c->opts.apply_kernel == 4) &&
        launch_apply_qs(c, level, u, y, flags, nullptr, 0))
      return;   // tensor-core kernel for P_p x P_q, 3 <= p <= 5, 1 <= q <= 5
    apply_pq(c, c->L[level], u, y, flags);
    c->launches++;
    return;
  }
  if (!c->det.on) {
    const DeviceLevel& L = c->L[level];
    if (L.p <= 2 && L.Ae1 && (c->opts.apply_kernel == 0 || c->opts.apply_kernel >= 3)) {
      if (c->E_own > 0) {
        if (L.p == 1)
          k_apply_em<6><<<(c->E_own + 127) / 128, 128, 0, c->stream>>>(c->E_own, (int64_t)c->E, L.conn, L.Ae1, u,
                                                                        y, flags);
        else
          k_apply_em<18><<<(c->E_own + 127) / 128, 128, 0, c->stream>>>(c->E_own, (int64_t)c->E, L.conn, L.Ae1,
                                                                         u, y, flags);
        CUDA_CHECK(cudaGetLastError());
      }
      c->launches++;
      return;
    }
  }
  // default (0): four elements per group of warps (k_apply_qs) at p = 3..5 (config 3 p = 5: 289 vs
  // 312 us for k_apply_warp; config 4 p = 3: 683 vs 800 us for k_apply_quad), the warp-per-element
  // kernel at p = 6 (699 vs 938 us)
  if (!c->det.on && (c->opts.apply_kernel == 4 || (c->opts.apply_kernel == 0 && c->L[level].p <= 5)) &&
      launch_apply_qs(c, level, u, y, flags, nullptr, 0))
    return;
  if (!c->det.on && c->opts.apply_kernel == 3 && launch_apply_quad(c, level, u, y, flags)) return;
  if (!c->det.on && (c->opts.apply_kernel == 0 || c->opts.apply_kernel >= 3) && launch_apply_warp(c, level, u, y, flags))
    return;
  if (!c->det.on && c->opts.apply_kernel != 1) {
    launch_apply_dmma(c, level, u, y, flags);
    return;
  }
  const DeviceLevel& L = c->L[level];
  switch (L.p) {
    case 1: apply_P<1>(c, L, u, y, flags); break;
    case 2: apply_P<2>(c, L, u, y, flags); break;
    case 3: apply_P<3>(c, L, u, y, flags); break;
    case 4: apply_P<4>(c, L, u, y, flags); break;
    case 5: apply_P<5>(c, L, u, y, flags); break;
    case 6: apply_P<6>(c, L, u, y, flags); break;
    case 7: apply_P<7>(c, L, u, y, flags); break;
    case 8: apply_P<8>(c, L, u, y, flags); break;
    default: throw SemError(SEM_EINVAL, "order out of range");
  }
  c->launches++;
}

// ============================================================== masked vector init
// mode 0: dst = free ? 0 : src     (masked apply: identity rows on Dirichlet nodes)
// mode 1: dst = free ? src : 0     (residual / RHS restricted to free nodes)
// mode 2: dst = owned&free ? src : 0   (partitioned: each global node counted once)
// mode 3: dst = Dirichlet ? src : dst  (identity rows, free entries kept)
__global__ void k_init_masked(int64_t n, const uint8_t* __restrict__ dmask, const uint8_t* __restrict__ ownfree,
                              const double* __restrict__ src, double* __restrict__ dst, int mode) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool dir = dmask[i];
    if (mode == 0) dst[i] = dir ? (src ? src[i] : 0.0) : 0.0;
    else if (mode == 1) dst[i] = dir ? 0.0 : (src ? src[i] : 0.0);
    else if (mode == 2) dst[i] = ownfree[i] ? (src ? src[i] : 0.0) : 0.0;
    else if (dir) dst[i] = src[i];
  }
}

static int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return (int)g;
}

void launch_init_masked(sem_ctx* c, int level, const double* src, double* dst, int mode) {
  const DeviceLevel& L = c->L[level];
  if (mode == 2 && !L.ownfree) mode = 1;  // single domain: every free node is owned
  k_init_masked<<<grid_for(L.n, 256), 256, 0, c->stream>>>(L.n, L.dmask, L.ownfree, src, dst, mode);
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
}

// ============================================================== Schwarz smoother
// One CTA (8 warps) per subdomain k.  B_k^-1 is stored as the lower triangle of
// 16x16 tiles (diagonal tiles full), row-major inside a tile, tiles in order
// (0,0),(1,0),(1,1),(2,0),...  Each warp streams whole tiles with coalesced
// 256-byte loads; row sums are reduced with a value-halving shuffle butterfly,
// column sums (the symmetric half) accumulated per lane; per-warp private
// accumulators in shared memory avoid atomics.
// the lane's 8 entries of a packed tile (layouts in k_pack_tiles)
__device__ __forceinline__ void load8(const double* tile, int lane, double (&a)[8]) {
#pragma unroll
  for (int m = 0; m < 8; ++m) a[m] = __ldg(tile + 32 * m + lane);
}
__device__ __forceinline__ void load8(const float* tile, int lane, double (&a)[8]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 v = __ldg(reinterpret_cast<const float2*>(tile + 64 * q) + lane);
    a[2 * q] = v.x;
    a[2 * q + 1] = v.y;
  }
}

template <class TT>
__global__ void __launch_bounds__(256) k_schwarz(const int32_t* __restrict__ sidx, const int64_t* __restrict__ sidx_off,
                                                 const int64_t* __restrict__ tile_off,
                                                 const TT* __restrict__ tiles, const double* __restrict__ W,
                                                 const double* __restrict__ r, double* __restrict__ u, int transpose,
                                                 int npad_max, const int32_t* __restrict__ slist) {
  extern __shared__ double sm[];
  double* x = sm;                 // [npad_max]
  double* yw = sm + npad_max;     // [8][npad_max]
  const int k = slist ? slist[blockIdx.x] : blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = sidx_off[k];
  const int np = (int)(sidx_off[k + 1] - base);
  const int T = np >> 4;
  for (int i = tid; i < np; i += 256) {
    const int g = sidx[base + i];
    double v = 0.0;
    if (g >= 0) {
      v = r[g];
      if (transpose) v *= W[g];
    }
    x[i] = v;
  }
  for (int i = tid; i < 8 * np; i += 256) yw[(i / np) * npad_max + (i % np)] = 0.0;
  __syncthreads();
  double* y = yw + warp * npad_max;
  const TT* tk = tiles + tile_off[k];
  const int ntiles = T * (T + 1) / 2;
  const int r0 = lane >> 4, cc = lane & 15;
  auto tile_apply = [&](const double (&a)[8], int I, int J) {
    const double xc = x[16 * J + cc];
    double v[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) v[m] = a[m] * xc;
    if (I != J) {
      double col = 0.0;
#pragma unroll
      for (int m = 0; m < 8; ++m) col = fma(a[m], x[16 * I + 2 * m + r0], col);
      col += __shfl_xor_sync(0xffffffffu, col, 16);
      if (r0 == 0) y[16 * J + cc] += col;
    }
    // value-halving butterfly: 8 row partials over the 16 lanes of a half-warp
    const bool b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
    double k4[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double send = b3 ? v[j] : v[j + 4];
      const double keep = b3 ? v[j + 4] : v[j];
      k4[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    double k2[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double send = b2 ? k4[j] : k4[j + 2];
      const double keep = b2 ? k4[j + 2] : k4[j];
      k2[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    double k1;
    {
      const double send = b1 ? k2[0] : k2[1];
      const double keep = b1 ? k2[1] : k2[0];
      k1 = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    k1 += __shfl_xor_sync(0xffffffffu, k1, 1);
    if ((lane & 1) == 0) {
      const int m = (b1 ? 1 : 0) + (b2 ? 2 : 0) + (b3 ? 4 : 0);
      y[16 * I + 2 * m + r0] += k1;
    }
  };
  // tiles t = warp, warp + 8, ...: (I, J) advanced incrementally along the packed lower triangle
  int I = 0, J = warp;
  while (J > I) { J -= I + 1; ++I; }
  for (int t = warp; t < ntiles; t += 8) {
    double a[8];
    load8(tk + (size_t)t * 256, lane, a);
    tile_apply(a, I, J);
    J += 8;
    while (J > I) { J -= I + 1; ++I; }
  }
  __syncthreads();
  for (int i = tid; i < np; i += 256) {
    const int g = sidx[base + i];
    if (g < 0) continue;
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += yw[w * npad_max + i];
    if (!transpose) s *= W[g];
    atomicAdd(u + g, s);
  }
}

void launch_schwarz(sem_ctx* c, int level, const double* r, double* u, int transpose) {
  const DeviceLevel& L = c->L[level];
  if (L.fdm) {
    launch_fdm(c, level, r, u, transpose);
    if (L.nsub == 0) return;  // else: the dense subdomains of an O35 hybrid follow
  }
  launch_schwarz_dense(c, level, r, u, transpose);
}

// the dense (exact local inverse) subdomains of a level: all of them, or the O35 subset of an
// FDM level
void launch_schwarz_dense(sem_ctx* c, int level, const double* r, double* u, int transpose) {
  const DeviceLevel& L = c->L[level];
  const int npad = 16 * L.max_tiles_1d;
  const int smem = 9 * npad * (int)sizeof(double);
  static int attr_set[kMaxDev] = {0}, attr_set32[kMaxDev] = {0};
  if (L.nsub == 0) return;
  if (smem > 48 * 1024) {
    smem_opt_in(k_schwarz<float>, smem, attr_set32);
    smem_opt_in(k_schwarz<double>, smem, attr_set);
  }
  // deterministic: one launch per subdomain colour (node-disjoint subdomains)
  const size_t ncol = c->det.on ? L.scol_off.size() - 1 : 1;
  for (size_t q = 0; q < ncol; ++q) {
    const int nb = c->det.on ? (int)(L.scol_off[q + 1] - L.scol_off[q]) : L.nsub;
    const int32_t* sl = c->det.on ? L.scol + L.scol_off[q] : nullptr;
    if (nb == 0) continue;
    if (L.tiles32)  // mixed precision: FP32 storage of the exact inverses, FP64 arithmetic
      k_schwarz<float><<<nb, 256, smem, c->stream>>>(L.sidx, L.sidx_off, L.tile_off, L.tiles32, L.W, r, u,
                                                     transpose, npad, sl);
    else
      k_schwarz<double><<<nb, 256, smem, c->stream>>>(L.sidx, L.sidx_off, L.tile_off, L.tiles, L.W, r, u,
                                                      transpose, npad, sl);
  }
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
}

// dense Schwarz sweep over a subset of the subdomains (dist.cu: interface subdomains first)
bool launch_schwarz_list(sem_ctx* c, int level, const double* r, double* u, int transpose, const int32_t* slist,
                         int nb) {
  const DeviceLevel& L = c->L[level];
  if (L.fdm || c->det.on || L.nsub == 0) return false;
  if (nb == 0) return true;
  const int npad = 16 * L.max_tiles_1d;
  const int smem = 9 * npad * (int)sizeof(double);
  static int attr_set[kMaxDev] = {0}, attr_set32[kMaxDev] = {0};
  if (smem > 48 * 1024) {
    smem_opt_in(k_schwarz<float>, smem, attr_set32);
    smem_opt_in(k_schwarz<double>, smem, attr_set);
  }
  if (L.tiles32)
    k_schwarz<float><<<nb, 256, smem, c->stream>>>(L.sidx, L.sidx_off, L.tile_off, L.tiles32, L.W, r, u, transpose,
                                                   npad, slist);
  else
    k_schwarz<double><<<nb, 256, smem, c->stream>>>(L.sidx, L.sidx_off, L.tile_off, L.tiles, L.W, r, u, transpose,
                                                    npad, slist);
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
  return true;
}

// ============================================================== transfers
// Prolongation u_f += P u_c with P evaluated element by element, each fine node
// written only by its owner element (first element containing it): P[j][i] =
// N_i^c(x_j^f) exactly as in P:285-291; restriction is its exact transpose.
__global__ void k_prolong(int E, int ntf, int n1f, int ntc, int n1c, const int32_t* __restrict__ connf,
                          const uint8_t* __restrict__ owner, const int32_t* __restrict__ connc,
                          const double* __restrict__ Itri, const double* __restrict__ I1,
                          const double* __restrict__ uc, double* __restrict__ uf) {
  extern __shared__ double sm[];
  const int Nf = ntf * n1f, Nc = ntc * n1c;
  double* ec = sm;               // [Nc]
  double* Tm = sm + Nc;          // [ntf][n1c]
  const int e = blockIdx.x;
  for (int i = threadIdx.x; i < Nc; i += blockDim.x) {
    const int g = connc[(size_t)e * Nc + i];
    ec[i] = (g >= 0) ? uc[g] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ntf * n1c; i += blockDim.x) {
    const int mf = i / n1c, lc = i % n1c;
    double s = 0.0;
    for (int mc = 0; mc < ntc; ++mc) s = fma(Itri[mf * ntc + mc], ec[mc + ntc * lc], s);
    Tm[i] = s;
  }
  __syncthreads();
  for (int n = threadIdx.x; n < Nf; n += blockDim.x) {
    if (!owner[(size_t)e * Nf + n]) continue;
    const int g = connf[(size_t)e * Nf + n];
    if (g < 0) continue;
    const int mf = n % ntf, lf = n / ntf;
    double s = 0.0;
    for (int lc = 0; lc < n1c; ++lc) s = fma(I1[lf * n1c + lc], Tm[mf * n1c + lc], s);
    uf[g] += s;
  }
}

__global__ void k_restrict(int E, int ntf, int n1f, int ntc, int n1c, const int32_t* __restrict__ connf,
                           const uint8_t* __restrict__ owner, const int32_t* __restrict__ connc,
                           const double* __restrict__ Itri, const double* __restrict__ I1,
                           const double* __restrict__ rf, double* __restrict__ rc, const int32_t* __restrict__ elist) {
  extern __shared__ double sm[];
  const int Nf = ntf * n1f, Nc = ntc * n1c;
  double* xf = sm;               // [Nf]
  double* S = sm + Nf;           // [ntf][n1c]
  const int e = elist ? elist[blockIdx.x] : blockIdx.x;
  for (int n = threadIdx.x; n < Nf; n += blockDim.x) {
    const int g = connf[(size_t)e * Nf + n];
    xf[n] = (owner[(size_t)e * Nf + n] && g >= 0) ? rf[g] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ntf * n1c; i += blockDim.x) {
    const int mf = i / n1c, lc = i % n1c;
    double s = 0.0;
    for (int lf = 0; lf < n1f; ++lf) s = fma(I1[lf * n1c + lc], xf[mf + ntf * lf], s);
    S[i] = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < Nc; i += blockDim.x) {
    const int g = connc[(size_t)e * Nc + i];
    if (g < 0) continue;
    const int mc = i % ntc, lc = i / ntc;
    double s = 0.0;
    for (int mf = 0; mf < ntf; ++mf) s = fma(Itri[mf * ntc + mc], S[mf * n1c + lc], s);
    atomicAdd(rc + g, s);
  }
}

void launch_prolong(sem_ctx* c, int level, const double* uc, double* uf) {
  const DeviceLevel& F = c->L[level];
  const DeviceLevel& C = c->L[level + 1];
  const int smem = (C.N + F.ref.nt * C.ref.n1) * (int)sizeof(double);
  if (c->E_own == 0) return;
  k_prolong<<<c->E_own, 128, smem, c->stream>>>(c->E_own, F.ref.nt, F.ref.n1, C.ref.nt, C.ref.n1, F.conn, F.owner, C.conn,
                                            F.Itri, F.I1, uc, uf);
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
}

void launch_restrict(sem_ctx* c, int level, const double* rf, double* rc) {
  const DeviceLevel& F = c->L[level];
  const DeviceLevel& C = c->L[level + 1];
  CUDA_CHECK(cudaMemsetAsync(rc, 0, sizeof(double) * C.n, c->stream));
  const int smem = (F.N + F.ref.nt * C.ref.n1) * (int)sizeof(double);
  if (c->E_own == 0) return;
  if (c->det.on) {  // deterministic: element colours
    for (size_t k = 0; k + 1 < c->det.ecol_off.size(); ++k) {
      const int cnt = (int)(c->det.ecol_off[k + 1] - c->det.ecol_off[k]);
      k_restrict<<<cnt, 128, smem, c->stream>>>(cnt, F.ref.nt, F.ref.n1, C.ref.nt, C.ref.n1, F.conn, F.owner, C.conn,
                                                F.Itri, F.I1, rf, rc, c->det.ecol + c->det.ecol_off[k]);
    }
  } else {
    k_restrict<<<c->E_own, 128, smem, c->stream>>>(c->E_own, F.ref.nt, F.ref.n1, C.ref.nt, C.ref.n1, F.conn, F.owner,
                                                   C.conn, F.Itri, F.I1, rf, rc, nullptr);
  }
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
}

// ============================================================== coarse solve
__global__ void k_gather(int64_t n, const int32_t* __restrict__ idx, const double* __restrict__ src,
                         double* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

// ---- packed symmetric coarse inverse: lower-triangular 64x64 tiles, tile rows I = 0..T-1
// each holding tiles J = 0..I (zero beyond n_c); tile t = I (I + 1) / 2 + J starts at t * 4096.
// Inside a tile, lane l = 4 a + b of a warp owns the 8 x 16 sub-block rows 8a.., columns 16b..;
// its k-th value (row 8a + k/16, column 16b + k%16) is stored at k * 32 + l, so every load
// instruction of the GEMV reads 256 contiguous bytes.  z = A x reads each stored entry once
// (half of the dense inverse; FP64, or FP32 storage with FP64 arithmetic under
// opts.mixed_precision, reading O36): warps stream contiguous tile ranges, row partials stay in
// registers along a tile row, column partials of off-diagonal tiles (the symmetric half) are
// reduce-scattered over the 8 row-lanes and added atomically.
__device__ __forceinline__ void tile_of(int64_t t, int64_t& I, int64_t& J) {
  I = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((I + 1) * (I + 2) / 2 <= t) ++I;
  while (I * (I + 1) / 2 > t) --I;
  J = t - I * (I + 1) / 2;
}

template <class TA>
__global__ void k_coarse_pack(int64_t n, int T, const double* __restrict__ A, TA* __restrict__ P) {
  const int64_t ntile = (int64_t)T * (T + 1) / 2;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < ntile * 4096;
       x += (int64_t)gridDim.x * blockDim.x) {
    int64_t I, J;
    tile_of(x >> 12, I, J);
    // FP64: value k of lane l at k * 32 + l; FP32: pairs (k, k + 1) at (k / 2) * 64 + 2 l + k % 2 (8-byte loads)
    const int w = (int)(x & 4095);
    const int k = sizeof(TA) == 8 ? w >> 5 : 2 * (w >> 6) + (w & 1), l = sizeof(TA) == 8 ? w & 31 : (w >> 1) & 31;
    const int64_t gi = 64 * I + 8 * (l >> 2) + (k >> 4), gj = 64 * J + 16 * (l & 3) + (k & 15);
    P[x] = (TA)((gi < n && gj < n) ? A[gi * n + gj] : 0.0);
  }
}

__device__ __forceinline__ void symv_flush_rows(double (&acc)[8], int64_t I, int lane, int64_t n,
                                                const int32_t* __restrict__ fidx, double* __restrict__ z) {
  // reduce-scatter the 8 row partials over the 4 column-lanes (lane bits 0, 1)
  const bool b1 = lane & 2, b0 = lane & 1;
  double v4[4], v2[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double snd = b1 ? acc[i] : acc[i + 4];
    v4[i] = (b1 ? acc[i + 4] : acc[i]) + __shfl_xor_sync(0xffffffffu, snd, 2);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double snd = b0 ? v4[i] : v4[i + 2];
    v2[i] = (b0 ? v4[i + 2] : v4[i]) + __shfl_xor_sync(0xffffffffu, snd, 1);
  }
  const int64_t r0 = 64 * I + 8 * (lane >> 2) + 4 * (b1 ? 1 : 0) + 2 * (b0 ? 1 : 0);
#pragma unroll
  for (int i = 0; i < 2; ++i)
    if (r0 + i < n) atomicAdd(z + fidx[r0 + i], v2[i]);
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0;
}

template <class TA>
__global__ void __launch_bounds__(256, 3) k_coarse_symv(int64_t n, int T, const TA* __restrict__ P,
                                                     const double* __restrict__ x, const int32_t* __restrict__ fidx,
                                                     double* __restrict__ z) {
  const int lane = threadIdx.x & 31, a = lane >> 2, b = lane & 3;
  const int64_t nwarp = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t ntile = (int64_t)T * (T + 1) / 2;
  const int64_t t0 = wid * ntile / nwarp, t1 = (wid + 1) * ntile / nwarp;
  if (t0 >= t1) return;
  int64_t I, J;
  tile_of(t0, I, J);
  double acc[8], xi[8];
  auto load_xi = [&]() {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t g = 64 * I + 8 * a + i;
      xi[i] = g < n ? x[g] : 0.0;
    }
  };
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0;
  load_xi();
  for (int64_t t = t0; t < t1; ++t) {
    const TA* tile = P + t * 4096 + lane;
    double xj[16], col[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int64_t g = 64 * J + 16 * b + j;
      xj[j] = g < n ? x[g] : 0.0;
      col[j] = 0.0;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {  // row 8a + c
      double v[16];
      if constexpr (sizeof(TA) == 8) {
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = (double)__ldcs(tile + (16 * c + k) * 32);
      } else {
        const float2* t2 = reinterpret_cast<const float2*>(tile - lane) + lane;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float2 f = __ldcs(t2 + (8 * c + k) * 32);
          v[2 * k] = f.x;
          v[2 * k + 1] = f.y;
        }
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int rr = c, cc = k;
        acc[rr] = fma(v[k], xj[cc], acc[rr]);
        col[cc] = fma(v[k], xi[rr], col[cc]);
      }
    }
    if (J != I) {  // z_J += A_IJ^T x_I: reduce-scatter the 16 column partials over lane bits 4, 3, 2
      const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
      double v8[8], v4[4], v2[2];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double snd = b4 ? col[i] : col[i + 8];
        v8[i] = (b4 ? col[i + 8] : col[i]) + __shfl_xor_sync(0xffffffffu, snd, 16);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double snd = b3 ? v8[i] : v8[i + 4];
        v4[i] = (b3 ? v8[i + 4] : v8[i]) + __shfl_xor_sync(0xffffffffu, snd, 8);
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double snd = b2 ? v4[i] : v4[i + 2];
        v2[i] = (b2 ? v4[i + 2] : v4[i]) + __shfl_xor_sync(0xffffffffu, snd, 4);
      }
      const int64_t c0 = 64 * J + 16 * b + 8 * (b4 ? 1 : 0) + 4 * (b3 ? 1 : 0) + 2 * (b2 ? 1 : 0);
#pragma unroll
      for (int i = 0; i < 2; ++i)
        if (c0 + i < n) atomicAdd(z + fidx[c0 + i], v2[i]);
    }
    if (++J > I || t + 1 == t1) {  // tile row done (or range end): z_I += its row partials
      symv_flush_rows(acc, I, lane, n, fidx, z);
      if (J > I) {
        ++I;
        J = 0;
        load_xi();
      }
    }
  }
}

__device__ __forceinline__ double warp_sum(double v);

// deterministic mode: z[fidx[i]] = sum_j A[i][j] x[j] over the full symmetric inverse, one warp
// per row, each lane summing a fixed column stride, a fixed shuffle tree (no atomics)
__global__ void k_coarse_gemv_det(int64_t n, const double* __restrict__ A, const double* __restrict__ x,
                                  const int32_t* __restrict__ fidx, double* __restrict__ z) {
  const int lane = threadIdx.x & 31;
  const int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n) return;
  const double* a = A + i * n;
  double s = 0.0;
  for (int64_t j = lane; j < n; j += 32) s = fma(a[j], x[j], s);
  s = warp_sum(s);
  if (lane == 0) z[fidx[i]] = s;
}

void launch_coarse(sem_ctx* c, const double* r, double* z) {
  const DeviceLevel& L = c->L.back();
  if (c->C.Afull) {
    CUDA_CHECK(cudaMemsetAsync(z, 0, sizeof(double) * L.n, c->stream));
    k_gather<<<grid_for(c->C.nc, 256), 256, 0, c->stream>>>(c->C.nc, c->C.fidx, r, c->C.x);
    k_coarse_gemv_det<<<(int)((c->C.nc + 7) / 8), 256, 0, c->stream>>>(c->C.nc, c->C.Afull, c->C.x, c->C.fidx, z);
    CUDA_CHECK(cudaGetLastError());
    c->launches += 2;
    return;
  }
  if (c->C.Apack || c->C.Apack32) {
    CUDA_CHECK(cudaMemsetAsync(z, 0, sizeof(double) * L.n, c->stream));
    k_gather<<<grid_for(c->C.nc, 256), 256, 0, c->stream>>>(c->C.nc, c->C.fidx, r, c->C.x);
    CUDA_CHECK(cudaGetLastError());
    const int T = (int)((c->C.nc + 63) / 64);
    const int64_t ntile = (int64_t)T * (T + 1) / 2;
    const int grid = (int)std::min<int64_t>(148 * 3, (ntile + 7) / 8);  // 3 resident CTAs per SM
    if (c->C.Apack)
      k_coarse_symv<double><<<grid, 256, 0, c->stream>>>(c->C.nc, T, c->C.Apack, c->C.x, c->C.fidx, z);
    else
      k_coarse_symv<float><<<grid, 256, 0, c->stream>>>(c->C.nc, T, c->C.Apack32, c->C.x, c->C.fidx, z);
    CUDA_CHECK(cudaGetLastError());
    c->launches += 2;
    return;
  }
  throw SemError(SEM_EINVAL, "exact coarse solve without a stored inverse");
}

// ============================================================== vector kernels
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block sums of (a, b): atomically added to out0 / out1, or (deterministic mode, part != NULL)
// written to part[2 blockIdx.x + {0, 1}] and summed in a fixed order by k_det_finalize.
__device__ __forceinline__ void block_sum2_atomic(double a, double b, double* out0, double* out1,
                                                  double* part = nullptr) {
  __shared__ double s0[32], s1[32];
  a = warp_sum(a);
  b = warp_sum(b);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { s0[w] = a; s1[w] = b; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    a = lane < nw ? s0[lane] : 0.0;
    b = lane < nw ? s1[lane] : 0.0;
    a = warp_sum(a);
    b = warp_sum(b);
    if (lane == 0) {
      if (part) {
        part[2 * blockIdx.x] = a;
        part[2 * blockIdx.x + 1] = b;
      } else {
        atomicAdd(out0, a);
        if (out1) atomicAdd(out1, b);
      }
    }
  }
}

// out0 += sum_b part[2b], out1 += sum_b part[2b+1] in a fixed order (one warp)
__global__ void k_det_finalize(int nb, const double* __restrict__ part, double* out0, double* out1) {
  const int lane = threadIdx.x;
  double a = 0.0, b = 0.0;
  for (int i = lane; i < nb; i += 32) {
    a += part[2 * i];
    b += part[2 * i + 1];
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if (lane == 0) {
    *out0 += a;
    if (out1) *out1 += b;
  }
}

void det_finalize(sem_ctx* c, int nb, double* out0, double* out1) {
  k_det_finalize<<<1, 32, 0, c->stream>>>(nb, c->det.part, out0, out1);
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
}

// out2[0] += a.b ; out2[1] += d.e (if d); over mask[i] != 0 only (if mask)
__global__ void k_dot2(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                       const double* __restrict__ d, const double* __restrict__ e, const uint8_t* __restrict__ mask,
                       double* out2, double* part) {
  double s0 = 0.0, s1 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (mask && !mask[i]) continue;
    s0 = fma(a[i], b[i], s0);
    if (d) s1 = fma(d[i], e[i], s1);
  }
  block_sum2_atomic(s0, s1, out2, d ? out2 + 1 : nullptr, part);
}

void launch_dot2(sem_ctx* c, int64_t n, const double* a, const double* b, const double* d, const double* e,
                 const uint8_t* mask, double* out2, bool clear) {
  if (clear) CUDA_CHECK(cudaMemsetAsync(out2, 0, sizeof(double) * (d ? 2 : 1), c->stream));
  const int gb = grid_for(n, 256);
  k_dot2<<<gb, 256, 0, c->stream>>>(n, a, b, d, e, mask, out2, c->det.part);
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
  if (c->det.part) det_finalize(c, gb, out2, d ? out2 + 1 : nullptr);
}

// alpha = num / den; u += alpha p; r -= alpha q; rr += r.r
__global__ void k_axpy_pcg(int64_t n, double* __restrict__ u, double* __restrict__ r, const double* __restrict__ p,
                           const double* __restrict__ q, const double* num, const double* den, double* rr,
                           const uint8_t* __restrict__ mask, double* part) {
  const double alpha = *num / *den;
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    u[i] = fma(alpha, p[i], u[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    if (!mask || mask[i]) s = fma(ri, ri, s);
  }
  block_sum2_atomic(s, 0.0, rr, nullptr, part);
}

void launch_axpy_pcg(sem_ctx* c, int64_t n, double* u, double* r, const double* p, const double* q,
                     const double* num, const double* den, double* rr, const uint8_t* mask, bool clear) {
  if (clear) CUDA_CHECK(cudaMemsetAsync(rr, 0, sizeof(double), c->stream));
  const int gb = grid_for(n, 256);
  k_axpy_pcg<<<gb, 256, 0, c->stream>>>(n, u, r, p, q, num, den, rr, mask, c->det.part);
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
  if (c->det.part) det_finalize(c, gb, rr, nullptr);
}

// p = z + beta p: beta = num[0] / den (mode 0); p = z (mode 1);
// beta = (num[0] - num[1]) / den (mode 2, flexible CG: z^T (r - r_old) / delta)
__global__ void k_xpby(int64_t n, double* __restrict__ p, const double* __restrict__ z, const double* num,
                       const double* den, int mode) {
  const double beta = mode == 1 ? 0.0 : (mode == 2 ? (num[0] - num[1]) / *den : num[0] / *den);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = mode == 1 ? z[i] : fma(beta, p[i], z[i]);
}

void launch_xpby(sem_ctx* c, int64_t n, double* p, const double* z, const double* num, const double* den,
                 int mode) {
  k_xpby<<<grid_for(n, 256), 256, 0, c->stream>>>(n, p, z, num, den, mode);
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
}

__global__ void k_axpy(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}

void launch_axpy(sem_ctx* c, int64_t n, double a, const double* x, double* y) {
  k_axpy<<<grid_for(n, 256), 256, 0, c->stream>>>(n, a, x, y);
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
}

// z = dinv .* r; out2[0] += z.r; out2[1] += r.r
__global__ void k_jacobi_dot(int64_t n, const double* __restrict__ d, const double* __restrict__ r,
                             double* __restrict__ z, double* out2, double* part) {
  double s0 = 0.0, s1 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = r[i], zi = d[i] * ri;
    z[i] = zi;
    s0 = fma(zi, ri, s0);
    s1 = fma(ri, ri, s1);
  }
  block_sum2_atomic(s0, s1, out2, out2 + 1, part);
}

void launch_jacobi_dot(sem_ctx* c, int64_t n, const double* dinv, const double* r, double* z, double* out2) {
  CUDA_CHECK(cudaMemsetAsync(out2, 0, 2 * sizeof(double), c->stream));
  const int gb = grid_for(n, 256);
  k_jacobi_dot<<<gb, 256, 0, c->stream>>>(n, dinv, r, z, out2, c->det.part);
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
  if (c->det.part) det_finalize(c, gb, out2, out2 + 1);
}

// diag[g] += Ae[e][n][n] over free nodes (setup)
__global__ void k_diag_accum(int64_t E, int N, const int32_t* __restrict__ conn, const double* __restrict__ Ae,
                             double* __restrict__ diag) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= E * N) return;
  const int64_t e = idx / N;
  const int n = (int)(idx % N);
  const int c = conn[idx];
  if (c >= 0) atomicAdd(diag + c, Ae[(e * N + n) * N + n]);
}

void launch_diag_accum_range(sem_ctx* c, const int32_t* conn, int N, int ne, const double* Ae, double* diag) {
  const int64_t tot = (int64_t)ne * N;
  k_diag_accum<<<(int)((tot + 255) / 256), 256, 0, c->stream>>>(ne, N, conn, Ae, diag);
  CUDA_CHECK(cudaGetLastError());
}

__global__ void k_invert_masked(int64_t n, const uint8_t* __restrict__ dmask, double* d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = (dmask[i] || d[i] == 0.0) ? 0.0 : 1.0 / d[i];
}

void launch_invert_masked(sem_ctx* c, int level, double* d) {
  const DeviceLevel& L = c->L[level];
  k_invert_masked<<<grid_for(L.n, 256), 256, 0, c->stream>>>(L.n, L.dmask, d);
  CUDA_CHECK(cudaGetLastError());
}

// phi = free ? uF : phiD
__global__ void k_combine(int64_t n, const uint8_t* __restrict__ dmask, const double* __restrict__ uF,
                          const double* __restrict__ phiD, double* __restrict__ phi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    phi[i] = dmask[i] ? phiD[i] : uF[i];
}

void launch_combine_phi(sem_ctx* c, int level, const double* uF, const double* phiD, double* phi) {
  const DeviceLevel& L = c->L[level];
  k_combine<<<grid_for(L.n, 256), 256, 0, c->stream>>>(L.n, L.dmask, uF, phiD, phi);
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
}

// ============================================================== setup kernels
// G = w detJ J^-1 J^-T from the finest nodal map (O-5, O7); J[i][c] = dx_i/dxi_c.
__global__ void k_geometry(int E, int Nf, int Q, const double* __restrict__ X, const double* __restrict__ gm,
                           const double* __restrict__ w, double* __restrict__ G, int* bad) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)E * Q) return;
  const int64_t e = idx / Q;
  const int q = (int)(idx % Q);
  double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  const double* Xe = X + e * Nf * 3;
  for (int n = 0; n < Nf; ++n) {
    const double dr = gm[((int64_t)n * 3 + 0) * Q + q];
    const double ds = gm[((int64_t)n * 3 + 1) * Q + q];
    const double dt = gm[((int64_t)n * 3 + 2) * Q + q];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double xi = Xe[n * 3 + i];
      J[i][0] = fma(xi, dr, J[i][0]);
      J[i][1] = fma(xi, ds, J[i][1]);
      J[i][2] = fma(xi, dt, J[i][2]);
    }
  }
  const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                     J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                     J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
  if (!(det > 0.0)) atomicExch(bad, 1);
  double Ji[3][3];
  const double id = 1.0 / det;
  Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) * id;
  Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
  Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
  Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) * id;
  Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
  Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
  Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) * id;
  Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
  Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
  const double s = w[q] * det;
  double g[6];
  int k = 0;
  for (int a = 0; a < 3; ++a)
    for (int b = a; b < 3; ++b) {
      g[k++] = s * (Ji[a][0] * Ji[b][0] + Ji[a][1] * Ji[b][1] + Ji[a][2] * Ji[b][2]);
    }
  for (int c2 = 0; c2 < 6; ++c2) G[(e * 6 + c2) * Q + q] = g[c2];
}

int launch_geometry(sem_ctx* c, int level, const double* X, const double* gm, int Nf, const double* w) {
  DeviceLevel& L = c->L[level];
  int* bad;
  CUDA_CHECK(cudaMalloc(&bad, sizeof(int)));
  CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
  const int64_t tot = (int64_t)c->E * L.Q;
  k_geometry<<<(int)((tot + 127) / 128), 128, 0, c->stream>>>(c->E, Nf, L.Q, X, gm, w, L.G, bad);
  CUDA_CHECK(cudaGetLastError());
  int hb = 0;
  CUDA_CHECK(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
  CUDA_CHECK(cudaFree(bad));
  return hb;
}

// Ae[e][i][j] = sum_q sum_cd D_c[q][i] G_cd[e][q] D_d[q][j]   (setup only)
__global__ void k_elem_matrices(int e0, int ne, int N, int Q, const double* __restrict__ D,
                                const double* __restrict__ G, double* __restrict__ Ae,
                                const int32_t* __restrict__ elist) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t NN = (int64_t)N * N;
  if (idx >= (int64_t)ne * NN) return;
  const int64_t le = idx / NN;
  const int i = (int)((idx % NN) / N), j = (int)(idx % N);
  const int64_t e = elist ? (int64_t)elist[le] : e0 + le;
  const double* g = G + e * 6 * Q;
  double s = 0.0;
  for (int q = 0; q < Q; ++q) {
    const double ri = D[(0 * Q + q) * N + i], si = D[(1 * Q + q) * N + i], ti = D[(2 * Q + q) * N + i];
    const double rj = D[(0 * Q + q) * N + j], sj = D[(1 * Q + q) * N + j], tj = D[(2 * Q + q) * N + j];
    const double gxx = g[0 * Q + q], gxy = g[1 * Q + q], gxz = g[2 * Q + q];
    const double gyy = g[3 * Q + q], gyz = g[4 * Q + q], gzz = g[5 * Q + q];
    s += ri * (gxx * rj + gxy * sj + gxz * tj) + si * (gxy * rj + gyy * sj + gyz * tj) +
         ti * (gxz * rj + gyz * sj + gzz * tj);
  }
  Ae[idx] = s;
}

void launch_elem_matrices(sem_ctx* c, int level, const double* D, double* Ae, int e0, int ne) {
  const DeviceLevel& L = c->L[level];
  const int64_t tot = (int64_t)ne * L.N * L.N;
  k_elem_matrices<<<(int)((tot + 255) / 256), 256, 0, c->stream>>>(e0, ne, L.N, L.Q, D, L.G, Ae, nullptr);
  CUDA_CHECK(cudaGetLastError());
}

void launch_elem_matrices_list(sem_ctx* c, int level, const double* D, double* Ae, const int32_t* elist, int ne) {
  const DeviceLevel& L = c->L[level];
  const int64_t tot = (int64_t)ne * L.N * L.N;
  k_elem_matrices<<<(int)((tot + 255) / 256), 256, 0, c->stream>>>(0, ne, L.N, L.Q, D, L.G, Ae, elist);
  CUDA_CHECK(cudaGetLastError());
}

// B_k = R_k A R_k^T from element matrices (principal submatrix of the assembled,
// Dirichlet-eliminated A on subdomain k); padded to npad with the identity.
__global__ void k_assemble_blocks(int N, const int32_t* __restrict__ conn, const int32_t* __restrict__ idx,
                                  const int64_t* __restrict__ off, const int32_t* __restrict__ elist,
                                  const int64_t* __restrict__ eoff, const double* __restrict__ Ae, int ebase,
                                  int k0, int npad, double* __restrict__ B, const int32_t* __restrict__ eslot) {
  extern __shared__ int ism[];
  int* sidx = ism;              // [npad]
  int* pos = ism + npad;        // [N]
  int* loc = pos + N;           // [N]
  __shared__ int nloc;
  const int k = k0 + blockIdx.x;
  const int64_t o = off[k];
  const int nk = (int)(off[k + 1] - o);
  for (int i = threadIdx.x; i < nk; i += blockDim.x) sidx[i] = idx[o + i];
  double* Bk = B + (size_t)blockIdx.x * npad * npad;
  for (int i = nk + threadIdx.x; i < npad; i += blockDim.x) Bk[(size_t)i * npad + i] = 1.0;
  __syncthreads();
  for (int64_t t = eoff[k]; t < eoff[k + 1]; ++t) {
    const int e = elist[t];
    if (threadIdx.x == 0) nloc = 0;
    __syncthreads();
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      const int c = conn[(size_t)e * N + n];
      int p = -1;
      if (c >= 0) {
        int lo = 0, hi = nk - 1;
        while (lo <= hi) {
          const int mid = (lo + hi) >> 1;
          const int v = sidx[mid];
          if (v == c) { p = mid; break; }
          if (v < c) lo = mid + 1; else hi = mid - 1;
        }
      }
      pos[n] = p;
      if (p >= 0) loc[atomicAdd(&nloc, 1)] = n;
    }
    __syncthreads();
    const int nl = nloc;
    const double* A = Ae + (size_t)(eslot ? eslot[t - eoff[k0]] : e - ebase) * N * N;
    for (int pr = threadIdx.x; pr < nl * nl; pr += blockDim.x) {
      const int i = loc[pr / nl], j = loc[pr % nl];
      Bk[(size_t)pos[i] * npad + pos[j]] += A[(size_t)i * N + j];
    }
    __syncthreads();
  }
}

void launch_assemble_blocks(sem_ctx* c, int level, const int32_t* idx, const int64_t* off, const int32_t* elist,
                            const int64_t* eoff, const double* Ae, int ebase, int k0, int nb, int npad, double* B,
                            const int32_t* eslot) {
  const DeviceLevel& L = c->L[level];
  const int smem = (npad + 2 * L.N) * (int)sizeof(int);
  k_assemble_blocks<<<nb, 256, smem, c->stream>>>(L.N, L.conn, idx, off, elist, eoff, Ae, ebase, k0, npad, B, eslot);
  CUDA_CHECK(cudaGetLastError());
}

// copy the lower 16x16 tiles of each inverse (full npad x npad, symmetric) into
// the streaming layout; entries beyond n_k are zeroed.
template <class TT>
__global__ void k_pack_tiles(const double* __restrict__ Binv, int k0, int npad, const int64_t* __restrict__ off,
                             const int64_t* __restrict__ tile_off, TT* __restrict__ tiles) {
  const int k = k0 + blockIdx.x;
  const int nk = (int)(off[k + 1] - off[k]);
  const int T = (nk + 15) / 16;
  const double* B = Binv + (size_t)blockIdx.x * npad * npad;
  TT* out = tiles + tile_off[k];
  const int ntiles = T * (T + 1) / 2;
  for (int64_t x = threadIdx.x; x < (int64_t)ntiles * 256; x += blockDim.x) {
    const int t = (int)(x / 256), rc = (int)(x % 256), r = rc / 16, cc = rc % 16;
    int I = 0;
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    const int J = t - I * (I + 1) / 2;
    const int gi = 16 * I + r, gj = 16 * J + cc;
    // entry (r, c) is value m = r / 2 of lane (r % 2) * 16 + c; every warp-wide load instruction
    // reads 256 contiguous bytes: FP64 m * 32 + lane, FP32 pairs (m / 2) * 64 + 2 lane + m % 2
    const int ln = (r & 1) * 16 + cc, mm = r >> 1;
    const int64_t dst = (int64_t)t * 256 + (sizeof(TT) == 8 ? mm * 32 + ln : (mm >> 1) * 64 + 2 * ln + (mm & 1));
    out[dst] = (TT)((gi < nk && gj < nk) ? B[(size_t)gi * npad + gj] : 0.0);
  }
}

void launch_pack_tiles(sem_ctx* c, int level, const double* Binv, int k0, int nb, int npad, const int64_t* off) {
  const DeviceLevel& L = c->L[level];
  if (L.tiles32) k_pack_tiles<float><<<nb, 256, 0, c->stream>>>(Binv, k0, npad, off, L.tile_off, L.tiles32);
  else k_pack_tiles<double><<<nb, 256, 0, c->stream>>>(Binv, k0, npad, off, L.tile_off, L.tiles);
  CUDA_CHECK(cudaGetLastError());
}

__global__ void k_to_float(int64_t n, const double* __restrict__ a, float* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (float)a[i];
}

void launch_coarse_pack(sem_ctx* c, int64_t n, const double* A, double* P, float* P32) {
  const int T = (int)((n + 63) / 64);
  if (P) k_coarse_pack<double><<<148 * 32, 256, 0, c->stream>>>(n, T, A, P);
  else k_coarse_pack<float><<<148 * 32, 256, 0, c->stream>>>(n, T, A, P32);
  CUDA_CHECK(cudaGetLastError());
}

void launch_to_float(sem_ctx* c, int64_t n, const double* a, float* b) {
  k_to_float<<<grid_for(n, 256), 256, 0, c->stream>>>(n, a, b);
  CUDA_CHECK(cudaGetLastError());
}

__global__ void k_set_identity(double* X, int nb, int npad) {
  const int64_t tot = (int64_t)nb * npad * npad;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = i % ((int64_t)npad * npad);
    X[i] = (w / npad == w % npad) ? 1.0 : 0.0;
  }
}

void launch_set_identity(sem_ctx* c, double* X, int nb, int npad) {
  k_set_identity<<<148 * 16, 256, 0, c->stream>>>(X, nb, npad);
  CUDA_CHECK(cudaGetLastError());
}

// dense free-free coarse matrix from P=1 element matrices
__global__ void k_assemble_coarse(int E, int N, const int32_t* __restrict__ conn, const int32_t* __restrict__ cmap,
                                  const double* __restrict__ Ae, double* __restrict__ A, int64_t nc) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t NN = (int64_t)N * N;
  if (idx >= (int64_t)E * NN) return;
  const int64_t e = idx / NN;
  const int i = (int)((idx % NN) / N), j = (int)(idx % N);
  const int ci = conn[e * N + i], cj = conn[e * N + j];
  if (ci < 0 || cj < 0) return;
  atomicAdd(A + (int64_t)cmap[ci] * nc + cmap[cj], Ae[idx]);
}

void launch_assemble_coarse(sem_ctx* c, const double* Ae, const int32_t* cmap, double* A, int64_t nc) {
  const DeviceLevel& L = c->L.back();
  const int64_t tot = (int64_t)c->E * L.N * L.N;
  k_assemble_coarse<<<(int)((tot + 255) / 256), 256, 0, c->stream>>>(c->E, L.N, L.conn, cmap, Ae, A, nc);
  CUDA_CHECK(cudaGetLastError());
}

// copy the lower triangle (column-major potri output) to the upper one
__global__ void k_symmetrize(double* A, int64_t n) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n * n) return;
  const int64_t i = idx / n, j = idx % n;  // row-major (i, j) = column-major (j, i)
  // potri (column-major, lower) wrote the row-major upper triangle; mirror it
  if (i > j) A[idx] = A[j * n + i];
}

void launch_symmetrize(sem_ctx* c, double* A, int64_t n) {
  k_symmetrize<<<(int)((n * n + 255) / 256), 256, 0, c->stream>>>(A, n);
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace sem
