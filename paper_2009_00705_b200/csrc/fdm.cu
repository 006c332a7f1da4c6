// FDM local solves of the Schwarz smoother on the GPU (reading O33; fdm.h).
//
// Setup: per column the generalised eigenproblem K_h S_h = M_h S_h L_h of its
// horizontal patch, per element K_v S_v = M_v S_v L_v of its vertical box
// (S^T M S = I), batched on the GPU: Cholesky M = L L^T (cuSOLVER
// potrfBatched), C = L^-1 K L^-T (cuBLAS trsmBatched), C = Q L Q^T (cuSOLVER
// XsyevBatched), S = L^-T Q.
//
// Apply (one sweep of eq 4.4 with the FDM local inverses):
//   x = R_k r (x W for S^-T) ;  x <- (S_h (x) S_v)^T x ;  x /= (l_h,a + l_v,b) ;
//   x <- (S_h (x) S_v) x ;  u += R_k^T x (x W for S^-1).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "fdm.h"
#include "internal.h"
#include "setup_util.h"

namespace sem {

#define CUBLAS_OK(x)                                                                     \
  do {                                                                                   \
    cublasStatus_t _s = (x);                                                             \
    if (_s != CUBLAS_STATUS_SUCCESS) throw SemError(SEM_ECUDA, std::string(#x) + " failed"); \
  } while (0)
#define CUSOLVER_OK(x)                                                                   \
  do {                                                                                   \
    cusolverStatus_t _s = (x);                                                           \
    if (_s != CUSOLVER_STATUS_SUCCESS)                                                   \
      throw SemError(SEM_ECUDA, std::string(#x) + " failed (status " + std::to_string((int)_s) + ")"); \
  } while (0)

__global__ void k_unpack_pairs(int n, const int64_t* __restrict__ off, const double* __restrict__ K,
                               const double* __restrict__ M, double* __restrict__ Kp, double* __restrict__ Mp) {
  const int b = blockIdx.x;
  const double* k = K + off[b];
  const double* m = M + off[b];
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) {  // symmetric: row-major = column-major
    Kp[(size_t)b * n * n + t] = k[t];
    Mp[(size_t)b * n * n + t] = m[t];
  }
}

// S (column-major [n][n], eigenvectors in columns) -> packed row-major S[i][a] (i node, a mode)
__global__ void k_pack_modes(int n, const int64_t* __restrict__ off, const int64_t* __restrict__ loff,
                             const double* __restrict__ Sp, const double* __restrict__ Wp, double* __restrict__ S,
                             double* __restrict__ lam) {
  const int b = blockIdx.x;
  const double* sp = Sp + (size_t)b * n * n;
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
    const int i = t / n, a = t % n;
    S[off[b] + t] = sp[i + (size_t)n * a];
  }
  for (int a = threadIdx.x; a < n; a += blockDim.x) lam[loff[b] + a] = Wp[(size_t)b * n + a];
}

// Generalised symmetric-definite eigenproblems K S = M S L for packed problems
// (sizes n[b], row-major blocks at off[b]); S packed the same way (device dS),
// eigenvalues at loff[b] (device dlam).  Problems are batched by size (no
// padding, so the eigensolver's backward error stays relative to each problem).
static void batched_geneig(sem_ctx* c, cusolverDnHandle_t sol, cublasHandle_t blas, const std::vector<int32_t>& n,
                           const std::vector<int64_t>& off, const std::vector<double>& K, const std::vector<double>& M,
                           const std::vector<int64_t>& loff, double* dS, double* dlam) {
  const int nb_all = (int)n.size();
  if (nb_all == 0) return;
  Scratch s0;
  double* dK = s0.put(K);
  double* dM = s0.put(M);
  std::vector<std::vector<int>> bysize(*std::max_element(n.begin(), n.end()) + 1);
  for (int b = 0; b < nb_all; ++b) bysize[n[b]].push_back(b);
  cusolverDnParams_t params;
  CUSOLVER_OK(cusolverDnCreateParams(&params));
  struct PG {
    cusolverDnParams_t p;
    ~PG() { cusolverDnDestroyParams(p); }
  } pg{params};
  const double one = 1.0;
  for (int np = 1; np < (int)bysize.size(); ++np) {
    const std::vector<int>& list = bysize[np];
    if (list.empty()) continue;
    size_t freeb = 0, totb = 0;
    CUDA_CHECK(cudaMemGetInfo(&freeb, &totb));
    const size_t per = (size_t)np * np * 8 * 2 + (size_t)np * 8 + 64;
    const int chunk = (int)std::max<size_t>(1, std::min<size_t>(std::min<size_t>((size_t)(freeb * 0.3) / per, 16384),
                                                                list.size()));
    Scratch sc;
    double* Kp = sc.get<double>((size_t)chunk * np * np);
    double* Mp = sc.get<double>((size_t)chunk * np * np);
    double* Wp = sc.get<double>((size_t)chunk * np);
    double** pK = sc.get<double*>(chunk);
    double** pM = sc.get<double*>(chunk);
    int* info = sc.get<int>(chunk);
    {
      std::vector<double*> hK(chunk), hM(chunk);
      for (int i = 0; i < chunk; ++i) {
        hK[i] = Kp + (size_t)i * np * np;
        hM[i] = Mp + (size_t)i * np * np;
      }
      CUDA_CHECK(cudaMemcpy(pK, hK.data(), chunk * sizeof(double*), cudaMemcpyHostToDevice));
      CUDA_CHECK(cudaMemcpy(pM, hM.data(), chunk * sizeof(double*), cudaMemcpyHostToDevice));
    }
    std::vector<int> hinfo(chunk);
    for (size_t b0 = 0; b0 < list.size(); b0 += chunk) {
      const int nb = (int)std::min<size_t>(chunk, list.size() - b0);
      std::vector<int64_t> o(nb), lo(nb);
      for (int i = 0; i < nb; ++i) {
        o[i] = off[list[b0 + i]];
        lo[i] = loff[list[b0 + i]];
      }
      Scratch s2;
      const int64_t* doff = s2.put(o);
      const int64_t* dloff = s2.put(lo);
      k_unpack_pairs<<<nb, 256, 0, c->stream>>>(np, doff, dK, dM, Kp, Mp);
      CUDA_CHECK(cudaGetLastError());
      CUSOLVER_OK(cusolverDnDpotrfBatched(sol, CUBLAS_FILL_MODE_LOWER, np, pM, np, info, nb));
      CUDA_CHECK(cudaMemcpyAsync(hinfo.data(), info, nb * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      CUDA_CHECK(cudaStreamSynchronize(c->stream));
      for (int i = 0; i < nb; ++i)
        if (hinfo[i] != 0)
          throw SemError(SEM_ESINGULAR, "FDM mass matrix not SPD (potrf info " + std::to_string(hinfo[i]) + ")");
      // C = L^-1 K L^-T
      CUBLAS_OK(cublasDtrsmBatched(blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                                   np, np, &one, (const double* const*)pM, np, pK, np, nb));
      CUBLAS_OK(cublasDtrsmBatched(blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT,
                                   np, np, &one, (const double* const*)pM, np, pK, np, nb));
      // C = Q L Q^T: batched XsyevBatched, or one cusolverDnDsyevd per problem where the
      // batched routine rejects the size (it does for some n)
      size_t wdev = 0, whost = 0;
      const cusolverStatus_t bs = cusolverDnXsyevBatched_bufferSize(
          sol, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, np, CUDA_R_64F, Kp, np, CUDA_R_64F, Wp,
          CUDA_R_64F, &wdev, &whost, nb);
      if (bs == CUSOLVER_STATUS_SUCCESS) {
        void* bdev = s2.get<char>(wdev);
        std::vector<char> bhost(std::max<size_t>(whost, 1));
        CUSOLVER_OK(cusolverDnXsyevBatched(sol, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, np,
                                           CUDA_R_64F, Kp, np, CUDA_R_64F, Wp, CUDA_R_64F, bdev, wdev, bhost.data(),
                                           whost, info, nb));
      } else {
        int lw = 0;
        CUSOLVER_OK(cusolverDnDsyevd_bufferSize(sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, np, Kp, np, Wp,
                                                &lw));
        double* work = s2.get<double>((size_t)std::max(lw, 1));
        for (int i = 0; i < nb; ++i)
          CUSOLVER_OK(cusolverDnDsyevd(sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, np,
                                       Kp + (size_t)i * np * np, np, Wp + (size_t)i * np, work, lw, info + i));
      }
      // S = L^-T Q
      CUBLAS_OK(cublasDtrsmBatched(blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT,
                                   np, np, &one, (const double* const*)pM, np, pK, np, nb));
      k_pack_modes<<<nb, 256, 0, c->stream>>>(np, doff, dloff, Kp, Wp, dS, dlam);
      CUDA_CHECK(cudaGetLastError());
      CUDA_CHECK(cudaStreamSynchronize(c->stream));
    }
  }
}

constexpr int FDM_NT = 8;     // n-tiles (of 8 box columns) per work unit
constexpr int FDM_NC = 8 * FDM_NT;
constexpr int FDM_LDR_MAX = 76;
constexpr int FDM_UD = 34;       // ints per unit descriptor of k_fdm_warp  // column-block row stride bound of the warp kernel (= 4 mod 8)
constexpr int FDM_LD = 72;    // shared-memory row stride in doubles (= 8 mod 16: conflict-free B-fragment reads)

// S_v, l_v of every element zero-padded to [nvp][nvp] / [nvp] (pad eigenvalue 1)
__global__ void k_pad_vertical(int E, int nvp, const int32_t* __restrict__ nv, const int64_t* __restrict__ voff,
                               const int64_t* __restrict__ lvoff, const double* __restrict__ Sv,
                               const double* __restrict__ lv, double* __restrict__ Svp, double* __restrict__ lvp) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int n = nv[e];
  for (int a = 0; a < nvp; ++a) {
    lvp[(size_t)e * nvp + a] = a < n ? lv[lvoff[e] + a] : 1.0;
    for (int b = 0; b < nvp; ++b)
      Svp[((size_t)e * nvp + a) * nvp + b] = (a < n && b < n) ? Sv[voff[e] + a * n + b] : 0.0;
  }
}

void k_pad_vertical_launch(sem_ctx* c, int li) {
  DeviceLevel& L = c->L[li];
  const int E = c->E, nvp = 8 * L.f_nvt;
  k_pad_vertical<<<(E + 127) / 128, 128, 0, c->stream>>>(E, nvp, L.f_nv, L.f_voff, L.f_lvoff, L.f_Sv, L.f_lv, L.f_Svp,
                                                        L.f_lvp);
  CUDA_CHECK(cudaGetLastError());
}

void setup_fdm(sem_ctx* c, int li, const FdmTopo& F, cusolverDnHandle_t sol, cublasHandle_t blas, int verbose) {
  DeviceLevel& L = c->L[li];
  const double t0 = now_ms();
  const int E = (int)F.col.size();
  const int ncol = F.ncol;
  // horizontal (per column) and vertical (per element) eigenpairs
  std::vector<int32_t> nh(ncol), nv(E);
  std::vector<int64_t> lhoff(ncol), lvoff(E);
  for (int q = 0; q < ncol; ++q) {
    nh[q] = (int32_t)(F.hoff[q + 1] - F.hoff[q]);
    lhoff[q] = F.hoff[q];
  }
  int64_t acc = 0;
  for (int e = 0; e < E; ++e) {
    nv[e] = F.nv[e];
    lvoff[e] = acc;
    acc += nv[e];
  }
  L.f_Sh = dalloc<double>(c, F.moff[ncol]);
  L.f_lh = dalloc<double>(c, F.hoff[ncol]);
  L.f_Sv = dalloc<double>(c, F.voff[E]);
  L.f_lv = dalloc<double>(c, acc);
  batched_geneig(c, sol, blas, nh, std::vector<int64_t>(F.moff.begin(), F.moff.end() - 1), F.Kh, F.Mh, lhoff, L.f_Sh,
                 L.f_lh);
  batched_geneig(c, sol, blas, nv, std::vector<int64_t>(F.voff.begin(), F.voff.end() - 1), F.Kv, F.Mv, lvoff, L.f_Sv,
                 L.f_lv);
  L.f_col = upload(c, F.col);
  L.f_cfirst = upload(c, F.cfirst);
  {  // 1D GLL stiffness / mass of the reference layer (per-stage vertical re-formation, stage.cu)
    const LevelRef R = make_level_ref(F.p, F.q > 0 ? F.q : F.p);
    const Rule1D gv = gauss_legendre_rule((F.q > 0 ? F.q : F.p) + 1);
    std::vector<double> km(2 * R.n1 * R.n1, 0.0);
    for (int a = 0; a < R.n1; ++a)
      for (int b = 0; b < R.n1; ++b)
        for (int q = 0; q < R.qv; ++q) {
          km[a * R.n1 + b] += gv.w[q] * R.Dt[q * R.n1 + a] * R.Dt[q * R.n1 + b];
          km[R.n1 * R.n1 + a * R.n1 + b] += gv.w[q] * R.Bt[q * R.n1 + a] * R.Bt[q * R.n1 + b];
        }
    L.f_kmref = upload(c, km);
  }
  L.f_hoff = upload(c, F.hoff);
  L.f_moff = upload(c, F.moff);
  L.f_nv = upload(c, F.nv);
  L.f_voff = upload(c, F.voff);
  L.f_lvoff = upload(c, lvoff);
  L.f_ioff = upload(c, F.ioff);
  L.f_idx = upload(c, F.idx);
  L.W = upload(c, F.W);
  L.f_colel = upload(c, F.colel);
  L.f_nzc = upload(c, F.nzc);
  L.f_cioff = upload(c, F.cioff);
  L.f_cidx = upload(c, F.cidx);
  L.f_z0 = upload(c, F.z0);
  {  // column-batched kernel: every element's box padded to NVT n-tiles of 8 columns,
     // work units = runs of <= FDM_NT / NVT consecutive elements of one column
    const int nvt = (F.nv_max + 7) / 8, nvp = 8 * nvt;
    L.f_nvt = nvt;
    L.f_mt = (F.nh_max + 7) / 8;
    std::vector<int4> units;
    L.f_warp = (L.f_mt <= 8 && nvt <= 2) ? 1 : 0;
    L.f_nph = 2 + (2 * F.overlap) / (F.q > 0 ? F.q : F.p);  // boxes j, j + k overlap iff k q <= q + 2 o
    const int per = L.f_warp ? 8 : FDM_NT / nvt;
    for (int q = 0; q < ncol; ++q)
      for (int64_t j = F.cfirst[q]; j < F.cfirst[q + 1]; j += per)
        units.push_back(make_int4(q, (int)j, (int)std::min<int64_t>(per, F.cfirst[q + 1] - j), 0));
    L.f_units = upload(c, units);
    L.f_nunits = (int)units.size();
    int nzu_max = 1;
    for (const int4& un : units) {
      const int e0 = F.colel[un.y], e1 = F.colel[un.y + un.z - 1];
      nzu_max = std::max(nzu_max, F.z0[e1] + F.nv[e1] - F.z0[e0]);
    }
    L.f_ldr = nzu_max + ((4 - nzu_max % 8) + 8) % 8;  // >= nzu_max, = 4 mod 8
    if (L.f_ldr > FDM_LDR_MAX && L.f_warp) {  // rebuild with the column kernel's units
      L.f_warp = 0;
      units.clear();
      const int per2 = FDM_NT / nvt;
      for (int q = 0; q < ncol; ++q)
        for (int64_t j = F.cfirst[q]; j < F.cfirst[q + 1]; j += per2)
          units.push_back(make_int4(q, (int)j, (int)std::min<int64_t>(per2, F.cfirst[q + 1] - j), 0));
      L.f_units = upload(c, units);
      L.f_nunits = (int)units.size();
    }
    L.f_Svp = dalloc<double>(c, (size_t)E * nvp * nvp);
    L.f_lvp = dalloc<double>(c, (size_t)E * nvp);
    k_pad_vertical<<<(E + 127) / 128, 128, 0, c->stream>>>(E, nvp, L.f_nv, L.f_voff, L.f_lvoff, L.f_Sv, L.f_lv,
                                                          L.f_Svp, L.f_lvp);
    CUDA_CHECK(cudaGetLastError());
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
  }
  {  // unit descriptors of the warp kernel (see k_fdm_warp)
    std::vector<int4> hu(L.f_nunits);
    CUDA_CHECK(cudaMemcpy(hu.data(), L.f_units, hu.size() * sizeof(int4), cudaMemcpyDeviceToHost));
    std::vector<int> ud((size_t)L.f_nunits * FDM_UD, 0);
    for (int i = 0; i < L.f_nunits; ++i) {
      int* d = &ud[(size_t)i * FDM_UD];
      const int q = hu[i].x, first = hu[i].y, cnt = hu[i].z;
      d[0] = q;
      d[1] = cnt;
      d[2] = (int)(F.hoff[q + 1] - F.hoff[q]);
      d[3] = F.nzc[q];
      d[4] = (int)(uint32_t)(F.moff[q] & 0xffffffffu);
      d[5] = (int)(F.moff[q] >> 32);
      d[6] = (int)(uint32_t)(F.cioff[q] & 0xffffffffu);
      d[7] = (int)(F.cioff[q] >> 32);
      d[8] = (int)(uint32_t)(F.hoff[q] & 0xffffffffu);
      d[9] = (int)(F.hoff[q] >> 32);
      for (int j = 0; j < cnt && j < 8; ++j) {
        const int e = F.colel[first + j];
        d[10 + j] = e;
        d[18 + j] = F.z0[e];
        d[26 + j] = F.nv[e];
      }
    }
    L.f_udesc = upload(c, ud);
  }
  L.fdm = 1;
  L.f_nh_max = F.nh_max;
  L.f_nv_max = F.nv_max;
  for (int e = 0; e < E; ++e)
    if (F.regular[e])
      for (int64_t t = F.ioff[e]; t < F.ioff[e + 1]; ++t) L.nk_sum += (F.idx[t] >= 0);
  {
    std::vector<uint8_t> skip(E);
    for (int e = 0; e < E; ++e) skip[e] = F.regular[e] ? 0 : 1;
    L.f_skip = upload(c, skip);
    if (c->opts.deterministic) {  // colours of node-disjoint FDM boxes (one k_fdm launch each)
      std::vector<int32_t> cl;
      colour_sets(E, F.ioff, F.idx, L.n, &skip, L.fcol_off, cl);
      L.fcol = upload(c, cl);
    }
  }
  // algorithmic bytes of one sweep (column-batched kernel): per column S_h, l_h and the patch
  // node ids [n_h][Z_c+1]; per element S_v, l_v
  L.f_bytes = 8 * (F.moff[ncol] + F.hoff[ncol] + F.voff[E] + acc) + 4 * F.cioff[ncol];
  L.schwarz_bytes += L.f_bytes;  // plus the dense part of an O35 hybrid (setup_schwarz ran first)
  if (verbose)
    fprintf(stderr, "[sem] level p=%d FDM: %d columns, n_h max %d, n_v max %d, %.1f MiB, %.0f ms\n", L.p, ncol,
            F.nh_max, F.nv_max, L.f_bytes / 1048576.0, now_ms() - t0);
}

// ---------------------------------------------------------------- apply
// One CTA per subdomain k.  Box x[a][b], a over the column's patch (n_h), b
// over the element's vertical range (n_v).
__global__ void __launch_bounds__(256) k_fdm(const int32_t* __restrict__ col, const int64_t* __restrict__ hoff,
                                             const int64_t* __restrict__ moff, const int32_t* __restrict__ nvv,
                                             const int64_t* __restrict__ voff, const int64_t* __restrict__ lvoff,
                                             const int64_t* __restrict__ ioff, const int32_t* __restrict__ idx,
                                             const double* __restrict__ Sh, const double* __restrict__ lh,
                                             const double* __restrict__ Sv, const double* __restrict__ lv,
                                             const double* __restrict__ W, const double* __restrict__ r,
                                             double* __restrict__ u, int transpose, int box_max,
                                             const uint8_t* __restrict__ skip, const int32_t* __restrict__ elist) {
  extern __shared__ double sm[];
  const int k = elist ? elist[blockIdx.x] : blockIdx.x;
  if (skip[k]) return;
  const int c = col[k];
  const int nh = (int)(hoff[c + 1] - hoff[c]);
  const int nv = nvv[k];
  const int nb = nh * nv;
  double* X = sm;             // [nh][nv]
  double* T = sm + box_max;   // [nh][nv]
  double* sv = T + box_max;   // [nv][nv]
  const int32_t* id = idx + ioff[k];
  const double* S = Sh + moff[c];      // S[i][a]
  const double* Lh = lh + hoff[c];
  const double* Lv = lv + lvoff[k];
  for (int t = threadIdx.x; t < nv * nv; t += blockDim.x) sv[t] = Sv[voff[k] + t];
  for (int t = threadIdx.x; t < nb; t += blockDim.x) {
    const int g = id[t];
    double v = 0.0;
    if (g >= 0) {
      v = r[g];
      if (transpose) v *= W[g];
    }
    X[t] = v;
  }
  __syncthreads();
  // T[a][b] = sum_i S[i][a] X[i][b]
  for (int t = threadIdx.x; t < nb; t += blockDim.x) {
    const int a = t / nv, b = t % nv;
    double s = 0.0;
    for (int i = 0; i < nh; ++i) s = fma(__ldg(S + (size_t)i * nh + a), X[i * nv + b], s);
    T[t] = s;
  }
  __syncthreads();
  // X[a][j] = sum_b T[a][b] S_v[b][j] / (l_h,a + l_v,j)
  for (int t = threadIdx.x; t < nb; t += blockDim.x) {
    const int a = t / nv, j = t % nv;
    double s = 0.0;
    for (int b = 0; b < nv; ++b) s = fma(T[a * nv + b], sv[b * nv + j], s);
    X[t] = s / (__ldg(Lh + a) + __ldg(Lv + j));
  }
  __syncthreads();
  // T[a][b] = sum_j X[a][j] S_v[b][j]
  for (int t = threadIdx.x; t < nb; t += blockDim.x) {
    const int a = t / nv, b = t % nv;
    double s = 0.0;
    for (int j = 0; j < nv; ++j) s = fma(X[a * nv + j], sv[b * nv + j], s);
    T[t] = s;
  }
  __syncthreads();
  // y[i][b] = sum_a S[i][a] T[a][b]; u += R_k^T y
  for (int t = threadIdx.x; t < nb; t += blockDim.x) {
    const int g = id[t];
    if (g < 0) continue;
    const int i = t / nv, b = t % nv;
    double s = 0.0;
    const double* Si = S + (size_t)i * nh;
    for (int a = 0; a < nh; ++a) s = fma(__ldg(Si + a), T[a * nv + b], s);
    if (!transpose) s *= W[g];
    atomicAdd(u + g, s);
  }
}


// S_h (n_h x n_h, row-major, global) -> Ss [ROWS][LDS] by 8-byte cp.async, zero-filled beyond n_h
// (source size 0).  16 threads per row, 16 rows per pass: row base and validity once per row,
// one compare + select per element (the flat t -> (t / ROWS, t % ROWS) map cost ~10 instructions
// per element, 11 % of k_fdm_cta<8>'s instructions); 128-byte runs per row
template <int ROWS, int LDS>
__device__ __forceinline__ void fdm_stage_Sh(double* __restrict__ Ss, const double* __restrict__ S, int nh, int tid) {
  const int ti = tid >> 4, ta = tid & 15;
  constexpr int NP = (ROWS + 15) / 16;
#pragma unroll
  for (int pi = 0; pi < NP; ++pi) {
    const int i = ti + 16 * pi;
    if (i < ROWS) {
      const bool rv = i < nh;
      const double* src = S + (rv ? i * nh : 0);
      const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(Ss + i * LDS + ta));
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const int a = ta + 16 * k;
        if (a < ROWS) {
          const bool v = rv && a < nh;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst + 128 * k), "l"(src + (v ? a : 0)),
                       "r"(v ? 8 : 0)
                       : "memory");
        }
      }
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// 1 / d for d = l_h + l_v > 0 (normal range): MUFU.RCP64H seed (~20 bits) + two Newton steps
// (2^-40, 2^-80: FP64 accurate); replaces the float round trip (two conversions + the IEEE
// float reciprocal's fix-up branch)
__device__ __forceinline__ double fdm_rcp(double d) {
  double rc;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(d));
  rc = fma(rc, fma(-d, rc, 1.0), rc);
  rc = fma(rc, fma(-d, rc, 1.0), rc);
  return rc;
}

__device__ __forceinline__ void fdm_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Column-batched FDM sweep on FP64 tensor cores.  One CTA per work unit = a run
// of consecutive layers of one column: they share S_h, l_h and the patch.
// Each element's box is padded to NVT n-tiles of 8 columns and the boxes are
// laid side by side in B [n_h][unit columns], so every contraction is a small
// GEMM on mma.sync.m8n8k4.f64 (fragments: A a0 = A[lane>>2][lane&3], B b0 =
// B[lane&3][lane>>2], C c_i = C[lane>>2][2(lane&3)+i]):
//   T  = S_h^T B                          (per warp job: one m-tile x one element)
//   T <- ((T S_v) ./ (l_h + l_v)) S_v^T   (same warp, in registers: the C fragment
//                                          is re-laid out as an A fragment by shuffles)
//   Y  = S_h T
// then every column node sums the boxes holding it (<= 3) and is scattered.
// MT = ceil(n_h_max / 8) m-tiles (k padded to 8 MT), NVT = ceil(n_v_max / 8).
template <int NVT>
__device__ __forceinline__ double c_to_a(const double (&acc)[NVT][2], int kt, int lane) {
  // A fragment (row lane>>2, col kt*4 + (lane&3)) of the 8 x 8NVT tile held as C fragments
  const int src = (lane & ~3) | (((kt & 1) << 1) + ((lane & 3) >> 1));
  const double x0 = __shfl_sync(0xffffffffu, acc[kt >> 1][0], src);
  const double x1 = __shfl_sync(0xffffffffu, acc[kt >> 1][1], src);
  return (lane & 1) ? x1 : x0;
}

template <int MT, int NVT>
__global__ void __launch_bounds__(256) k_fdm_col(const int4* __restrict__ units, const int32_t* __restrict__ colel,
                                                 const int64_t* __restrict__ hoff, const int64_t* __restrict__ moff,
                                                 const int64_t* __restrict__ cioff, const int32_t* __restrict__ nzc,
                                                 const int32_t* __restrict__ cidx, const int32_t* __restrict__ z0,
                                                 const int32_t* __restrict__ nvv, const double* __restrict__ Sh,
                                                 const double* __restrict__ lh, const double* __restrict__ Svp,
                                                 const double* __restrict__ lvp, const double* __restrict__ W,
                                                 const double* __restrict__ r, double* __restrict__ u, int transpose,
                                                 const uint8_t* __restrict__ skip) {
  constexpr int ROWS = 8 * MT, KT = 2 * MT, NVP = 8 * NVT, EMAX = FDM_NT / NVT, LD = FDM_LD;
  extern __shared__ __align__(16) double sm[];
  double* Bc = sm;              // [ROWS][LD]  boxes, later Y
  double* Tm = Bc + ROWS * LD;  // [ROWS][LD]  column block R[h][z - zlo] first, then T
  __shared__ int ez0[EMAX], env[EMAX], eid[EMAX];
  const int4 U = units[blockIdx.x];
  const int c = U.x, first = U.y, cnt = U.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nh = (int)(hoff[c + 1] - hoff[c]);
  const int nz = nzc[c];
  const int32_t* ci = cidx + cioff[c];
  const double* S = Sh + moff[c];
  const double* Lh = lh + hoff[c];
  __shared__ int eskip[EMAX];
  if (tid < cnt) {
    const int e = colel[first + tid];
    eid[tid] = e;
    ez0[tid] = z0[e];
    env[tid] = nvv[e];
    eskip[tid] = skip[e];
  }
  __syncthreads();
  const int zlo = ez0[0], nzu = ez0[cnt - 1] + env[cnt - 1] - zlo;
  // 1. gather the unit's column block R[h][z] (x W for S^-T) into Tm
  for (int t = tid; t < nh * nzu; t += blockDim.x) {
    const int h = t / nzu, zz = t - h * nzu;
    const int g = ci[h * nz + zlo + zz];
    double v = 0.0;
    if (g >= 0) {
      v = r[g];
      if (transpose) v *= W[g];
    }
    Tm[h * LD + zz] = v;
  }
  __syncthreads();
  // 2. expand into padded boxes B[h][j*NVP + b] (zero rows >= nh, zero padding columns)
  for (int t = tid; t < ROWS * FDM_NC; t += blockDim.x) {
    const int h = t / FDM_NC, col = t - h * FDM_NC, j = col / NVP, b = col - j * NVP;
    double v = 0.0;
    if (h < nh && j < cnt && b < env[j] && !eskip[j]) v = Tm[h * LD + ez0[j] - zlo + b];
    Bc[h * LD + col] = v;
  }
  __syncthreads();
  // 3. T = S_h^T B, vertical transform in registers, T -> Tm
  for (int job = warp; job < MT * cnt; job += 8) {
    const int mt = job / cnt, j = job - mt * cnt;
    const int e = eid[j];
    double acc[NVT][2];
#pragma unroll
    for (int n = 0; n < NVT; ++n) acc[n][0] = acc[n][1] = 0.0;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const int i = kt * 4 + (lane & 3), a = mt * 8 + (lane >> 2);
      const double af = (i < nh && a < nh) ? __ldg(S + i * nh + a) : 0.0;
      const double* bp = Bc + (kt * 4 + (lane & 3)) * LD + j * NVP + (lane >> 2);
#pragma unroll
      for (int n = 0; n < NVT; ++n) fdm_dmma(acc[n][0], acc[n][1], af, bp[8 * n]);
    }
    // V = T S_v (k over b)
    const double* sv = Svp + (size_t)e * NVP * NVP;
    double v[NVT][2];
#pragma unroll
    for (int n = 0; n < NVT; ++n) v[n][0] = v[n][1] = 0.0;
#pragma unroll
    for (int kt = 0; kt < 2 * NVT; ++kt) {
      const double a = c_to_a<NVT>(acc, kt, lane);
#pragma unroll
      for (int n = 0; n < NVT; ++n)
        fdm_dmma(v[n][0], v[n][1], a, __ldg(sv + (kt * 4 + (lane & 3)) * NVP + n * 8 + (lane >> 2)));
    }
    // V ./= (l_h,a + l_v,jj)
    {
      const int a = mt * 8 + (lane >> 2);
      const double la = a < nh ? __ldg(Lh + a) : 1.0;
      const double* lv = lvp + (size_t)e * NVP;
#pragma unroll
      for (int n = 0; n < NVT; ++n)
#pragma unroll
        for (int i = 0; i < 2; ++i) v[n][i] /= (la + __ldg(lv + n * 8 + 2 * (lane & 3) + i));
    }
    // T = V S_v^T (k over jj): B[k=jj][n=b] = S_v[b][jj]
#pragma unroll
    for (int n = 0; n < NVT; ++n) acc[n][0] = acc[n][1] = 0.0;
#pragma unroll
    for (int kt = 0; kt < 2 * NVT; ++kt) {
      const double a = c_to_a<NVT>(v, kt, lane);
#pragma unroll
      for (int n = 0; n < NVT; ++n)
        fdm_dmma(acc[n][0], acc[n][1], a, __ldg(sv + (n * 8 + (lane >> 2)) * NVP + kt * 4 + (lane & 3)));
    }
#pragma unroll
    for (int n = 0; n < NVT; ++n)
      *reinterpret_cast<double2*>(Tm + (mt * 8 + (lane >> 2)) * LD + j * NVP + n * 8 + 2 * (lane & 3)) =
          make_double2(acc[n][0], acc[n][1]);
  }
  __syncthreads();
  // 4. Y = S_h T -> Bc   (A[m=i][k=a] = S[i][a]); rows a >= nh of T are zero
  for (int job = warp; job < MT * cnt; job += 8) {
    const int mt = job / cnt, j = job - mt * cnt;
    double acc[NVT][2];
#pragma unroll
    for (int n = 0; n < NVT; ++n) acc[n][0] = acc[n][1] = 0.0;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const int i = mt * 8 + (lane >> 2), a = kt * 4 + (lane & 3);
      const double af = (i < nh && a < nh) ? __ldg(S + i * nh + a) : 0.0;
      const double* bp = Tm + (kt * 4 + (lane & 3)) * LD + j * NVP + (lane >> 2);
#pragma unroll
      for (int n = 0; n < NVT; ++n) fdm_dmma(acc[n][0], acc[n][1], af, bp[8 * n]);
    }
#pragma unroll
    for (int n = 0; n < NVT; ++n)
      *reinterpret_cast<double2*>(Bc + (mt * 8 + (lane >> 2)) * LD + j * NVP + n * 8 + 2 * (lane & 3)) =
          make_double2(acc[n][0], acc[n][1]);
  }
  __syncthreads();
  // 5. every column node of the unit sums the boxes holding it, scatter (x W for S^-1)
  for (int t = tid; t < nh * nzu; t += blockDim.x) {
    const int h = t / nzu, zz = t - h * nzu;
    const int g = ci[h * nz + zlo + zz];
    if (g < 0) continue;
    const int z = zlo + zz;
    double s = 0.0;
#pragma unroll 4
    for (int j = 0; j < cnt; ++j) {
      const int dz = z - ez0[j];
      if (dz >= 0 && dz < env[j]) s += Bc[h * LD + j * NVP + dz];
    }
    if (!transpose) s *= W[g];
    atomicAdd(u + g, s);
  }
}

// Warp-per-element FDM sweep (MT <= 8, NVT <= 2).  One CTA per work unit of
// <= 8 consecutive layers of one column; warp j runs the whole local solve of
// element j in registers on mma.sync.m8n8k4.f64:
//   B1 = box of element j from the column block Rc (shared)
//   T  = S_h^T B1      A = S^T from shared S, B = B1 (registers)
//   T <- ((T S_v) ./ (l_h + l_v)) S_v^T       C -> A fragments by shuffles
//   Y  = S_h T          A = S from shared S, B = T (C -> B fragments by shuffles)
//   Yacc[h][z] += Y     (shared atomics: neighbouring boxes overlap in z)
// then every column node is scattered once.  Row strides = 4 mod 8 doubles:
// conflict-free for both fragment patterns (4 rows x 8 and 8 rows x 4).
template <int MT, int NVT>
__global__ void __launch_bounds__(256, NVT == 1 ? (MT <= 4 ? 4 : 3) : 2) k_fdm_warp(const int4* __restrict__ units, const int32_t* __restrict__ colel,
                                                  const int64_t* __restrict__ hoff, const int64_t* __restrict__ moff,
                                                  const int64_t* __restrict__ cioff, const int32_t* __restrict__ nzc,
                                                  const int32_t* __restrict__ cidx, const int32_t* __restrict__ z0,
                                                  const int32_t* __restrict__ nvv, const double* __restrict__ Sh,
                                                  const double* __restrict__ lh, const double* __restrict__ Svp,
                                                  const double* __restrict__ lvp, const double* __restrict__ W,
                                                  const double* __restrict__ r, double* __restrict__ u, int transpose,
                                                  int ldr, const uint8_t* __restrict__ skip, int nph,
                                                  const int* __restrict__ udesc, const int* __restrict__ ulist) {
  constexpr int ROWS = 8 * MT, KT = 2 * MT, NVP = 8 * NVT, LDS = ROWS + 4;
  extern __shared__ __align__(16) double sm[];
  double* Ss = sm;                  // [ROWS][LDS]  S_h (row i node, col a mode), zero padded
  double* Rc = Ss + ROWS * LDS;     // [ROWS][ldr]  column block, later the accumulator
  // unit descriptor (precomputed at setup, one coalesced load): [0] column, [1] elements,
  // [2] n_h, [3] Z_c + 1, [4..5] S_h offset, [6..7] node-id offset, [8..9] l_h offset,
  // [10..17] element ids, [18..25] z0, [26..33] n_v
  __shared__ int ud[FDM_UD];
  // warp-uniform values go through a lane-0 broadcast: ptxas then sees the branches on them as
  // uniform (no WARPSYNC.ALL + NOP in front of the mma.sync's they guard)
  const int tid = threadIdx.x, lane = tid & 31, warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int ub = ulist ? __ldg(ulist + blockIdx.x) : (int)blockIdx.x;   // unit (or the listed subset's)
  if (tid < FDM_UD) ud[tid] = __ldg(udesc + (size_t)ub * FDM_UD + tid);
  __syncthreads();
  const int c = ud[0], cnt = ud[1], nh = ud[2], nz = ud[3];
  const int64_t mo = (int64_t)(uint32_t)ud[4] | ((int64_t)ud[5] << 32);
  const int64_t co = (int64_t)(uint32_t)ud[6] | ((int64_t)ud[7] << 32);
  const int64_t ho = (int64_t)(uint32_t)ud[8] | ((int64_t)ud[9] << 32);
  const int* eid = ud + 10;
  const int* ez0 = ud + 18;
  const int* env = ud + 26;
  const int32_t* ci = cidx + co;
  const double* S = Sh + mo;
  (void)c;
  (void)units;
  (void)colel;
  (void)hoff;
  (void)moff;
  (void)cioff;
  (void)nzc;
  (void)z0;
  (void)nvv;
  fdm_stage_Sh<ROWS, LDS>(Ss, S, nh, tid);   // in flight during the column-block gather
  const int zlo = ez0[0], nzu = ez0[cnt - 1] + env[cnt - 1] - zlo;
  // column block gather: warp w owns the rows h = w + 8 i (i < MT), its lanes the z positions
  // z = lane + 32 zi (coalesced connectivity reads, no index division); the next z block's node
  // ids load behind this block's values.  Every entry of Rc is written (zeros outside the unit)
  {
    const int nzi = (ldr + 31) >> 5;
    int gid[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int h = warp + 8 * i;
      gid[i] = (h < nh && lane < nzu) ? __ldg(ci + h * nz + zlo + lane) : -1;
    }
    for (int zi = 0; zi < nzi; ++zi) {
      const int z = lane + 32 * zi, zn1 = z + 32;
      double val[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) val[i] = gid[i] >= 0 ? r[gid[i]] : 0.0;
      if (transpose) {
#pragma unroll
        for (int i = 0; i < MT; ++i)
          if (gid[i] >= 0) val[i] *= __ldg(W + gid[i]);
      }
      int gn[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int h = warp + 8 * i;
        gn[i] = (h < nh && zn1 < nzu) ? __ldg(ci + h * nz + zlo + zn1) : -1;
      }
      if (z < ldr) {
#pragma unroll
        for (int i = 0; i < MT; ++i) Rc[(warp + 8 * i) * ldr + z] = val[i];
      }
#pragma unroll
      for (int i = 0; i < MT; ++i) gid[i] = gn[i];
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const bool active = __shfl_sync(0xffffffffu, (int)(warp < cnt && !skip[eid[warp < cnt ? warp : 0]]), 0) != 0;
  const int j = warp < cnt ? warp : 0;
  const int zb = ez0[j] - zlo, nvj = env[j];
  double b1[KT][NVT];
#pragma unroll
  for (int kt = 0; kt < KT; ++kt)
#pragma unroll
    for (int n = 0; n < NVT; ++n) {
      const int col = n * 8 + (lane >> 2);
      b1[kt][n] = (active && col < nvj) ? Rc[(kt * 4 + (lane & 3)) * ldr + zb + col] : 0.0;
    }
  __syncthreads();
  for (int t = tid; t < ROWS * ldr; t += 256) Rc[t] = 0.0;  // Rc becomes the accumulator
  __syncthreads();
  double yk[MT][NVT][2];
  if (active) {
    const int e = eid[j];
    // T = S_h^T B1 over the unit's mtu = ceil(n_h / 8) tiles (S_h is zero beyond n_h: the
    // skipped tiles are exact zeros); for MT >= 5 only (the guards cost more than they save at
    // the small tile counts of p <= 3: measured on config 5's p = 2, 3 levels)
    const int mtu = MT >= 5 ? __shfl_sync(0xffffffffu, (nh + 7) / 8, 0) : MT, ktu = 2 * mtu;
    // the element's vertical modes and the first horizontal eigenvalue: loads in flight behind
    // the first GEMM (their latency sat on the vertical step's first use)
    const double* sv = Svp + (size_t)e * NVP * NVP;
    const double* lv = lvp + (size_t)e * NVP;
    double s1[2 * NVT][NVT], s2[2 * NVT][NVT], lvv[NVT][2];
#pragma unroll
    for (int kt = 0; kt < 2 * NVT; ++kt)
#pragma unroll
      for (int n = 0; n < NVT; ++n) {
        s1[kt][n] = __ldg(sv + (kt * 4 + (lane & 3)) * NVP + n * 8 + (lane >> 2));
        s2[kt][n] = __ldg(sv + (n * 8 + (lane >> 2)) * NVP + kt * 4 + (lane & 3));
      }
#pragma unroll
    for (int n = 0; n < NVT; ++n)
#pragma unroll
      for (int i = 0; i < 2; ++i) lvv[n][i] = __ldg(lv + n * 8 + 2 * (lane & 3) + i);
    const double* Lh = lh + ho;
    double la_next = (lane >> 2) < nh ? __ldg(Lh + (lane >> 2)) : 1.0;
    double T[MT][NVT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
      for (int n = 0; n < NVT; ++n) T[mt][n][0] = T[mt][n][1] = 0.0;
      if (mt >= mtu) continue;
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        if (kt >= ktu) break;
        const double af = Ss[(kt * 4 + (lane & 3)) * LDS + mt * 8 + (lane >> 2)];
#pragma unroll
        for (int n = 0; n < NVT; ++n) fdm_dmma(T[mt][n][0], T[mt][n][1], af, b1[kt][n]);
      }
    }
    // vertical: T <- ((T S_v) ./ (l_h + l_v)) S_v^T, per m-tile
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      if (mt >= mtu) break;
      double v[NVT][2];
#pragma unroll
      for (int n = 0; n < NVT; ++n) v[n][0] = v[n][1] = 0.0;
#pragma unroll
      for (int kt = 0; kt < 2 * NVT; ++kt) {
        const double a = c_to_a<NVT>(T[mt], kt, lane);
#pragma unroll
        for (int n = 0; n < NVT; ++n) fdm_dmma(v[n][0], v[n][1], a, s1[kt][n]);
      }
      const double la = la_next;   // this tile's l_h; the next tile's load issued now
      if (mt + 1 < MT) {
        const int an = (mt + 1) * 8 + (lane >> 2);
        la_next = an < nh ? __ldg(Lh + an) : 1.0;
      }
#pragma unroll
      for (int n = 0; n < NVT; ++n)
#pragma unroll
        for (int i = 0; i < 2; ++i) {  // v /= (l_h + l_v)
          const double d = la + lvv[n][i];
          v[n][i] *= fdm_rcp(d);
        }
#pragma unroll
      for (int n = 0; n < NVT; ++n) T[mt][n][0] = T[mt][n][1] = 0.0;
#pragma unroll
      for (int kt = 0; kt < 2 * NVT; ++kt) {
        const double a = c_to_a<NVT>(v, kt, lane);
#pragma unroll
        for (int n = 0; n < NVT; ++n) fdm_dmma(T[mt][n][0], T[mt][n][1], a, s2[kt][n]);
      }
    }
    // B fragments of T for Y = S_h T: B[k=a][n=col] = T[a][col]
    double b2[KT][NVT];
    {
      const int cr = (lane >> 2) & 1;
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        const int src = ((((kt & 1) << 2) + (lane & 3)) << 2) | ((lane >> 2) >> 1);
#pragma unroll
        for (int n = 0; n < NVT; ++n) {
          const double x0 = __shfl_sync(0xffffffffu, T[kt >> 1][n][0], src);
          const double x1 = __shfl_sync(0xffffffffu, T[kt >> 1][n][1], src);
          b2[kt][n] = cr ? x1 : x0;
        }
      }
    }
    // Y = S_h T (kept in registers, added to the column block by phases below)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
      for (int n = 0; n < NVT; ++n) yk[mt][n][0] = yk[mt][n][1] = 0.0;
      if (mt >= mtu) continue;
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        if (kt >= ktu) break;
        const double af = Ss[(mt * 8 + (lane >> 2)) * LDS + kt * 4 + (lane & 3)];
#pragma unroll
        for (int n = 0; n < NVT; ++n) fdm_dmma(yk[mt][n][0], yk[mt][n][1], af, b2[kt][n]);
      }
    }
  }
  // boxes j and j + k overlap only for k < nph: in phase ph the warps j = ph mod nph add
  // their (mutually disjoint) boxes with plain shared-memory adds
  for (int ph = 0; ph < nph; ++ph) {
    if (active && j % nph == ph) {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int i = mt * 8 + (lane >> 2);
        if (i < nh) {
#pragma unroll
          for (int n = 0; n < NVT; ++n)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int col = n * 8 + 2 * (lane & 3) + q;
              if (col < nvj) Rc[i * ldr + zb + col] += yk[mt][n][q];
            }
        }
      }
    }
    __syncthreads();
  }
  __syncthreads();
  {  // scatter every column node of the unit once (the gather's (row, z) map)
    const int nzi = (nzu + 31) >> 5;
    int gid[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int h = warp + 8 * i;
      gid[i] = (h < nh && lane < nzu) ? __ldg(ci + h * nz + zlo + lane) : -1;
    }
    for (int zi = 0; zi < nzi; ++zi) {
      const int z = lane + 32 * zi, zn1 = z + 32;
      double val[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) val[i] = gid[i] >= 0 ? Rc[(warp + 8 * i) * ldr + z] : 0.0;
      if (!transpose) {
#pragma unroll
        for (int i = 0; i < MT; ++i)
          if (gid[i] >= 0) val[i] *= __ldg(W + gid[i]);
      }
      int gn[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int h = warp + 8 * i;
        gn[i] = (h < nh && zn1 < nzu) ? __ldg(ci + h * nz + zlo + zn1) : -1;
      }
#pragma unroll
      for (int i = 0; i < MT; ++i)
        if (gid[i] >= 0) atomicAdd(u + gid[i], val[i]);
#pragma unroll
      for (int i = 0; i < MT; ++i) gid[i] = gn[i];
    }
  }
}

// CTA-shared FDM sweep for NVT = 2 (p >= 6: boxes of p + 3 vertical nodes, which the warp
// kernel pads to 16 columns).  The unit's elements share their column's S_h, so
//   Tall = S_h^T Rc               over the whole column block, CTA-wide (n-tiles of the z range)
//   warp j: T_j = Tall[:, box j];  T_j <- ((T_j S_v) ./ (l_h + l_v)) S_v^T   (registers)
//   Zs = [T_1 | T_2 | ...]        the boxes stacked without padding (n_v,j columns each)
//   Ys = S_h Zs                   CTA-wide over the stacked columns
//   u += sum_j Ys[:, box j]       summed per column node, scattered once (x W for S^-1)
// Same arithmetic per box as k_fdm_warp; ~40 % fewer DMMAs at p = 6.
// C[8 mtu][ncol] = A B on the CTA's 8 warps, jobs of 2 m-tiles x 2 n-tiles (four independent
// accumulator chains); A fragment a0 = A[m][k] read through (m, k) -> aidx, B from Bs[k][n] (ld ldb).
// Only the unit's mtu = ceil(n_h / 8) row / contraction tiles: S_h is zero beyond n_h, so the
// skipped tiles contribute exact zeros (and later steps read no row >= 8 mtu)
// one 2 x 2-tile job of fdm_cta_gemm with its tile validity at compile time: no branch inside the
// k loop (with run-time `if (m2)` / `if (n2)` around the mma.sync, ptxas put a WARPSYNC.ALL + NOP
// in front of every DMMA and a branch per m-tile: 3 issue slots per DMMA)
template <int MT, bool AT, bool M2, bool N2>
__device__ __forceinline__ void fdm_cta_job(const double* __restrict__ Ss, const double* __restrict__ Bs,
                                            double* __restrict__ Cs, int ldb, int ncol, int m0, int n0, int KT,
                                            int r4, int c4) {
  constexpr int ROWS = 8 * MT, LDS = ROWS + 4;
  double cc[2][2][2] = {};
  const double* pa = AT ? Ss + c4 * LDS + m0 * 8 + r4 : Ss + (m0 * 8 + r4) * LDS + c4;
  const double* pb = Bs + c4 * ldb + n0 * 8 + r4;
#pragma unroll 4
  for (int kt = 0; kt < KT; ++kt) {
    double af[2], bf[2];
    af[0] = pa[0];
    if (M2) af[1] = AT ? pa[8] : pa[8 * LDS];
    bf[0] = pb[0];
    if (N2) bf[1] = pb[8];
    pa += AT ? 4 * LDS : 4;
    pb += 4 * ldb;
    fdm_dmma(cc[0][0][0], cc[0][0][1], af[0], bf[0]);
    if (N2) fdm_dmma(cc[0][1][0], cc[0][1][1], af[0], bf[1]);
    if (M2) fdm_dmma(cc[1][0][0], cc[1][0][1], af[1], bf[0]);
    if (M2 && N2) fdm_dmma(cc[1][1][0], cc[1][1][1], af[1], bf[1]);
  }
#pragma unroll
  for (int x = 0; x < (M2 ? 2 : 1); ++x)
#pragma unroll
    for (int n = 0; n < (N2 ? 2 : 1); ++n)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int col = (n0 + n) * 8 + 2 * c4 + i;
        if (col < ncol) Cs[((m0 + x) * 8 + r4) * ldb + col] = cc[x][n][i];
      }
}

template <int MT, bool AT>
__device__ __forceinline__ void fdm_cta_gemm(const double* __restrict__ Ss, const double* __restrict__ Bs,
                                             double* __restrict__ Cs, int ldb, int ncol, int warp, int lane, int mtu) {
  const int r4 = lane >> 2, c4 = lane & 3;
  const int nt = (ncol + 7) / 8, np = (nt + 1) / 2, MP = (mtu + 1) / 2, KT = 2 * mtu;
  const int minv = 65536 / MP + 1;   // job / MP for job < 2^10 (MP <= 4): one multiply instead of a division
  for (int job = warp; job < MP * np; job += 8) {
    const int jn = (job * minv) >> 16, m0 = 2 * (job - jn * MP), n0 = 2 * jn;
    const bool m2 = m0 + 1 < mtu, n2 = n0 + 1 < nt;   // warp-uniform
    if (m2 && n2) fdm_cta_job<MT, AT, true, true>(Ss, Bs, Cs, ldb, ncol, m0, n0, KT, r4, c4);
    else if (m2) fdm_cta_job<MT, AT, true, false>(Ss, Bs, Cs, ldb, ncol, m0, n0, KT, r4, c4);
    else if (n2) fdm_cta_job<MT, AT, false, true>(Ss, Bs, Cs, ldb, ncol, m0, n0, KT, r4, c4);
    else fdm_cta_job<MT, AT, false, false>(Ss, Bs, Cs, ldb, ncol, m0, n0, KT, r4, c4);
  }
}

template <int MT>
__global__ void __launch_bounds__(256, 2) k_fdm_cta(const int32_t* __restrict__ cidx, const double* __restrict__ Sh,
                                                   const double* __restrict__ lh, const double* __restrict__ Svp,
                                                   const double* __restrict__ lvp, const double* __restrict__ W,
                                                   const double* __restrict__ r, double* __restrict__ u, int transpose,
                                                   int ldb, const uint8_t* __restrict__ skip,
                                                   const int* __restrict__ udesc, const int* __restrict__ ulist) {
  constexpr int NVT = 2, ROWS = 8 * MT, NVP = 8 * NVT, LDS = ROWS + 4;
  extern __shared__ __align__(16) double sm[];
  double* Ss = sm;                  // [ROWS][LDS]  S_h (row i node, col a mode), zero padded
  double* B1 = Ss + ROWS * LDS;     // [ROWS][ldb]  column block Rc, then the stacked boxes Zs
  double* B2 = B1 + ROWS * ldb;     // [ROWS][ldb]  Tall, then Ys
  __shared__ int ud[FDM_UD];
  __shared__ int soff[9];
  __shared__ int sk[8];
  // warp-uniform values go through a lane-0 broadcast: ptxas then sees the branches on them as
  // uniform (no WARPSYNC.ALL + NOP in front of the mma.sync's they guard)
  const int tid = threadIdx.x, lane = tid & 31, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), r4 = lane >> 2, c4 = lane & 3;
  const int ub = ulist ? __ldg(ulist + blockIdx.x) : (int)blockIdx.x;   // unit (or the listed subset's)
  if (tid < FDM_UD) ud[tid] = __ldg(udesc + (size_t)ub * FDM_UD + tid);
  __syncthreads();
  const int cnt = ud[1], nh = ud[2], nz = ud[3];
  const int64_t mo = (int64_t)(uint32_t)ud[4] | ((int64_t)ud[5] << 32);
  const int64_t co = (int64_t)(uint32_t)ud[6] | ((int64_t)ud[7] << 32);
  const int64_t ho = (int64_t)(uint32_t)ud[8] | ((int64_t)ud[9] << 32);
  const int* eid = ud + 10;
  const int* ez0 = ud + 18;
  const int* env = ud + 26;
  const int32_t* ci = cidx + co;
  const double* S = Sh + mo;
  if (tid < cnt) sk[tid] = skip[eid[tid]];
  if (tid == 0) {
    int acc = 0;
    for (int j = 0; j < cnt; ++j) {
      soff[j] = acc;
      acc += env[j];
    }
    soff[cnt] = acc;
  }
  const int zlo = ez0[0], nzu = ez0[cnt - 1] + env[cnt - 1] - zlo;
  // gather / scatter map: warp w owns the column rows h = w + 8 i (i < MT), its lanes the z
  // positions z = lane + 32 zi: coalesced connectivity reads, no index division.  Node ids of
  // the first z block, in flight together with the S_h loads
  const int nzi = (nzu + 31) >> 5;
  int gid0[2][MT];   // z blocks 0 and 1 (n_zu <= 64: the whole unit) in one batch of loads
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int h = warp + 8 * i, z = lane + 32 * b;
      gid0[b][i] = (h < nh && z < nzu) ? __ldg(ci + h * nz + zlo + z) : -1;
    }
  // S_h -> shared, completed with the column block below: the bytes stream in while the gather's
  // dependent loads are in flight
  fdm_stage_Sh<ROWS, LDS>(Ss, S, nh, tid);
  // column block (x W for S^-T): the n_h x n_zu valid entries; rows >= n_h zeroed (they meet the
  // zero columns of S_h^T: stale shared memory there could hold non-finite values), columns
  // >= n_zu only reach output columns no later step reads
  for (int zi = 0; zi < nzi; zi += 2) {
    int gid[2][MT];
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int h = warp + 8 * i, z = lane + 32 * (zi + b);
        gid[b][i] = zi == 0 ? gid0[b][i] : ((h < nh && z < nzu) ? __ldg(ci + h * nz + zlo + z) : -1);
      }
    double val[2][MT];
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int i = 0; i < MT; ++i) val[b][i] = gid[b][i] >= 0 ? r[gid[b][i]] : 0.0;
    if (transpose) {
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int i = 0; i < MT; ++i)
          if (gid[b][i] >= 0) val[b][i] *= __ldg(W + gid[b][i]);
    }
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int i = 0; i < MT; ++i)
        if (gid[b][i] >= 0) B1[(warp + 8 * i) * ldb + lane + 32 * (zi + b)] = val[b][i];
  }
  for (int t = nh * ldb + tid; t < ROWS * ldb; t += 256) B1[t] = 0.0;
  // per-box vertical modes of warp j, loaded before step 1 (latency hidden behind it)
  double s1[4][2], s2[4][2], lvv[2][2], lav[MT];
  if (warp < cnt) {
    const int e = eid[warp];
    const double* sv = Svp + (size_t)e * NVP * NVP;
    const double* lv = lvp + (size_t)e * NVP;
#pragma unroll
    for (int kt = 0; kt < 2 * NVT; ++kt)
#pragma unroll
      for (int n = 0; n < NVT; ++n) {
        s1[kt][n] = __ldg(sv + (kt * 4 + c4) * NVP + n * 8 + r4);
        s2[kt][n] = __ldg(sv + (n * 8 + r4) * NVP + kt * 4 + c4);
      }
#pragma unroll
    for (int n = 0; n < NVT; ++n)
#pragma unroll
      for (int i = 0; i < 2; ++i) lvv[n][i] = __ldg(lv + n * 8 + 2 * c4 + i);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) lav[mt] = mt * 8 + r4 < nh ? __ldg(lh + ho + mt * 8 + r4) : 1.0;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  // 1. Tall = S_h^T Rc -> B2
  const int mtu = __shfl_sync(0xffffffffu, (nh + 7) / 8, 0);
  fdm_cta_gemm<MT, true>(Ss, B1, B2, ldb, __shfl_sync(0xffffffffu, nzu, 0), warp, lane, mtu);
  __syncthreads();
  // the scatter's first chunk (step 4): node ids now, weights before step 3, both in flight
  // behind the vertical step and the second GEMM (the same (h, z) <- t map as the gather)
  int g4[2][MT];   // block 0's ids behind step 2, block 1's behind step 3
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int h = warp + 8 * i;
    g4[0][i] = (h < nh && lane < nzu) ? __ldg(ci + h * nz + zlo + lane) : -1;
  }
  // step 4's table, built here (it depends on the unit descriptor only; the barrier after step 2
  // publishes it).  The boxes are ordered by layer and their z ranges increase with j: per z the
  // stacked-column offsets of its (non-skipped) boxes, ascending j (fixed summation order)
  constexpr int ZO = 4;
  __shared__ __align__(8) short zo[2 * 8 * 16 + 2][ZO];
  __shared__ unsigned char zn[2 * 8 * 16 + 2];
  for (int z = tid; z < nzu; z += 256) {
    int k = 0;
    for (int j = 0; j < cnt; ++j) {
      const int zz = z - (ez0[j] - zlo);
      if (zz >= 0 && zz < env[j] && !sk[j]) {
        if (k < ZO) zo[z][k] = (short)(soff[j] + zz);
        ++k;
      }
    }
    for (int q = k; q < ZO; ++q) zo[z][q] = 0;
    zn[z] = (unsigned char)k;
  }
  // 2. warp j: vertical transform and scaling of box j, stored compactly into Zs (B1)
  if (__shfl_sync(0xffffffffu, (int)(warp < cnt && !sk[warp < cnt ? warp : 0]), 0)) {
    const int j = warp, zb = ez0[j] - zlo, nvj = __shfl_sync(0xffffffffu, env[j], 0), so = soff[j];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      if (mt >= mtu) break;
      double v[NVT][2];
#pragma unroll
      for (int n = 0; n < NVT; ++n) v[n][0] = v[n][1] = 0.0;
#pragma unroll
      for (int kt = 0; kt < 2 * NVT; ++kt) {  // A[a][col] = T_j[a][col] (zero beyond the box)
        if (kt >= 2 && kt * 4 >= nvj) continue;   // k-steps beyond the box: exact zeros (n_v >= 8; n_v = p + 3 <= 11 needs 3 of 4)
        const int col = kt * 4 + c4;
        const double a = col < nvj ? B2[(mt * 8 + r4) * ldb + zb + col] : 0.0;
#pragma unroll
        for (int n = 0; n < NVT; ++n) fdm_dmma(v[n][0], v[n][1], a, s1[kt][n]);
      }
      const double la = lav[mt];
#pragma unroll
      for (int n = 0; n < NVT; ++n)
#pragma unroll
        for (int i = 0; i < 2; ++i) {  // v /= (l_h + l_v)
          const double d = la + lvv[n][i];
          v[n][i] *= fdm_rcp(d);
        }
      double t2[NVT][2];
#pragma unroll
      for (int n = 0; n < NVT; ++n) t2[n][0] = t2[n][1] = 0.0;
#pragma unroll
      for (int kt = 0; kt < 2 * NVT; ++kt) {
        if (kt >= 2 && kt * 4 >= nvj) continue;   // k-steps beyond the box: exact zeros (n_v >= 8; n_v = p + 3 <= 11 needs 3 of 4)
        const double a = c_to_a<NVT>(v, kt, lane);
#pragma unroll
        for (int n = 0; n < NVT; ++n) fdm_dmma(t2[n][0], t2[n][1], a, s2[kt][n]);
      }
#pragma unroll
      for (int n = 0; n < NVT; ++n)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int col = n * 8 + 2 * c4 + i;
          if (col < nvj) B1[(mt * 8 + r4) * ldb + so + col] = t2[n][i];
        }
    }
  }
  __syncthreads();
  double w4[2][MT];   // block 0's weights behind step 3, block 1's behind block 0's sums (registers)
#pragma unroll
  for (int i = 0; i < MT; ++i) w4[0][i] = (!transpose && g4[0][i] >= 0) ? __ldg(W + g4[0][i]) : 1.0;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int h = warp + 8 * i, z = lane + 32;
    g4[1][i] = (h < nh && z < nzu) ? __ldg(ci + h * nz + zlo + z) : -1;
  }
  // 3. Ys = S_h Zs -> B2 over the stacked columns
  fdm_cta_gemm<MT, false>(Ss, B1, B2, ldb, __shfl_sync(0xffffffffu, soff[cnt], 0), warp, lane, mtu);
#pragma unroll
  for (int i = 0; i < MT; ++i) w4[1][i] = (!transpose && g4[1][i] >= 0) ? __ldg(W + g4[1][i]) : 1.0;
  __syncthreads();
  // 4. every column node of the unit: sum of the boxes holding it (table of step 2), scatter
  // (x W for S^-1).  Same (row, z) map as the gather, two z blocks per pass (node ids and
  // weights of the first pass loaded behind steps 2 and 3); a lane's table entry is read once
  // per z block and serves its MT rows
  for (int zi = 0; zi < nzi; zi += 2) {
    if (zi > 0) {
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int h = warp + 8 * i, z = lane + 32 * (zi + b);
          g4[b][i] = (h < nh && z < nzu) ? __ldg(ci + h * nz + zlo + z) : -1;
        }
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int i = 0; i < MT; ++i) w4[b][i] = (!transpose && g4[b][i] >= 0) ? __ldg(W + g4[b][i]) : 1.0;
    }
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int z = lane + 32 * (zi + b);
      const bool zv = z < nzu;
      const int nk = zv ? zn[z] : 0;
      int o[ZO];
      {
        const short4 t4 = zv ? *reinterpret_cast<const short4*>(zo[z]) : make_short4(0, 0, 0, 0);
        o[0] = t4.x, o[1] = t4.y, o[2] = t4.z, o[3] = t4.w;
      }
      double acc[MT];
      if (__all_sync(0xffffffffu, nk <= ZO)) {
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const double* row = B2 + (warp + 8 * i) * ldb;   // rows < 8 MT: inside B2 for every i
          double a = 0.0;
#pragma unroll
          for (int q = 0; q < ZO; ++q) {
            const double x = row[o[q]];
            a += q < nk ? x : 0.0;
          }
          acc[i] = a;
        }
      } else {  // more boxes than tabulated (not met for the box sizes of this kernel): walk the run
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const double* row = B2 + (warp + 8 * i) * ldb;
          double a = 0.0;
          for (int j = 0; j < cnt; ++j) {
            const int zz = z - (ez0[j] - zlo);
            if (zv && zz >= 0 && zz < env[j] && !sk[j]) a += row[soff[j] + zz];
          }
          acc[i] = a;
        }
      }
#pragma unroll
      for (int i = 0; i < MT; ++i)
        if (g4[b][i] >= 0) atomicAdd(u + g4[b][i], acc[i] * w4[b][i]);
    }
  }
}

template <int MT>
static void fdm_cta_launch(sem_ctx* c, const DeviceLevel& L, const double* r, double* u, int transpose,
                           const int* ulist = nullptr, int nu = -1) {
  const int ldz0 = 8 * L.f_nv_max, ldz = ldz0 + ((4 - ldz0 % 8) + 8) % 8;
  const int ldb = std::max(L.f_ldr, ldz);
  const int smem = (8 * MT * (8 * MT + 4) + 2 * 8 * MT * ldb) * (int)sizeof(double);
  static int attr[kMaxDev] = {0};
  smem_opt_in(k_fdm_cta<MT>, smem, attr);
  const int nb = ulist ? nu : L.f_nunits;
  if (nb == 0) return;
  k_fdm_cta<MT><<<nb, 256, smem, c->stream>>>(L.f_cidx, L.f_Sh, L.f_lh, L.f_Svp, L.f_lvp, L.W, r, u, transpose, ldb,
                                              L.f_skip, L.f_udesc, ulist);
  CUDA_CHECK(cudaGetLastError());
}

static bool fdm_cta_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SEM_FDM_CTA");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

template <int MT, int NVT>
static void fdm_warp_launch(sem_ctx* c, const DeviceLevel& L, const double* r, double* u, int transpose,
                            const int* ulist, int nu) {
  const int smem = (8 * MT * (8 * MT + 4) + 8 * MT * L.f_ldr) * (int)sizeof(double);
  static int attr[kMaxDev] = {0};
  smem_opt_in(k_fdm_warp<MT, NVT>, smem, attr);
  const int nb = ulist ? nu : L.f_nunits;
  if (nb == 0) return;
  k_fdm_warp<MT, NVT><<<nb, 256, smem, c->stream>>>(L.f_units, L.f_colel, L.f_hoff, L.f_moff, L.f_cioff, L.f_nzc,
                                                     L.f_cidx, L.f_z0, L.f_nv, L.f_Sh, L.f_lh, L.f_Svp, L.f_lvp, L.W,
                                                     r, u, transpose, L.f_ldr, L.f_skip, L.f_nph, L.f_udesc, ulist);
  CUDA_CHECK(cudaGetLastError());
}

template <int NVT>
static void fdm_warp_dispatch(sem_ctx* c, const DeviceLevel& L, const double* r, double* u, int transpose,
                              const int* ulist = nullptr, int nu = -1) {
  switch (L.f_mt) {
    case 1: fdm_warp_launch<1, NVT>(c, L, r, u, transpose, ulist, nu); break;
    case 2: fdm_warp_launch<2, NVT>(c, L, r, u, transpose, ulist, nu); break;
    case 3: fdm_warp_launch<3, NVT>(c, L, r, u, transpose, ulist, nu); break;
    case 4: fdm_warp_launch<4, NVT>(c, L, r, u, transpose, ulist, nu); break;
    case 5: fdm_warp_launch<5, NVT>(c, L, r, u, transpose, ulist, nu); break;
    case 6: fdm_warp_launch<6, NVT>(c, L, r, u, transpose, ulist, nu); break;
    case 7: fdm_warp_launch<7, NVT>(c, L, r, u, transpose, ulist, nu); break;
    default: fdm_warp_launch<8, NVT>(c, L, r, u, transpose, ulist, nu); break;
  }
}

template <int MT, int NVT>
static void fdm_col_launch(sem_ctx* c, const DeviceLevel& L, const double* r, double* u, int transpose) {
  {
    const cudaError_t pending = cudaGetLastError();
    if (pending != cudaSuccess)
      throw SemError(SEM_ECUDA, std::string("error pending before the FDM sweep: ") + cudaGetErrorString(pending));
  }
  const int smem = 2 * 8 * MT * FDM_LD * (int)sizeof(double);
  static int attr[kMaxDev] = {0};
  smem_opt_in(k_fdm_col<MT, NVT>, smem, attr);
  k_fdm_col<MT, NVT><<<L.f_nunits, 256, smem, c->stream>>>(L.f_units, L.f_colel, L.f_hoff, L.f_moff, L.f_cioff,
                                                            L.f_nzc, L.f_cidx, L.f_z0, L.f_nv, L.f_Sh, L.f_lh,
                                                            L.f_Svp, L.f_lvp, L.W, r, u, transpose, L.f_skip);
  CUDA_CHECK(cudaGetLastError());
}

template <int NVT>
static void fdm_col_dispatch(sem_ctx* c, const DeviceLevel& L, const double* r, double* u, int transpose) {
  switch (L.f_mt) {
    case 1: fdm_col_launch<1, NVT>(c, L, r, u, transpose); break;
    case 2: fdm_col_launch<2, NVT>(c, L, r, u, transpose); break;
    case 3: fdm_col_launch<3, NVT>(c, L, r, u, transpose); break;
    case 4: fdm_col_launch<4, NVT>(c, L, r, u, transpose); break;
    case 5: fdm_col_launch<5, NVT>(c, L, r, u, transpose); break;
    case 6: fdm_col_launch<6, NVT>(c, L, r, u, transpose); break;
    case 7: fdm_col_launch<7, NVT>(c, L, r, u, transpose); break;
    case 8: fdm_col_launch<8, NVT>(c, L, r, u, transpose); break;
    case 9: fdm_col_launch<9, NVT>(c, L, r, u, transpose); break;
    case 10: fdm_col_launch<10, NVT>(c, L, r, u, transpose); break;
    case 11: fdm_col_launch<11, NVT>(c, L, r, u, transpose); break;
    case 12: fdm_col_launch<12, NVT>(c, L, r, u, transpose); break;
    case 13: fdm_col_launch<13, NVT>(c, L, r, u, transpose); break;
    case 14: fdm_col_launch<14, NVT>(c, L, r, u, transpose); break;
    case 15: fdm_col_launch<15, NVT>(c, L, r, u, transpose); break;
    default: fdm_col_launch<16, NVT>(c, L, r, u, transpose); break;
  }
}

static int fdm_simple() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("SEM_FDM_SIMPLE");
    v = (s && atoi(s)) ? 1 : 0;
  }
  return v;
}

// Which FDM sweep kernel a level runs (sem_info.smoother_kernel; the dispatch below)
int fdm_kernel_choice(const DeviceLevel& L) {
  if (!L.fdm) return SEM_SMOOTHER_DENSE;
  if (!L.fcol_off.empty()) return SEM_SMOOTHER_FDM_GENERIC;   // deterministic mode: colour batches of k_fdm
  if (!fdm_simple() && L.f_warp) {
    if (L.f_nvt == 1) return SEM_SMOOTHER_FDM_WARP1;
    if (fdm_cta_enabled() && L.f_mt >= 5) return SEM_SMOOTHER_FDM_CTA;  // p >= 6: CTA-shared horizontal transforms
    return SEM_SMOOTHER_FDM_WARP2;
  }
  if (!fdm_simple() && L.f_mt <= 16 && L.f_nvt <= 3) return SEM_SMOOTHER_FDM_COL;
  return SEM_SMOOTHER_FDM_GENERIC;
}

// FDM sweep over a subset of the column units (dist.cu: interface units first, the rest while the
// exchange is in flight); the column-unit kernels only, false for the others
bool launch_fdm_list(sem_ctx* c, int level, const double* r, double* u, int transpose, const int* ulist, int nu) {
  const DeviceLevel& L = c->L[level];
  const int kind = fdm_kernel_choice(L);
  if (kind == SEM_SMOOTHER_FDM_WARP1) fdm_warp_dispatch<1>(c, L, r, u, transpose, ulist, nu);
  else if (kind == SEM_SMOOTHER_FDM_WARP2) fdm_warp_dispatch<2>(c, L, r, u, transpose, ulist, nu);
  else if (kind == SEM_SMOOTHER_FDM_CTA) {
    switch (L.f_mt) {
      case 5: fdm_cta_launch<5>(c, L, r, u, transpose, ulist, nu); break;
      case 6: fdm_cta_launch<6>(c, L, r, u, transpose, ulist, nu); break;
      case 7: fdm_cta_launch<7>(c, L, r, u, transpose, ulist, nu); break;
      default: fdm_cta_launch<8>(c, L, r, u, transpose, ulist, nu); break;
    }
  } else return false;
  c->launches++;
  return true;
}

void launch_fdm(sem_ctx* c, int level, const double* r, double* u, int transpose) {
  const DeviceLevel& L = c->L[level];
  if (c->E_own == 0) return;
  const int kind = fdm_kernel_choice(L);
  if (kind == SEM_SMOOTHER_FDM_WARP1 || kind == SEM_SMOOTHER_FDM_WARP2 || kind == SEM_SMOOTHER_FDM_CTA) {
    if (kind == SEM_SMOOTHER_FDM_WARP1) fdm_warp_dispatch<1>(c, L, r, u, transpose);
    else if (kind == SEM_SMOOTHER_FDM_CTA) {
      switch (L.f_mt) {
        case 5: fdm_cta_launch<5>(c, L, r, u, transpose); break;
        case 6: fdm_cta_launch<6>(c, L, r, u, transpose); break;
        case 7: fdm_cta_launch<7>(c, L, r, u, transpose); break;
        default: fdm_cta_launch<8>(c, L, r, u, transpose); break;
      }
    } else fdm_warp_dispatch<2>(c, L, r, u, transpose);
    c->launches++;
    return;
  }
  if (kind == SEM_SMOOTHER_FDM_COL) {
    if (L.f_nvt == 1) fdm_col_dispatch<1>(c, L, r, u, transpose);
    else if (L.f_nvt == 2) fdm_col_dispatch<2>(c, L, r, u, transpose);
    else fdm_col_dispatch<3>(c, L, r, u, transpose);
    c->launches++;
    return;
  }
  const int box = L.f_nh_max * L.f_nv_max;
  const int smem = (2 * box + L.f_nv_max * L.f_nv_max) * (int)sizeof(double);
  static int attr[kMaxDev] = {0};
  smem_opt_in(k_fdm, smem, attr);
  if (c->det.on) {  // deterministic: one launch per colour of node-disjoint FDM boxes
    for (size_t q = 0; q + 1 < L.fcol_off.size(); ++q) {
      const int nb = (int)(L.fcol_off[q + 1] - L.fcol_off[q]);
      if (nb == 0) continue;
      k_fdm<<<nb, 256, smem, c->stream>>>(L.f_col, L.f_hoff, L.f_moff, L.f_nv, L.f_voff, L.f_lvoff, L.f_ioff, L.f_idx,
                                          L.f_Sh, L.f_lh, L.f_Sv, L.f_lv, L.W, r, u, transpose, box, L.f_skip,
                                          L.fcol + L.fcol_off[q]);
    }
  } else {
    k_fdm<<<c->E_own, 256, smem, c->stream>>>(L.f_col, L.f_hoff, L.f_moff, L.f_nv, L.f_voff, L.f_lvoff, L.f_ioff,
                                              L.f_idx, L.f_Sh, L.f_lh, L.f_Sv, L.f_lv, L.W, r, u, transpose, box,
                                              L.f_skip, nullptr);
  }
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
}

}  // namespace sem
