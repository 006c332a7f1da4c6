// Static condensation of the element-interior nodes (the
// supplement's "Static Condensation", condensed system eq
// (laplacecondensed) P:655-657, interior recovery P:663; reading O43).
//
// Element-interior nodes (triangle lattice i, j, k >= 1 and 0 < l < q) belong to
// one element only, so A_ii is block diagonal with one ni x ni block per element.
// Per element the library keeps (formed once on the device from the element
// matrices, Cholesky + two triangular solves per block, cuSOLVER/cuBLAS batched):
//   H_e    = -A_ii^{-1} A_ib     [ni][nb]  (discrete-harmonic extension of the skeleton values)
//   Ainv_e =  A_ii^{-1}          [ni][ni]
// The condensed PCG runs on full-length vectors whose interior entries are kept as
// the harmonic extension of their skeleton entries: S p_b = (A E p_b)_b and
// (A E p_b)_i = 0, so one operator apply per iteration serves as the S-apply; the
// iterate u = E u_b + [0; A_ii^{-1} b_i] is the full solution at every step and its
// residual is the full system's (zero on the interior nodes).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <string>
#include <vector>

#include "internal.h"
#include "setup_util.h"

namespace sem {

struct Condense {
  int ni = 0, nb = 0, N = 0, E = 0;
  int32_t* loc = nullptr;   // [ni + nb]: local interior node ids, then the skeleton ones
  double* H = nullptr;      // [E][nb][ni] column-major ni x nb per element
  double* Ainv = nullptr;   // [E][ni][ni]
  int64_t bytes = 0;
  ~Condense() {
    cudaFree(loc);
    cudaFree(H);
    cudaFree(Ainv);
  }
};

namespace {

#define CB_CHECK(x)                                                                              \
  do {                                                                                           \
    if ((x) != CUBLAS_STATUS_SUCCESS) throw SemError(SEM_ECUDA, std::string(#x) + " failed");    \
  } while (0)
#define CS_CHECK(x)                                                                              \
  do {                                                                                           \
    if ((x) != CUSOLVER_STATUS_SUCCESS) throw SemError(SEM_ECUDA, std::string(#x) + " failed");  \
  } while (0)

template <class T>
T* raw_alloc(size_t count) {
  void* p = nullptr;
  if (cudaMalloc(&p, (count ? count : 1) * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();
    throw SemError(SEM_ENOMEM, "static condensation: cudaMalloc of " + std::to_string(count * sizeof(T)) +
                                   " bytes failed");
  }
  return (T*)p;
}

// Aii[le] (ni x ni), H[e] <- A_ib (ni x nb), Ainv[e] <- I, all column-major, from the
// row-major element matrices Ae[le][N][N] of elements e0 .. e0+ne
__global__ void k_cond_gather(int ne, int e0, int N, int ni, int nb, const int32_t* __restrict__ loc,
                              const double* __restrict__ Ae, double* __restrict__ Aii, double* __restrict__ H,
                              double* __restrict__ Ainv) {
  const int per = ni * ni + ni * nb;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)ne * per) return;
  const int le = (int)(idx / per), t = (int)(idx % per);
  const double* a = Ae + (int64_t)le * N * N;
  const int64_t e = e0 + le;
  if (t < ni * ni) {
    const int j = t / ni, k = t % ni;   // column j, row k
    Aii[(int64_t)le * ni * ni + t] = a[(int64_t)loc[k] * N + loc[j]];
    Ainv[e * ni * ni + t] = (j == k) ? 1.0 : 0.0;
  } else {
    const int s = t - ni * ni, j = s / ni, k = s % ni;
    H[e * ni * nb + s] = a[(int64_t)loc[k] * N + loc[ni + j]];
  }
}

// dst[i_k] (+)= sum_j M_e[k][j] src[s_j] for every element, one warp per element:
// M_e column-major ni x m; s_j = the m source nodes loc_src, i_k = the interior nodes.
// Dirichlet sources (conn < 0) count as 0 (masked vectors); interior nodes never are.
__global__ void k_cond_apply(int E, int N, int ni, int m, const int32_t* __restrict__ conn,
                             const int32_t* __restrict__ loc_i, const int32_t* __restrict__ loc_src,
                             const double* __restrict__ M, const double* __restrict__ src, double* __restrict__ dst,
                             int add) {
  extern __shared__ double s_src[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = blockIdx.x * (int64_t)(blockDim.x >> 5) + w;
  if (e >= E) return;
  double* s = s_src + (int64_t)w * m;
  const int32_t* ce = conn + e * N;
  for (int j = lane; j < m; j += 32) {
    const int32_t g = ce[loc_src[j]];
    s[j] = g >= 0 ? src[g] : 0.0;
  }
  __syncwarp();
  const double* Me = M + e * (int64_t)ni * m;
  for (int k = lane; k < ni; k += 32) {
    double acc = 0.0;
#pragma unroll 4
    for (int j = 0; j < m; ++j) acc = fma(Me[(int64_t)j * ni + k], s[j], acc);
    const int32_t g = ce[loc_i[k]];
    dst[g] = add ? dst[g] + acc : acc;
  }
}

__global__ void k_cond_zero(int E, int N, int ni, const int32_t* __restrict__ conn, const int32_t* __restrict__ loc_i,
                            double* __restrict__ v) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)E * ni) return;
  const int64_t e = idx / ni;
  v[conn[e * N + loc_i[idx % ni]]] = 0.0;
}

void cond_launch(sem_ctx* c, const double* M, int m, const int32_t* loc_src, const double* src, double* dst, int add) {
  const Condense& K = *c->cond;
  if (K.ni == 0) return;
  const int wpb = 4;
  const int smem = wpb * m * (int)sizeof(double);
  static int cache[kMaxDev] = {0};
  smem_opt_in(k_cond_apply, smem, cache);
  k_cond_apply<<<(K.E + wpb - 1) / wpb, 32 * wpb, smem, c->stream>>>(K.E, K.N, K.ni, m, c->L[0].conn, K.loc, loc_src,
                                                                   M, src, dst, add);
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
}

}  // namespace

void condense_setup(sem_ctx* c) {
  if (c->cond) return;
  DeviceLevel& L = c->L[0];
  const int p = L.p, q = L.q, N = L.N, E = c->E;
  std::vector<int32_t> li, lb;
  for (int n = 0; n < N; ++n) {
    const int i = L.ref.li[n], j = L.ref.lj[n], l = L.ref.ll[n], k = p - i - j;
    ((i > 0 && j > 0 && k > 0 && l > 0 && l < q) ? li : lb).push_back(n);
  }
  for (int e = 0; e < E; ++e)
    for (int32_t n : li)
      if (L.dir_host[L.conn_host[(size_t)e * N + n]])
        throw SemError(SEM_EINVAL, "static condensation: an element-interior node is a Dirichlet node");
  Condense* K = new Condense;
  c->cond = K;   // owned by the ctx from here (freed by condense_destroy on any throw below too)
  K->ni = (int)li.size();
  K->nb = (int)lb.size();
  K->N = N;
  K->E = E;
  std::vector<int32_t> loc(li);
  loc.insert(loc.end(), lb.begin(), lb.end());
  K->loc = raw_alloc<int32_t>(loc.size());
  CUDA_CHECK(cudaMemcpy(K->loc, loc.data(), loc.size() * 4, cudaMemcpyHostToDevice));
  const int ni = K->ni, nb = K->nb;
  if (ni == 0) return;   // no interior nodes (p < 3 or q < 2): the condensed system is the full one
  size_t freeb = 0, totb = 0;
  CUDA_CHECK(cudaMemGetInfo(&freeb, &totb));
  const size_t need = (size_t)E * ni * (nb + ni) * 8;
  if (need > freeb * 0.7)
    throw SemError(SEM_ENOMEM, "static condensation needs " + std::to_string(need >> 20) + " MiB of " +
                                   std::to_string(freeb >> 20) + " MiB free");
  K->H = raw_alloc<double>((size_t)E * ni * nb);
  K->Ainv = raw_alloc<double>((size_t)E * ni * ni);
  K->bytes = (int64_t)need;

  cublasHandle_t blas;
  cusolverDnHandle_t sol;
  CB_CHECK(cublasCreate(&blas));
  CS_CHECK(cusolverDnCreate(&sol));
  struct HG {
    cublasHandle_t b;
    cusolverDnHandle_t s;
    ~HG() {
      cublasDestroy(b);
      cusolverDnDestroy(s);
    }
  } hg{blas, sol};
  CB_CHECK(cublasSetStream(blas, c->stream));
  CS_CHECK(cusolverDnSetStream(sol, c->stream));
  Scratch sc;
  const double* d_D = sc.put(L.ref.Dfull);
  CUDA_CHECK(cudaMemGetInfo(&freeb, &totb));
  const size_t per = (size_t)N * N * 8 + (size_t)ni * ni * 8 + 3 * sizeof(void*) + 4;
  const int cap = (int)std::max<size_t>(1, std::min<size_t>({(size_t)E, (size_t)(freeb * 0.3 / per), 16384}));
  double* Ae = sc.get<double>((size_t)cap * N * N);
  double* Aii = sc.get<double>((size_t)cap * ni * ni);
  double** dA = sc.get<double*>(cap);
  double** dH = sc.get<double*>(cap);
  double** dX = sc.get<double*>(cap);
  int* dinfo = sc.get<int>(cap);
  std::vector<double*> hA(cap), hH(cap), hX(cap);
  std::vector<int> hinfo(cap);
  const double one = 1.0, mone = -1.0;
  for (int e0 = 0; e0 < E; e0 += cap) {
    const int ne = std::min(cap, E - e0);
    for (int t = 0; t < ne; ++t) {
      hA[t] = Aii + (size_t)t * ni * ni;
      hH[t] = K->H + (size_t)(e0 + t) * ni * nb;
      hX[t] = K->Ainv + (size_t)(e0 + t) * ni * ni;
    }
    CUDA_CHECK(cudaMemcpyAsync(dA, hA.data(), ne * sizeof(double*), cudaMemcpyHostToDevice, c->stream));
    CUDA_CHECK(cudaMemcpyAsync(dH, hH.data(), ne * sizeof(double*), cudaMemcpyHostToDevice, c->stream));
    CUDA_CHECK(cudaMemcpyAsync(dX, hX.data(), ne * sizeof(double*), cudaMemcpyHostToDevice, c->stream));
    launch_elem_matrices(c, 0, d_D, Ae, e0, ne);
    const int64_t tot = (int64_t)ne * (ni * ni + ni * nb);
    k_cond_gather<<<(int)((tot + 255) / 256), 256, 0, c->stream>>>(ne, e0, N, ni, nb, K->loc, Ae, Aii, K->H, K->Ainv);
    CUDA_CHECK(cudaGetLastError());
    CS_CHECK(cusolverDnDpotrfBatched(sol, CUBLAS_FILL_MODE_LOWER, ni, dA, ni, dinfo, ne));
    CUDA_CHECK(cudaMemcpyAsync(hinfo.data(), dinfo, ne * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    // H = -L^-T L^-1 A_ib ; Ainv = L^-T L^-1 I
    CB_CHECK(cublasDtrsmBatched(blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, ni,
                                nb, &mone, (const double* const*)dA, ni, dH, ni, ne));
    CB_CHECK(cublasDtrsmBatched(blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, ni,
                                nb, &one, (const double* const*)dA, ni, dH, ni, ne));
    CB_CHECK(cublasDtrsmBatched(blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, ni,
                                ni, &one, (const double* const*)dA, ni, dX, ni, ne));
    CB_CHECK(cublasDtrsmBatched(blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, ni,
                                ni, &one, (const double* const*)dA, ni, dX, ni, ne));
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
    for (int t = 0; t < ne; ++t)
      if (hinfo[t] != 0)
        throw SemError(SEM_ESINGULAR, "interior block of element " + std::to_string(e0 + t) +
                                          " is not SPD (potrf info " + std::to_string(hinfo[t]) + ")");
  }
}

void condense_destroy(sem_ctx* c) {
  delete c->cond;
  c->cond = nullptr;
}

// v_i = H v_b (v's interior entries become the discrete-harmonic extension of its skeleton entries)
void cond_extend(sem_ctx* c, double* v) {
  const Condense& K = *c->cond;
  cond_launch(c, K.H, K.nb, K.loc + K.ni, v, v, 0);
}

// dst_i += A_ii^{-1} src_i
void cond_interior(sem_ctx* c, const double* src, double* dst) {
  const Condense& K = *c->cond;
  cond_launch(c, K.Ainv, K.ni, K.loc, src, dst, 1);
}

// v_i = 0
void cond_zero(sem_ctx* c, double* v) {
  const Condense& K = *c->cond;
  if (K.ni == 0) return;
  const int64_t tot = (int64_t)K.E * K.ni;
  k_cond_zero<<<(int)((tot + 255) / 256), 256, 0, c->stream>>>(K.E, K.N, K.ni, c->L[0].conn, K.loc, v);
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
}

void cond_sizes(const sem_ctx* c, int* ni, int* nb, int64_t* bytes) {
  *ni = c->cond ? c->cond->ni : 0;
  *nb = c->cond ? c->cond->nb : 0;
  *bytes = c->cond ? c->cond->bytes : 0;
}

}  // namespace sem
