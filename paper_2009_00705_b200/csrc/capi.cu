// C ABI (include/sem_pmg.h): setup ("pre-compute S^-1 and A on all grids
// and re-use them"), V-cycle (Alg 4.1), PDC (Alg 4.2), PCG (Alg 4.3).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "fdm.h"
#include "internal.h"
#include "partition.h"
#include "setup_util.h"

using namespace sem;

static thread_local std::string g_last_error;

namespace sem {

#define CUBLAS_CHECK(x)                                                                  \
  do {                                                                                   \
    cublasStatus_t _s = (x);                                                             \
    if (_s != CUBLAS_STATUS_SUCCESS) throw SemError(SEM_ECUDA, std::string(#x) + " failed"); \
  } while (0)
#define CUSOLVER_CHECK(x)                                                                \
  do {                                                                                   \
    cusolverStatus_t _s = (x);                                                           \
    if (_s != CUSOLVER_STATUS_SUCCESS) throw SemError(SEM_ECUDA, std::string(#x) + " failed"); \
  } while (0)

std::vector<int> schedule_for(int p, const sem_opts& o) {
  std::vector<int> s;
  if (o.levels && o.n_levels > 0) {
    for (int i = 0; i < o.n_levels; ++i) s.push_back(o.levels[i]);
    if (s[0] != p) throw SemError(SEM_EINVAL, "levels[0] must equal p");
    const bool aniso = o.levels_z != nullptr;
    for (size_t i = 1; i < s.size(); ++i)
      if ((aniso ? s[i] > s[i - 1] : s[i] >= s[i - 1]) || s[i] < 1)
        throw SemError(SEM_EINVAL, "levels must decrease to >= 1");
    if (s.back() != 1) throw SemError(SEM_EINVAL, "the coarsest level must be P=1 (P:222-223)");
    return s;
  }
  s.push_back(p);  // P -> ceil((P+1)/2), strict-decrease guard (O18)
  while (s.back() > 1) {
    int c = (s.back() + 2) / 2;
    if (c >= s.back()) c = s.back() - 1;
    s.push_back(c);
  }
  return s;
}

// (P_xy, P_z) schedules (reading O19): explicit (opts.levels + opts.levels_z), or
// semi-coarsening of the larger order first -- to max(smaller, ceil((larger+1)/2)) with the
// strict-decrease guard -- until the orders agree, then the isotropic rule
void schedule_pq(int p, int pz, const sem_opts& o, std::vector<int>& sp, std::vector<int>& sq) {
  sp.clear();
  sq.clear();
  if (o.levels && o.n_levels > 0) {
    sp = schedule_for(p, o);
    if (o.levels_z) {
      sq.assign(o.levels_z, o.levels_z + o.n_levels);
      if (sq[0] != pz) throw SemError(SEM_EINVAL, "levels_z[0] must equal pz");
      for (size_t i = 1; i < sq.size(); ++i)
        if (sq[i] > sq[i - 1] || sq[i] < 1 || (sq[i] == sq[i - 1] && sp[i] == sp[i - 1]))
          throw SemError(SEM_EINVAL, "every level must coarsen at least one direction");
      if (sq.back() != 1) throw SemError(SEM_EINVAL, "the coarsest level must be (1,1)");
    } else {
      if (pz != p) throw SemError(SEM_EINVAL, "an anisotropic finest level needs levels_z");
      sq = sp;
    }
    return;
  }
  auto next = [](int a) {
    int c = (a + 2) / 2;
    return c >= a ? a - 1 : c;
  };
  int a = p, b = pz;
  sp.push_back(a);
  sq.push_back(b);
  while (a != b) {
    if (a > b) a = std::max(b, next(a));
    else b = std::max(a, next(b));
    sp.push_back(a);
    sq.push_back(b);
  }
  while (a > 1) {
    a = next(a);
    sp.push_back(a);
    sq.push_back(a);
  }
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ------------------------------------------------------------------ deterministic mode
void colour_sets(int64_t nsets, const std::vector<int64_t>& off, const std::vector<int32_t>& idx, int64_t nnodes,
                 const std::vector<uint8_t>* skip, std::vector<int64_t>& coff, std::vector<int32_t>& clist) {
  for (int words = 2;; words *= 2) {  // colour bitsets per node, widened until the greedy colouring fits
    std::vector<uint64_t> used((size_t)nnodes * words, 0);
    std::vector<int> col(nsets, -1);
    int ncol = 0;
    bool ok = true;
    for (int64_t k = 0; k < nsets && ok; ++k) {
      if (skip && (*skip)[k]) continue;
      std::vector<uint64_t> m(words, 0);
      for (int64_t t = off[k]; t < off[k + 1]; ++t)
        if (idx[t] >= 0)
          for (int w = 0; w < words; ++w) m[w] |= used[(size_t)idx[t] * words + w];
      int cc = -1;
      for (int w = 0; w < words && cc < 0; ++w)
        if (~m[w]) cc = 64 * w + __builtin_ctzll(~m[w]);
      if (cc < 0) {
        ok = false;
        break;
      }
      col[k] = cc;
      ncol = std::max(ncol, cc + 1);
      for (int64_t t = off[k]; t < off[k + 1]; ++t)
        if (idx[t] >= 0) used[(size_t)idx[t] * words + cc / 64] |= 1ull << (cc % 64);
    }
    if (!ok) continue;
    coff.assign(ncol + 1, 0);
    for (int64_t k = 0; k < nsets; ++k)
      if (col[k] >= 0) coff[col[k] + 1]++;
    for (int q = 0; q < ncol; ++q) coff[q + 1] += coff[q];
    clist.assign(coff[ncol], 0);
    std::vector<int64_t> pos(coff.begin(), coff.end() - 1);
    for (int64_t k = 0; k < nsets; ++k)
      if (col[k] >= 0) clist[pos[col[k]]++] = (int32_t)k;   // ascending set id within a colour
    return;
  }
}

// ------------------------------------------------------------------ Schwarz setup
void setup_schwarz(sem_ctx* c, int li, const SchwarzTopo& S, cublasHandle_t blas, cusolverDnHandle_t sol,
                   const double* d_D, int verbose) {
  DeviceLevel& L = c->L[li];
  const int E = (int)S.off.size() - 1;  // subdomains (one per owned element, or the dense subset of O35)
  L.nsub = E;
  double t0 = now_ms();
  double t1 = now_ms();
  // padded index lists and tile offsets
  std::vector<int64_t> poff(E + 1, 0), toff(E + 1, 0);
  int maxT = 0;
  for (int k = 0; k < E; ++k) {
    int nk = (int)(S.off[k + 1] - S.off[k]);
    int T = (nk + 15) / 16;
    maxT = std::max(maxT, T);
    L.nk_sum += nk;
    L.packed += (int64_t)nk * (nk + 1) / 2;
    poff[k + 1] = poff[k] + 16 * (int64_t)T;
    toff[k + 1] = toff[k] + 256 * (int64_t)T * (T + 1) / 2;
  }
  std::vector<int32_t> pidx(poff[E], -1);
  for (int k = 0; k < E; ++k)
    std::copy(S.idx.begin() + S.off[k], S.idx.begin() + S.off[k + 1], pidx.begin() + poff[k]);
  L.max_tiles_1d = maxT;
  L.schwarz_bytes = toff[E] * 8;
  size_t freeb = 0, totb = 0;
  CUDA_CHECK(cudaMemGetInfo(&freeb, &totb));
  if (c->opts.mixed_precision) L.schwarz_bytes /= 2;
  if ((size_t)L.schwarz_bytes > freeb * 0.92)
    throw SemError(SEM_ENOMEM, "dense Schwarz inverses of level p=" + std::to_string(L.p) + " need " +
                                   std::to_string(L.schwarz_bytes >> 20) + " MiB of " + std::to_string(freeb >> 20) +
                                   " MiB free; reduce overlap (0 = block Jacobi)");
  L.sidx = upload(c, pidx);
  L.sidx_off = upload(c, poff);
  L.tile_off = upload(c, toff);
  if (c->opts.mixed_precision) L.tiles32 = dalloc<float>(c, (size_t)toff[E]);
  else L.tiles = dalloc<double>(c, (size_t)toff[E]);
  L.W = upload(c, S.W);
  if (c->opts.deterministic) {  // colours of node-disjoint subdomains (one k_schwarz launch each)
    std::vector<int32_t> cl;
    colour_sets(E, S.off, S.idx, L.n, nullptr, L.scol_off, cl);
    L.scol = upload(c, cl);
  }

  Scratch sc;
  const int32_t* d_idx = sc.put(S.idx);
  const int64_t* d_off = sc.put(S.off);
  const int32_t* d_el = sc.put(S.elist);
  const int64_t* d_eoff = sc.put(S.eoff);
  const int npad = 16 * maxT;
  CUDA_CHECK(cudaMemGetInfo(&freeb, &totb));
  // element matrices are formed per chunk of subdomains, only for the element
  // range the chunk's subdomains touch (keeps setup memory bounded)
  const size_t ae_elem = (size_t)L.N * L.N * 8;
  int64_t max_el = 1;  // elements touched by one subdomain (the chunks below use compact element lists)
  for (int k = 0; k < E; ++k) max_el = std::max<int64_t>(max_el, S.eoff[k + 1] - S.eoff[k]);
  int64_t cap = std::min<int64_t>(c->E, std::max<int64_t>((int64_t)(freeb * 0.25 / ae_elem), max_el));
  double* Ae = sc.get<double>((size_t)cap * L.N * L.N);
  CUDA_CHECK(cudaMemGetInfo(&freeb, &totb));
  size_t per = (size_t)npad * npad * 8 * 2 + 64;
  size_t nb_max = std::max<size_t>(1, std::min<size_t>((size_t)(freeb * 0.6) / per, 8192));
  int nb = (int)std::min<size_t>(nb_max, (size_t)E);
  double* B = sc.get<double>((size_t)nb * npad * npad);
  double* X = sc.get<double>((size_t)nb * npad * npad);
  double** dA = sc.get<double*>(nb);
  double** dX = sc.get<double*>(nb);
  int* dinfo = sc.get<int>(nb);
  {
    std::vector<double*> hA(nb), hX(nb);
    for (int i = 0; i < nb; ++i) {
      hA[i] = B + (size_t)i * npad * npad;
      hX[i] = X + (size_t)i * npad * npad;
    }
    CUDA_CHECK(cudaMemcpy(dA, hA.data(), nb * sizeof(double*), cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(dX, hX.data(), nb * sizeof(double*), cudaMemcpyHostToDevice));
  }
  const double one = 1.0, zero = 0.0;
  std::vector<int> hinfo(nb);
  // element matrices are formed per chunk of subdomains, only for the elements the
  // chunk's subdomains touch (a compact list: subsets of O35 are scattered)
  std::vector<int32_t> ulist, slots, stamp(c->E, -1);
  int32_t* d_ulist = sc.get<int32_t>((size_t)cap);
  int32_t* d_slots = sc.get<int32_t>((size_t)std::max<int64_t>(1, S.eoff[E]));
  for (int k0 = 0; k0 < E;) {
    int cnt = 0;
    ulist.clear();
    while (k0 + cnt < E && cnt < nb) {
      const int k = k0 + cnt;
      int64_t add = 0;
      for (int64_t t = S.eoff[k]; t < S.eoff[k + 1]; ++t) add += (stamp[S.elist[t]] != k0);
      if (cnt > 0 && (int64_t)ulist.size() + add > cap) break;
      for (int64_t t = S.eoff[k]; t < S.eoff[k + 1]; ++t)
        if (stamp[S.elist[t]] != k0) {
          stamp[S.elist[t]] = k0;
          ulist.push_back(S.elist[t]);
        }
      ++cnt;
    }
    std::sort(ulist.begin(), ulist.end());
    slots.resize(S.eoff[k0 + cnt] - S.eoff[k0]);
    for (int64_t t = S.eoff[k0]; t < S.eoff[k0 + cnt]; ++t)
      slots[t - S.eoff[k0]] = (int32_t)(std::lower_bound(ulist.begin(), ulist.end(), S.elist[t]) - ulist.begin());
    CUDA_CHECK(cudaMemcpyAsync(d_ulist, ulist.data(), ulist.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CUDA_CHECK(cudaMemcpyAsync(d_slots, slots.data(), slots.size() * 4, cudaMemcpyHostToDevice, c->stream));
    launch_elem_matrices_list(c, li, d_D, Ae, d_ulist, (int)ulist.size());
    CUDA_CHECK(cudaMemsetAsync(B, 0, (size_t)cnt * npad * npad * 8, c->stream));
    launch_assemble_blocks(c, li, d_idx, d_off, d_el, d_eoff, Ae, 0, k0, cnt, npad, B, d_slots);
    launch_set_identity(c, X, cnt, npad);  // X <- I for every block
    CUSOLVER_CHECK(cusolverDnDpotrfBatched(sol, CUBLAS_FILL_MODE_LOWER, npad, dA, npad, dinfo, cnt));
    CUDA_CHECK(cudaMemcpyAsync(hinfo.data(), dinfo, cnt * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
    for (int i = 0; i < cnt; ++i)
      if (hinfo[i] != 0)
        throw SemError(SEM_ESINGULAR, "Schwarz block of element " + std::to_string(k0 + i) + " on level p=" +
                                          std::to_string(L.p) + " is not SPD (potrf info " + std::to_string(hinfo[i]) +
                                          ")");
    // X = L^-1 ; B = X^T X = (L L^T)^-1
    CUBLAS_CHECK(cublasDtrsmBatched(blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                                    npad, npad, &one, (const double* const*)dA, npad, dX, npad, cnt));
    CUBLAS_CHECK(cublasDgemmStridedBatched(blas, CUBLAS_OP_T, CUBLAS_OP_N, npad, npad, npad, &one, X, npad,
                                           (long long)npad * npad, X, npad, (long long)npad * npad, &zero, B, npad,
                                           (long long)npad * npad, cnt));
    launch_pack_tiles(c, li, B, k0, cnt, npad, d_off);
    k0 += cnt;
  }
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
  if (verbose)
    fprintf(stderr, "[sem] level p=%d schwarz: topo %.0f ms, blocks+inverse %.0f ms, max n_k %d, %.1f MiB\n", L.p,
            t1 - t0, now_ms() - t1, S.max_nk, L.schwarz_bytes / 1048576.0);
}

// ------------------------------------------------------------------ coarse setup
void setup_coarse(sem_ctx* c, const LevelTopo& topo, cusolverDnHandle_t sol, const double* d_D) {
  DeviceLevel& L = c->L.back();
  if (L.p != 1 || L.q != 1) throw SemError(SEM_EINVAL, "the coarsest level must be P=1 in both directions");
  const int E = c->E;
  std::vector<int32_t> cmap(topo.n, -1), fidx;
  for (int64_t i = 0; i < topo.n; ++i)
    if (!topo.dir[i]) {
      cmap[i] = (int32_t)fidx.size();
      fidx.push_back((int32_t)i);
    }
  const int64_t nc = (int64_t)fidx.size();
  const int mode = c->opts.coarse_solver;
  const bool dense = (mode == 2) || (mode == 0 && nc <= 46000);
  if (mode == 2 && nc > 46000)
    throw SemError(SEM_EUNSUPPORTED, "dense coarse inverse requested for " + std::to_string(nc) +
                                         " free P=1 nodes (limit 46000); use coarse_solver = 0 or 1");
  if (!dense) {  // Jacobi-preconditioned CG on the matrix-free P=1 operator (reading O9)
    c->C.iterative = 1;
    c->C.nc = nc;
    c->C.dinv = dalloc<double>(c, L.n);
    c->C.r = dalloc<double>(c, L.n);
    c->C.z = dalloc<double>(c, L.n);
    c->C.p = dalloc<double>(c, L.n);
    c->C.q = dalloc<double>(c, L.n);
    CUDA_CHECK(cudaMemsetAsync(c->C.dinv, 0, sizeof(double) * L.n, c->stream));
    Scratch sc;
    double* off = sc.get<double>((size_t)L.n);   // A[i][node above i] (vertical edges)
    CUDA_CHECK(cudaMemsetAsync(off, 0, sizeof(double) * L.n, c->stream));
    const int64_t chunk = std::min<int64_t>(E, 1 << 20);
    double* Ae = sc.get<double>((size_t)chunk * L.N * L.N);
    for (int64_t e0 = 0; e0 < E; e0 += chunk) {
      const int ne = (int)std::min<int64_t>(chunk, E - e0);
      launch_elem_matrices(c, (int)c->L.size() - 1, d_D, Ae, (int)e0, ne);
      launch_diag_accum_range(c, L.conn + (size_t)e0 * L.N, L.N, ne, Ae, c->C.dinv);
      launch_offdiag_accum(c, L.conn + (size_t)e0 * L.N, ne, Ae, off);
    }
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
    setup_coarse_lines(c, topo.conn, topo.dir, c->C.dinv, off);
    setup_coarse_agg(c, d_D, (void*)sol);
    return;
  }
  c->C.nc = nc;
  c->C.fidx = upload(c, fidx);
  c->C.x = dalloc<double>(c, nc);
  Scratch sc;
  c->C.Ainv = sc.get<double>((size_t)nc * nc);  // full inverse in scratch; stored packed (FP64) or FP32
  if (nc == 0) return;
  double* Ae = sc.get<double>((size_t)E * L.N * L.N);
  launch_elem_matrices(c, (int)c->L.size() - 1, d_D, Ae, 0, E);
  int32_t* d_cmap = sc.put(cmap);
  CUDA_CHECK(cudaMemsetAsync(c->C.Ainv, 0, (size_t)nc * nc * 8, c->stream));
  launch_assemble_coarse(c, Ae, d_cmap, c->C.Ainv, nc);
  int lwork = 0;
  CUSOLVER_CHECK(cusolverDnDpotrf_bufferSize(sol, CUBLAS_FILL_MODE_LOWER, (int)nc, c->C.Ainv, (int)nc, &lwork));
  int lwork2 = 0;
  CUSOLVER_CHECK(cusolverDnDpotri_bufferSize(sol, CUBLAS_FILL_MODE_LOWER, (int)nc, c->C.Ainv, (int)nc, &lwork2));
  double* work = sc.get<double>(std::max(lwork, lwork2));
  int* dinfo = sc.get<int>(1);
  int hinfo = 0;
  CUSOLVER_CHECK(cusolverDnDpotrf(sol, CUBLAS_FILL_MODE_LOWER, (int)nc, c->C.Ainv, (int)nc, work, lwork, dinfo));
  CUDA_CHECK(cudaMemcpyAsync(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
  if (hinfo != 0) throw SemError(SEM_ESINGULAR, "coarse Cholesky failed (info " + std::to_string(hinfo) + ")");
  CUSOLVER_CHECK(cusolverDnDpotri(sol, CUBLAS_FILL_MODE_LOWER, (int)nc, c->C.Ainv, (int)nc, work, lwork2, dinfo));
  CUDA_CHECK(cudaMemcpyAsync(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
  if (hinfo != 0) throw SemError(SEM_ESINGULAR, "coarse inverse failed (info " + std::to_string(hinfo) + ")");
  launch_symmetrize(c, c->C.Ainv, nc);
  if (c->opts.deterministic) {  // full symmetric inverse, row-wise fixed-order GEMV (k_coarse_gemv_det)
    c->C.Afull = dalloc<double>(c, (size_t)nc * nc);
    CUDA_CHECK(cudaMemcpyAsync(c->C.Afull, c->C.Ainv, (size_t)nc * nc * 8, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
    c->C.Ainv = nullptr;
    return;
  }
  {  // packed lower-triangular tiles (FP64, or FP32 storage under mixed precision, O36):
     // the GEMV reads half of the symmetric inverse
    const int64_t T = (nc + 63) / 64, len = T * (T + 1) / 2 * 4096;
    if (c->opts.mixed_precision) c->C.Apack32 = dalloc<float>(c, (size_t)len);
    else c->C.Apack = dalloc<double>(c, (size_t)len);
    launch_coarse_pack(c, nc, c->C.Ainv, c->C.Apack, c->C.Apack32);
  }
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
  c->C.Ainv = nullptr;  // scratch, freed on return
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
}

void setup_fdm(sem_ctx* c, int li, const FdmTopo& F, cusolverDnHandle_t sol, cublasHandle_t blas, int verbose);

// the dense coarse inverse re-formed from the coarsest level's current G (FNPF strategy II at
// initialisation; cuSOLVER, setup-time only)
void coarse_rebuild_dense(sem_ctx* c) {
  DeviceLevel& L = c->L.back();
  LevelTopo T;
  T.p = L.p;
  T.N = L.N;
  T.n = L.n;
  T.nfree = L.nfree;
  T.conn = L.conn_host;
  T.dir = L.dir_host;
  cusolverDnHandle_t sol;
  CUSOLVER_CHECK(cusolverDnCreate(&sol));
  struct HG {
    cusolverDnHandle_t s;
    ~HG() { cusolverDnDestroy(s); }
  } hg{sol};
  CUSOLVER_CHECK(cusolverDnSetStream(sol, c->stream));
  Scratch s2;
  c->C.Apack = nullptr;
  c->C.Apack32 = nullptr;
  c->C.Afull = nullptr;
  setup_coarse(c, T, sol, s2.put(L.ref.Dfull));
}

void check_opts(const sem_opts& o) {
  if (o.local_solve < 0 || o.local_solve > 1) throw SemError(SEM_EINVAL, "bad options: local_solve");
  if (o.mixed_precision < 0 || o.mixed_precision > 1) throw SemError(SEM_EINVAL, "bad options: mixed_precision");
  if (o.deterministic < 0 || o.deterministic > 1) throw SemError(SEM_EINVAL, "bad options: deterministic");
  if (o.pz < 0 || o.pz > 8) throw SemError(SEM_EINVAL, "bad options: pz");
  if (o.coarse_agg < -1 || o.coarse_agg > 8192) throw SemError(SEM_EINVAL, "bad options: coarse_agg (-1..8192)");
  if (o.nu1 < 0 || o.nu2 < 0 || o.overlap < -1 || o.outer < 0 || o.outer > 2 || o.apply_kernel < 0 ||
      o.apply_kernel > 4 || o.coarse_solver < 0 || o.coarse_solver > 2 || !(o.coarse_rtol > 0) ||
      o.coarse_maxit < 1 || o.nranks < 1 || o.nranks > 64 || o.rank < 0 || o.rank >= o.nranks)
    throw SemError(SEM_EINVAL, "bad options");
}

void prepare_global(const sem_mesh* mesh, int p, const sem_opts& o, GlobalModel& gm) {
  if (!mesh || !mesh->prism || !mesh->face_tag || mesh->n_prism <= 0 || (!mesh->xyz && !mesh->node_xyz))
    throw SemError(SEM_EINVAL, "mesh arrays missing");
  if (p < 1 || p > 8) throw SemError(SEM_EINVAL, "order p must be in 1..8");
  const int E = mesh->n_prism;
  HostMesh& hm = gm.hm;
  hm.nv = mesh->n_vert;
  hm.E = E;
  hm.prism.assign(mesh->prism, mesh->prism + (size_t)E * 6);
  hm.tag.assign(mesh->face_tag, mesh->face_tag + (size_t)E * 5);
  for (auto v : hm.prism)
    if (v < 0 || v >= hm.nv) throw SemError(SEM_EINVAL, "prism vertex index out of range");
  if (mesh->xyz) hm.xyz.assign(mesh->xyz, mesh->xyz + (size_t)hm.nv * 3);
  gm.P = p;
  gm.PZ = o.pz > 0 ? o.pz : p;
  if (gm.PZ > 8) throw SemError(SEM_EINVAL, "vertical order pz must be in 1..8");
  schedule_pq(p, gm.PZ, o, gm.sched, gm.schedz);
  if (gm.PZ != p || gm.sched != gm.schedz) {
    if (o.nranks > 1)
      throw SemError(SEM_EUNSUPPORTED, "anisotropic (P_xy, P_z) levels: single domain only");
  }
  gm.user_part.clear();
  if (mesh->part && o.nranks > 1) {
    gm.user_part.assign(mesh->part, mesh->part + E);
    for (int r : gm.user_part)
      if (r < 0 || r >= o.nranks) throw SemError(SEM_EINVAL, "sem_mesh.part: rank out of range");
  }
  if (gm.sched.size() > 16) throw SemError(SEM_EINVAL, "too many levels");
  const int Nf = n_prism(p, gm.PZ);
  gm.X.resize((size_t)E * Nf * 3);
  std::vector<double>& X = gm.X;
  if (mesh->node_xyz) {
    std::copy(mesh->node_xyz, mesh->node_xyz + X.size(), X.begin());
  } else {  // straight-sided: linear wedge map from the 6 vertices
    std::vector<double> rst = reference_nodes(p, gm.PZ);
#pragma omp parallel for
    for (int e = 0; e < E; ++e)
      for (int n = 0; n < Nf; ++n) {
        const double r = rst[3 * n], s = rst[3 * n + 1], t = rst[3 * n + 2];
        const double lam[3] = {-(r + s) / 2, (1 + r) / 2, (1 + s) / 2};
        for (int i = 0; i < 3; ++i) {
          double x = 0;
          for (int a = 0; a < 3; ++a) {
            x += lam[a] * (1 - t) / 2 * hm.xyz[3 * (size_t)hm.prism[(size_t)e * 6 + a] + i];
            x += lam[a] * (1 + t) / 2 * hm.xyz[3 * (size_t)hm.prism[(size_t)e * 6 + 3 + a] + i];
          }
          X[((size_t)e * Nf + n) * 3 + i] = x;
        }
      }
  }
  double tm = now_ms();
  Entities ent;
  if (gm.sched[0] >= 2 || gm.schedz[0] >= 2) ent = build_entities(hm);
  gm.topo.resize(gm.sched.size());
  for (size_t li = 0; li < gm.sched.size(); ++li) gm.topo[li] = number_level(hm, ent, gm.sched[li], gm.schedz[li]);
  if (o.verbose) fprintf(stderr, "[sem] numbering %.0f ms\n", now_ms() - tm);
}

// host coordinates of a level's nodes: the finest nodal map X (order pf) evaluated at the
// level's reference nodes; in the global build the owner element's value is kept
void level_xyz(DeviceLevel& L, int pf, const std::vector<double>& X, const std::vector<int32_t>& conn,
               const std::vector<uint8_t>& own, int E, bool all_elements, int qf) {
  if (qf < 0) qf = pf;
  const LevelRef& R = L.ref;
  const int Nf = n_prism(pf, qf);
  L.xyz.assign((size_t)L.n * 3, 0.0);
  std::vector<double> It, I1;
  transfer_matrices(L.p, pf, It, I1, R.q, qf);  // order-(pf, qf) basis at this level's nodes
  const int ntl = R.nt, n1l = R.n1, ntf = n_tri(pf), n1f = qf + 1;
#pragma omp parallel for
  for (int e = 0; e < E; ++e)
    for (int l = 0; l < n1l; ++l)
      for (int m = 0; m < ntl; ++m) {
        const int n = m + ntl * l;
        if (!all_elements && !own[(size_t)e * L.N + n]) continue;
        double x[3] = {0, 0, 0};
        for (int lf = 0; lf < n1f; ++lf)
          for (int mf = 0; mf < ntf; ++mf) {
            const double w = It[(size_t)m * ntf + mf] * I1[(size_t)l * n1f + lf];
            if (w == 0.0) continue;
            const double* Xn = &X[((size_t)e * Nf + mf + ntf * lf) * 3];
            x[0] += w * Xn[0];
            x[1] += w * Xn[1];
            x[2] += w * Xn[2];
          }
        const int32_t g = conn[(size_t)e * L.N + n];
        L.xyz[3 * (size_t)g] = x[0];
        L.xyz[3 * (size_t)g + 1] = x[1];
        L.xyz[3 * (size_t)g + 2] = x[2];
      }
}

// Device data of the levels lids (indices into gm.topo, finest first) for the
// whole mesh (part == nullptr; gsch = global Schwarz topologies, computed here
// when null) or for one rank's partition.
void build_levels(sem_ctx* c, const GlobalModel& gm, const std::vector<int>& lids, const LocalPart* part,
                  const std::vector<SchwarzTopo>* gsch) {
  const sem_opts& o = c->opts;
  const int p = gm.P, pz = gm.PZ;
  const int Nf = n_prism(p, pz);
  const int nl = (int)lids.size();
  c->PZ = pz;
  const int E = part ? (int)part->elems.size() : gm.hm.E;
  c->E = E;
  c->E_own = part ? part->E_own : E;
  c->P = p;
  // finest nodal map of the held elements
  std::vector<double> Xl;
  const std::vector<double>* Xp = &gm.X;
  if (part) {
    Xl.resize((size_t)E * Nf * 3);
    for (int i = 0; i < E; ++i)
      std::copy(gm.X.begin() + (size_t)part->elems[i] * Nf * 3, gm.X.begin() + ((size_t)part->elems[i] + 1) * Nf * 3,
                Xl.begin() + (size_t)i * Nf * 3);
    Xp = &Xl;
  }
  const std::vector<double>& X = *Xp;
  c->L.resize(nl);
  cublasHandle_t blas;
  cusolverDnHandle_t sol;
  CUBLAS_CHECK(cublasCreate(&blas));
  CUSOLVER_CHECK(cusolverDnCreate(&sol));
  struct HG {
    cublasHandle_t b;
    cusolverDnHandle_t s;
    ~HG() {
      cublasDestroy(b);
      cusolverDnDestroy(s);
    }
  } hg{blas, sol};
  CUBLAS_CHECK(cublasSetStream(blas, c->stream));
  CUSOLVER_CHECK(cusolverDnSetStream(sol, c->stream));

  Scratch sc;
  double* d_X = sc.put(X);
  for (int li = 0; li < nl; ++li) {
    DeviceLevel& L = c->L[li];
    const int lid = lids[li];
    const LevelTopo& GT = gm.topo[lid];
    const std::vector<int32_t>& conn = part ? part->L[lid].conn : GT.conn;
    const std::vector<uint8_t>& dir = part ? part->L[lid].dir : GT.dir;
    const std::vector<uint8_t>& own = part ? part->L[lid].owner : GT.owner;
    L.p = gm.sched[lid];
    L.q = gm.schedz[lid];
    L.ref = make_level_ref(L.p, L.q);
    L.N = L.ref.N;
    L.Q = L.ref.Q;
    L.n = part ? part->L[lid].n : GT.n;
    L.nfree = part ? part->L[lid].nfree : GT.nfree;
    // signed connectivity: Dirichlet nodes as ~gid
    std::vector<int32_t> sc_conn(conn.size());
    for (size_t t = 0; t < conn.size(); ++t) sc_conn[t] = dir[conn[t]] ? ~conn[t] : conn[t];
    L.conn = upload(c, sc_conn);
    L.owner = upload(c, own);
    L.dmask = upload(c, dir);
    L.dir_host = dir;
    if (part) {
      L.gid_host = part->L[lid].gid;
      L.owned_host = part->L[lid].owned;
      std::vector<uint8_t> of(L.n);
      for (int64_t i = 0; i < L.n; ++i) of[i] = part->L[lid].owned[i] && !dir[i];
      L.ownfree = upload(c, of);
      L.owned_dev = upload(c, part->L[lid].owned);
      L.gid = upload(c, part->L[lid].gid);
    }
    // reference matrices: B0 Br Bs [qt][ntp], Bt Dt [n1][n1]
    const LevelRef& R = L.ref;
    const int ntp = R.nt | 1;
    std::vector<double> mats((size_t)3 * R.qt * ntp + 2 * R.n1 * R.n1, 0.0);
    for (int a = 0; a < R.qt; ++a)
      for (int m = 0; m < R.nt; ++m) {
        mats[(size_t)0 * R.qt * ntp + a * ntp + m] = R.B0[a * R.nt + m];
        mats[(size_t)1 * R.qt * ntp + a * ntp + m] = R.Br[a * R.nt + m];
        mats[(size_t)2 * R.qt * ntp + a * ntp + m] = R.Bs[a * R.nt + m];
      }
    for (int i = 0; i < R.n1 * R.n1; ++i) {
      mats[(size_t)3 * R.qt * ntp + i] = R.Bt[i];
      mats[(size_t)3 * R.qt * ntp + R.n1 * R.n1 + i] = R.Dt[i];
    }
    L.mats = upload(c, mats);
    if (L.p == L.q) {
      L.frag = upload(c, dmma_fragments(R));
      if (L.p <= 6) L.wmats = upload(c, warp_apply_mats(R));
      if (L.p >= 3 && L.p <= 6) L.qmats = upload(c, quad_apply_mats(R));
    } else if (L.p >= 3 && L.p <= 5 && L.q >= 1 && L.q <= 5) {  // (P_xy, P_z) levels: k_apply_qs<p, q>
      const std::vector<double> qm = quad_apply_mats(R);
      if (!qm.empty()) L.qmats = upload(c, qm);
    }
    // geometric factors from the finest nodal map (all held elements)
    L.G = dalloc<double>(c, (size_t)E * 6 * L.Q);
    {
      Scratch s2;
      double* d_gm = s2.put(geometry_matrix(p, L.p, pz, L.q));
      double* d_w = s2.put(R.wq);
      if (launch_geometry(c, li, d_X, d_gm, Nf, d_w)) throw SemError(SEM_EBADELEM, "detJ <= 0 at a cubature point");
      build_g_tiles(c, li);
    }
    // node coordinates of this level (fine map evaluated at the level's nodes)
    level_xyz(L, p, X, conn, own, E, part != nullptr, pz);
    if (!part) {  // kept for sem_update_geometry (single domain)
      L.conn_host = conn;
      L.owner_host = own;
    }
    if (li + 1 < nl) {
      std::vector<double> It, I1;
      transfer_matrices(L.p, gm.sched[lids[li + 1]], It, I1, L.q, gm.schedz[lids[li + 1]]);
      L.Itri = upload(c, It);
      L.I1 = upload(c, I1);
    }
    L.u = dalloc<double>(c, L.n);
    L.f = dalloc<double>(c, L.n);
    L.r = dalloc<double>(c, L.n);
    if (part) L.d = dalloc<double>(c, L.n);
  }
  sc.release(d_X);
  // smoothers (all but the coarsest) and, in the global build, the coarse solver
  for (int li = 0; li < nl; ++li) {
    Scratch s2;
    double* d_D = s2.put(c->L[li].ref.Dfull);
    const int lid = lids[li];
    if ((o.apply_kernel == 0 || o.apply_kernel >= 3) && c->L[li].p == c->L[li].q) build_p1_matrices(c, li, d_D);
    if (li + 1 < nl) {
      double t0 = now_ms();
      if (part && o.local_solve == 1) {  // partitioned FDM / exact-dense hybrid (O33, O35)
        const FdmTopo& F = part->F[lid];
        bool any = false;
        for (uint8_t r : F.regular) any |= !r;
        if (any) setup_schwarz(c, li, schwarz_subset(part->L[lid].S, F.regular), blas, sol, d_D, o.verbose);
        setup_fdm(c, li, F, sol, blas, o.verbose);
      } else if (part) {
        setup_schwarz(c, li, part->L[lid].S, blas, sol, d_D, o.verbose);
      } else if (gsch) {
        setup_schwarz(c, li, (*gsch)[lid], blas, sol, d_D, o.verbose);
      } else if (o.local_solve == 1) {
        const int ov = o.overlap >= 0 ? o.overlap : (c->L[li].p + 2) / 2;  // refined: ceil((P+1)/2)
        FdmTopo F = fdm_topology(gm.hm, gm.topo[lid], gm.X, p, ov, gm.PZ);
        if (o.verbose) fprintf(stderr, "[sem] level p=%d FDM topology %.0f ms\n", c->L[li].p, now_ms() - t0);
        int64_t nirr = 0;
        for (uint8_t r : F.regular) nirr += !r;
        if (nirr > 0) {  // reading O35: exact dense local inverses on the irregular subdomains
          SchwarzTopo S = schwarz_topology(gm.topo[lid], E, ov, std::min(32, std::max(1, omp_get_max_threads())));
          SchwarzTopo Sd = schwarz_subset(S, F.regular);
          // W of the hybrid smoother: counts over the FDM boxes of the regular and the O15 sets of the others
          std::vector<double> cnt(gm.topo[lid].n, 0.0);
          for (int e = 0; e < E; ++e)
            if (F.regular[e]) {
              for (int64_t t = F.ioff[e]; t < F.ioff[e + 1]; ++t)
                if (F.idx[t] >= 0) cnt[F.idx[t]] += 1.0;
            } else {
              for (int64_t t = S.off[e]; t < S.off[e + 1]; ++t) cnt[S.idx[t]] += 1.0;
            }
          for (int64_t i = 0; i < gm.topo[lid].n; ++i)
            F.W[i] = gm.topo[lid].dir[i] ? 0.0 : 1.0 / cnt[i];
          setup_schwarz(c, li, Sd, blas, sol, d_D, o.verbose);
          if (o.verbose) fprintf(stderr, "[sem] level p=%d hybrid: %lld of %d subdomains dense (O35)\n", c->L[li].p,
                                 (long long)nirr, E);
        }
        setup_fdm(c, li, F, sol, blas, o.verbose);
      } else {
        const int ov = o.overlap >= 0 ? o.overlap : (c->L[li].p + 2) / 2;  // refined: ceil((P+1)/2)
        SchwarzTopo S = schwarz_topology(gm.topo[lid], E, ov, std::min(32, std::max(1, omp_get_max_threads())));
        if (o.verbose) fprintf(stderr, "[sem] level p=%d schwarz topology %.0f ms\n", c->L[li].p, now_ms() - t0);
        setup_schwarz(c, li, S, blas, sol, d_D, o.verbose);
      }
    } else if (!part) {
      setup_coarse(c, gm.topo[lid], sol, d_D);
    }
  }
  // solver work
  const int64_t n0 = c->L[0].n;
  c->pw = dalloc<double>(c, n0);
  c->qw = dalloc<double>(c, n0);
  c->zw = dalloc<double>(c, n0);
  c->bw = dalloc<double>(c, n0);
  c->xw = dalloc<double>(c, n0);
  c->host_in = dalloc<double>(c, n0);
  c->host_in2 = dalloc<double>(c, n0);
  c->host_out = dalloc<double>(c, n0);
  c->scal = dalloc<double>(c, 32);
  c->rw_old = dalloc<double>(c, n0);
  CUDA_CHECK(cudaMallocHost(&c->hscal, 32 * sizeof(double)));
  CUDA_CHECK(cudaEventCreate(&c->ev0));
  CUDA_CHECK(cudaEventCreate(&c->ev1));
}

void do_setup(const sem_mesh* mesh, int p, const sem_opts* opts, sem_ctx* c) {
  NvtxRange nv("sem_setup");
  const double t_start = now_ms();
  if (opts) c->opts = *opts;
  else sem_default_opts(&c->opts);
  const sem_opts& o = c->opts;
  check_opts(o);
  if (o.device >= 0) CUDA_CHECK(cudaSetDevice(o.device));
  CUDA_CHECK(cudaGetDevice(&c->device));
  c->stream = (cudaStream_t)o.stream;
  GlobalModel gm;
  prepare_global(mesh, p, o, gm);
  c->E_global = gm.hm.E;
  if (o.nranks > 1) {
    if (o.deterministic) throw SemError(SEM_EUNSUPPORTED, "deterministic mode: single-domain ctx only");
    setup_distributed(c, gm);
  } else {
    std::vector<int> lids(gm.sched.size());
    for (size_t i = 0; i < lids.size(); ++i) lids[i] = (int)i;
    build_levels(c, gm, lids, nullptr, nullptr);
    if (o.deterministic) {  // element colours: elements sharing a vertex (hence any node) differ
      const DeviceLevel& Lc = c->L.back();
      const std::vector<int32_t>& cv = Lc.conn_host;
      std::vector<int64_t> off(c->E + 1);
      for (int e = 0; e <= c->E; ++e) off[e] = (int64_t)e * Lc.N;
      std::vector<int32_t> cl;
      colour_sets(c->E, off, cv, Lc.n, nullptr, c->det.ecol_off, cl);
      c->det.ecol = upload(c, cl);
      c->det.part = dalloc<double>(c, 2 * 8192);
      c->det.on = 1;
    }
    // one finest-level apply, timed for the work-unit count of every solve (O25)
    const int64_t n0 = c->L[0].n;
    CUDA_CHECK(cudaMemsetAsync(c->pw, 0, sizeof(double) * n0, c->stream));
    for (int i = 0; i < 2; ++i) launch_apply(c, 0, c->pw, c->qw, 0);
    CUDA_CHECK(cudaEventRecord(c->ev0, c->stream));
    for (int i = 0; i < 5; ++i) launch_apply(c, 0, c->pw, c->qw, 0);
    CUDA_CHECK(cudaEventRecord(c->ev1, c->stream));
    CUDA_CHECK(cudaEventSynchronize(c->ev1));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    c->t_apply_ms = ms / 5.0;
  }
  CUDA_CHECK(cudaDeviceSynchronize());
  c->launches = 0;
  c->setup_ms = now_ms() - t_start;
  if (o.verbose) fprintf(stderr, "[sem] setup %.0f ms, device %.1f MiB\n", c->setup_ms, c->device_bytes / 1048576.0);
}

void read_scalars(sem_ctx* c, int n);

void coarse_solve(sem_ctx* c, const double* f, double* u) {
  if (c->C.iterative) coarse_pcg(c, f, u);
  else launch_coarse(c, f, u);
}

// ------------------------------------------------------------------ V-cycle (Alg 4.1)
void vcycle(sem_ctx* c, int li, const double* f, double* u) {
  NvtxRange nv(nvtx_level_name(li));
  const int nl = (int)c->L.size();
  if (li == nl - 1) {  // coarsest: exact solve (O10, O26)
    coarse_solve(c, f, u);
    return;
  }
  DeviceLevel& L = c->L[li];
  const sem_opts& o = c->opts;
  const int post_t = o.literal_smoother ? 0 : 1;
  CUDA_CHECK(cudaMemsetAsync(u, 0, sizeof(double) * L.n, c->stream));
  // line 1: nu1 pre-smoothing steps u <- u + S^-1 (f - A u)
  for (int m = 0; m < o.nu1; ++m) {
    if (m == 0) {
      launch_schwarz(c, li, f, u, 0);  // u = 0: the residual is f
    } else {
      launch_init_masked(c, li, f, L.r, 1);
      launch_apply(c, li, u, L.r, AP_NEGATE);
      launch_schwarz(c, li, L.r, u, 0);
    }
  }
  // line 2: r = f - A u
  launch_init_masked(c, li, f, L.r, 1);
  if (o.nu1 > 0) launch_apply(c, li, u, L.r, AP_NEGATE);
  // line 3: restrict; lines 4-6: coarse solve or recursion
  DeviceLevel& C = c->L[li + 1];
  launch_restrict(c, li, L.r, C.f);
  vcycle(c, li + 1, C.f, C.u);
  // lines 7-8: prolong and correct
  launch_prolong(c, li, C.u, u);
  // line 9: nu2 post-smoothing steps with S^-T (reading O14) or S^-1 (literal)
  for (int m = 0; m < o.nu2; ++m) {
    launch_init_masked(c, li, f, L.r, 1);
    launch_apply(c, li, u, L.r, AP_NEGATE);
    launch_schwarz(c, li, L.r, u, post_t);
  }
}

// z = V(r) for PCG on the ctx's own buffers, replayed from a CUDA graph: the V-cycle is a
// fixed sequence of ~100 small launches (launch-bound on small configs).  Captured on a
// private stream after one eager run (function attributes set), replayed on the solve's
// stream.  Not used with the iterative coarse solve (host syncs) or partitioned ctxs;
// SEM_NO_GRAPHS=1 disables it.
void vcycle_pcg(sem_ctx* c, const double* r, double* z) {
  static const int off = [] {
    const char* e = getenv("SEM_NO_GRAPHS");
    return (e && atoi(e)) ? 1 : 0;
  }();
  const int slot = (z == c->pw) ? 0 : ((z == c->zw) ? 1 : -1);
  if (off || slot < 0 || r != c->bw || c->vc_eager < 1) {
    vcycle(c, 0, r, z);
    c->vc_eager++;
    return;
  }
  if (!c->vc_graph[slot]) {
    if (!c->cap_stream) CUDA_CHECK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
    cudaStream_t keep = c->stream;
    c->stream = c->cap_stream;
    const int64_t l0 = c->launches;
    cudaGraph_t g = nullptr;
    CUDA_CHECK(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
    try {
      vcycle(c, 0, r, z);
    } catch (...) {
      cudaStreamEndCapture(c->cap_stream, &g);
      if (g) cudaGraphDestroy(g);
      c->stream = keep;
      throw;
    }
    CUDA_CHECK(cudaStreamEndCapture(c->cap_stream, &g));
    c->stream = keep;
    c->vc_graph_launches[slot] = c->launches - l0;
    c->launches = l0;
    CUDA_CHECK(cudaGraphInstantiate(&c->vc_graph[slot], g, 0));
    CUDA_CHECK(cudaGraphDestroy(g));
  }
  CUDA_CHECK(cudaGraphLaunch(c->vc_graph[slot], c->stream));
  c->launches += c->vc_graph_launches[slot];
}

void read_scalars(sem_ctx* c, int n) {
  CUDA_CHECK(cudaMemcpyAsync(c->hscal, c->scal, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
}

// ------------------------------------------------------------------ solve
int do_solve(sem_ctx* c, const double* rhs, const double* phiD, double tol, double* phi, sem_report* rep,
             int guess = 0, int cond = 0) {
  NvtxRange nv(cond ? "laplace_solve_condensed" : "laplace_solve");
  if (!phiD || !phi) throw SemError(SEM_EINVAL, "dirichlet_phi and phi are required");
  if (!(tol >= 0.0)) throw SemError(SEM_EINVAL, "tol must be >= 0");
  DeviceLevel& L = c->L[0];
  const sem_opts& o = c->opts;
  const int64_t n = L.n;
  sem_report R;
  memset(&R, 0, sizeof(R));
  coarse_reset_iters(c);
  CUDA_CHECK(cudaEventRecord(c->ev0, c->stream));
  double* u = c->xw;   // free-node iterate
  double* r = c->bw;   // residual
  double* p = c->pw;
  double* q = c->qw;
  double* z = c->zw;
  double* sc = c->scal;
  // lift: v = phi_D on Dirichlet nodes (0 elsewhere), b_F = rhs_F - A_FD phi_D
  launch_init_masked(c, 0, phiD, q, 0);
  launch_init_masked(c, 0, rhs, r, 1);
  launch_apply(c, 0, q, r, AP_GATHER_ALL | AP_NEGATE);
  CUDA_CHECK(cudaMemsetAsync(u, 0, sizeof(double) * n, c->stream));
  if (o.outer != 0)  // PDC / MG recompute r = b_F - A_FF u from the kept b_F
    CUDA_CHECK(cudaMemcpyAsync(c->rw_old, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  launch_dot2(c, n, r, r, nullptr, nullptr, nullptr, sc + 4);
  read_scalars(c, 5);
  const double nf = std::sqrt(c->hscal[4]);
  R.norm_f = nf;
  const double thresh = tol * nf + o.atol;
  double rn = nf;
  if (cond) {
    // static condensation (NEXT-3; condense.cu): u = E u_b + [0; A_ii^-1 b_i] with
    // u_b = phi_b (warm start) or 0, r = b_F - A_FF u (zero on the interior nodes)
    if (guess) {
      launch_init_masked(c, 0, phi, u, 1);
      cond_extend(c, u);
    }
    cond_interior(c, r, u);
    launch_apply(c, 0, u, r, AP_NEGATE);
    cond_zero(c, r);
    launch_dot2(c, n, r, r, nullptr, nullptr, nullptr, sc + 6);
    read_scalars(c, 7);
    rn = std::sqrt(c->hscal[6]);
  } else if (guess) {  // warm start (NEXT-1, the paper's per-stage solves): u_F = phi_F, r = b_F - A_FF u_F
    launch_init_masked(c, 0, phi, u, 1);
    launch_apply(c, 0, u, r, AP_NEGATE);
    launch_dot2(c, n, r, r, nullptr, nullptr, nullptr, sc + 6);
    read_scalars(c, 7);
    rn = std::sqrt(c->hscal[6]);
  }
  R.res_hist[R.n_hist++] = rn;
  int status = SEM_OK;
  if (rn <= thresh) {
    R.converged = 1;
  } else if (o.outer == 0) {
    // Alg 4.3: p = V(r); delta = p^T r.  With an iterative coarse solve the
    // preconditioner is not exactly linear: flexible CG (Polak-Ribiere beta)
    const bool flex = c->C.iterative != 0;
    vcycle_pcg(c, r, p);
    if (cond) cond_extend(c, p);   // condensed preconditioner E (V r)_b
    R.vcycles++;
    int dcur = 8, dnew = 10;  // [d] = z^T r, [d+1] = z^T r_old
    launch_dot2(c, n, p, r, nullptr, nullptr, nullptr, sc + dcur);
    while (R.iters < o.imax) {
      // q = A p (masked: p is 0 on Dirichlet nodes)
      CUDA_CHECK(cudaMemsetAsync(q, 0, sizeof(double) * n, c->stream));
      launch_apply(c, 0, p, q, 0);
      if (cond) cond_zero(c, q);     // (A E p_b)_i = 0: q = [S p_b; 0]
      launch_dot2(c, n, p, q, nullptr, nullptr, nullptr, sc + 1);
      if (flex) CUDA_CHECK(cudaMemcpyAsync(c->rw_old, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
      // alpha = delta / p^T q; u += alpha p; r -= alpha q; ||r||^2
      launch_axpy_pcg(c, n, u, r, p, q, sc + dcur, sc + 1, sc + 3);
      R.iters++;
      read_scalars(c, 4);
      if (!(c->hscal[1] > 0.0)) {
        status = SEM_EBREAKDOWN;
        break;
      }
      rn = std::sqrt(c->hscal[3]);
      if (R.n_hist < 256) R.res_hist[R.n_hist++] = rn;
      if (rn <= thresh) {
        R.converged = 1;
        break;
      }
      // z = V(r); beta = z^T r / delta (flexible: z^T (r - r_old) / delta); p = z + beta p
      vcycle_pcg(c, r, z);
      if (cond) cond_extend(c, z);
      R.vcycles++;
      if (flex) {
        launch_dot2(c, n, z, r, z, c->rw_old, nullptr, sc + dnew);
        launch_xpby(c, n, p, z, sc + dnew, sc + dcur, 2);
      } else {
        launch_dot2(c, n, z, r, nullptr, nullptr, nullptr, sc + dnew);
        launch_xpby(c, n, p, z, sc + dnew, sc + dcur, 0);
      }
      std::swap(dcur, dnew);
    }
  } else {
    // Alg 4.2 (PDC; reading O13) and stand-alone MG: u <- u - MG(-r) = u + V(r)
    const double* bF = c->rw_old;  // b_F of the lift (kept below)
    while (R.iters < o.imax) {
      vcycle(c, 0, r, z);
      if (cond) cond_extend(c, z);
      R.vcycles++;
      launch_axpy(c, n, 1.0, z, u);
      // r = b_F - A_FF u (one operator apply per iteration)
      CUDA_CHECK(cudaMemcpyAsync(r, bF, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
      launch_apply(c, 0, u, r, AP_NEGATE);
      if (cond) cond_zero(c, r);
      R.iters++;
      launch_dot2(c, n, r, r, nullptr, nullptr, nullptr, sc + 3);
      read_scalars(c, 4);
      rn = std::sqrt(c->hscal[3]);
      if (R.n_hist < 256) R.res_hist[R.n_hist++] = rn;
      if (rn <= thresh) {
        R.converged = 1;
        break;
      }
    }
  }
  launch_combine_phi(c, 0, u, phiD, phi);
  CUDA_CHECK(cudaEventRecord(c->ev1, c->stream));
  CUDA_CHECK(cudaEventSynchronize(c->ev1));
  float ms = 0.f;
  CUDA_CHECK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  R.t_ms = ms;
  R.wu = c->t_apply_ms > 0 ? ms / c->t_apply_ms : 0.0;
  R.coarse_iters = (int)coarse_iters(c, false);
  coarse_count_launches(c, R.coarse_iters);
  R.rel_res = nf > 0 ? rn / nf : 0.0;
  if (R.n_hist > 1) {
    const int m = R.n_hist - 1;
    R.q_mean = std::pow(R.res_hist[m] / R.res_hist[0], 1.0 / m);
  }
  if (status == SEM_OK && !R.converged) status = SEM_ENOTCONV;
  if (rep) *rep = R;
  return status;
}

int fail(const SemError& e) {
  g_last_error = e.what();
  return e.code;
}

}  // namespace sem

// ====================================================================== C ABI
extern "C" {

void sem_default_opts(sem_opts* o) {
  memset(o, 0, sizeof(*o));
  o->nu1 = 3;
  o->nu2 = 3;
  o->overlap = 1;
  o->literal_smoother = 0;
  o->outer = 0;
  o->levels = nullptr;
  o->n_levels = 0;
  o->atol = 0.0;
  o->imax = 200;
  o->stream = nullptr;
  o->device = -1;
  o->verbose = 0;
  o->apply_kernel = 0;
  o->coarse_solver = 0;
  o->coarse_rtol = 1e-10;
  o->coarse_maxit = 20000;
  o->nranks = 1;
  o->rank = 0;
  o->nccl_id = nullptr;
  o->pz = 0;
  o->levels_z = nullptr;
  o->coarse_agg = -1;
}

int sem_reference_nodes(int p, double* rst) {
  if (p < 1 || p > 8 || !rst) return SEM_EINVAL;
  std::vector<double> v = reference_nodes(p);
  std::copy(v.begin(), v.end(), rst);
  return SEM_OK;
}

int sem_reference_nodes_pq(int p, int pz, double* rst) {
  if (p < 1 || p > 8 || pz < 1 || pz > 8 || !rst) return SEM_EINVAL;
  std::vector<double> v = reference_nodes(p, pz);
  std::copy(v.begin(), v.end(), rst);
  return SEM_OK;
}

int sem_setup(const sem_mesh* mesh, int p, const sem_opts* opts, sem_ctx** out) {
  if (!out) return SEM_EINVAL;
  *out = nullptr;
  sem_ctx* c = new sem_ctx();
  int caller_dev = -1;
  cudaGetDevice(&caller_dev);
  struct Restore {
    int d;
    ~Restore() {
      if (d >= 0) cudaSetDevice(d);
    }
  } restore{caller_dev};
  try {
    do_setup(mesh, p, opts, c);
  } catch (const SemError& e) {
    sem_destroy(c);
    return fail(e);
  } catch (const std::exception& e) {
    sem_destroy(c);
    g_last_error = e.what();
    return SEM_EINVAL;
  }
  *out = c;
  return SEM_OK;
}

int sem_get_info(const sem_ctx* c, sem_info* info) {
  if (!c || !info) return SEM_EINVAL;
  memset(info, 0, sizeof(*info));
  if (c->dist) {
    dist_info(c, info);
    info->setup_ms = c->setup_ms;
    return SEM_OK;
  }
  info->n_dof = c->L[0].n;
  info->n_free = c->L[0].nfree;
  info->n_elem = c->E;
  info->n_levels = (int)c->L.size();
  info->coarse_agg = c->C.nagg;
  for (size_t i = 0; i < c->L.size(); ++i) {
    info->level_p[i] = c->L[i].p;
    info->level_pz[i] = c->L[i].q;
    info->level_n_dof[i] = c->L[i].n;
    info->level_n_free[i] = c->L[i].nfree;
    info->schwarz_bytes[i] = c->L[i].schwarz_bytes;
    info->schwarz_nk_sum[i] = c->L[i].nk_sum;
    info->schwarz_packed[i] = c->L[i].packed;
    info->smoother_kernel[i] = (i + 1 < c->L.size()) ? fdm_kernel_choice(c->L[i]) : SEM_SMOOTHER_NONE;
    info->smoother_mt[i] = c->L[i].fdm ? c->L[i].f_mt : 0;
  }
  info->coarse_n = c->C.nc;
  info->device_bytes = c->device_bytes;
  info->setup_ms = c->setup_ms;
  return SEM_OK;
}

int sem_node_xyz(const sem_ctx* c, int level, double* xyz, int on_device) {
  const int nl = c ? (c->dist ? dist_levels(c) : (int)c->L.size()) : 0;
  if (!c || !xyz || level < 0 || level >= nl) return SEM_EINVAL;
  DeviceGuard guard(c->device);
  const auto& v = c->dist ? dist_xyz(c, level) : c->L[level].xyz;
  if (on_device) {
    if (cudaMemcpy(xyz, v.data(), v.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) return SEM_ECUDA;
  } else {
    std::copy(v.begin(), v.end(), xyz);
  }
  return SEM_OK;
}

int sem_dirichlet_mask(const sem_ctx* c, int level, uint8_t* mask, int on_device) {
  const int nl = c ? (c->dist ? dist_levels(c) : (int)c->L.size()) : 0;
  if (!c || !mask || level < 0 || level >= nl) return SEM_EINVAL;
  DeviceGuard guard(c->device);
  const auto& v = c->dist ? dist_dir(c, level) : c->L[level].dir_host;
  if (on_device) {
    if (cudaMemcpy(mask, v.data(), v.size(), cudaMemcpyHostToDevice) != cudaSuccess) return SEM_ECUDA;
  } else {
    std::copy(v.begin(), v.end(), mask);
  }
  return SEM_OK;
}

int sem_apply_laplace(sem_ctx* c, const double* u, double* y, int level, int masked) {
  if (!c || !u || !y || u == y) return SEM_EINVAL;
  DeviceGuard guard(c->device);
  if (c->dist) {
    try {
      return dist_apply(c, u, y, level, masked);
    } catch (const SemError& e) {
      return fail(e);
    }
  }
  if (level < 0 || level >= (int)c->L.size()) return SEM_EINVAL;
  try {
    if (masked) {
      launch_init_masked(c, level, u, y, 0);
      launch_apply(c, level, u, y, 0);
    } else {
      CUDA_CHECK(cudaMemsetAsync(y, 0, sizeof(double) * c->L[level].n, c->stream));
      launch_apply(c, level, u, y, AP_GATHER_ALL | AP_SCATTER_ALL);
    }
  } catch (const SemError& e) {
    return fail(e);
  }
  return SEM_OK;
}

int pmg_vcycle(sem_ctx* c, const double* r, double* z) {
  if (!c || !r || !z || r == z) return SEM_EINVAL;
  DeviceGuard guard(c->device);
  try {
    if (c->dist) return dist_vcycle(c, r, z);
    vcycle(c, 0, r, z);
  } catch (const SemError& e) {
    return fail(e);
  }
  return SEM_OK;
}

int laplace_solve(sem_ctx* c, const double* rhs, const double* phiD, double tol, double* phi, sem_report* rep) {
  if (!c) return SEM_EINVAL;
  DeviceGuard guard(c->device);
  try {
    if (c->dist) {
      if (!phiD || !phi || !(tol >= 0.0)) return SEM_EINVAL;
      return dist_solve(c, rhs, phiD, tol, phi, rep);
    }
    return do_solve(c, rhs, phiD, tol, phi, rep);
  } catch (const SemError& e) {
    return fail(e);
  }
}

int laplace_solve_condensed(sem_ctx* c, const double* rhs, const double* phiD, double tol, double* phi, int guess,
                            sem_report* rep) {
  if (!c) return SEM_EINVAL;
  if (c->dist) return SEM_EUNSUPPORTED;
  DeviceGuard guard(c->device);
  try {
    if (!phiD || !phi) throw SemError(SEM_EINVAL, "dirichlet_phi and phi are required");
    if (!c->cond) {
      try {
        condense_setup(c);
      } catch (...) {
        condense_destroy(c);
        throw;
      }
    }
    return do_solve(c, rhs, phiD, tol, phi, rep, guess ? 1 : 0, 1);
  } catch (const SemError& e) {
    return fail(e);
  }
}

int sem_condensed_info(sem_ctx* c, int* n_interior, int* n_skeleton, int64_t* bytes) {
  if (!c || !n_interior || !n_skeleton || !bytes) return SEM_EINVAL;
  if (c->dist) return SEM_EUNSUPPORTED;
  DeviceGuard guard(c->device);
  try {
    if (!c->cond) {
      try {
        condense_setup(c);
      } catch (...) {
        condense_destroy(c);
        throw;
      }
    }
    cond_sizes(c, n_interior, n_skeleton, bytes);
  } catch (const SemError& e) {
    return fail(e);
  }
  return SEM_OK;
}

int sem_update_geometry(sem_ctx* c, const double* node_xyz, int strategy) {
  if (!c || !node_xyz || (strategy != 1 && strategy != 2 && strategy != 4)) return SEM_EINVAL;
  if (c->dist) return SEM_EUNSUPPORTED;
  DeviceGuard guard(c->device);
  try {
    if (strategy == 4 && c->L.size() > 1 && (!c->L[0].fdm || !c->C.iterative))
      throw SemError(SEM_EUNSUPPORTED, "strategy III (4) re-forms smoothers and coarse preconditioner every stage: "
                                       "needs local_solve = 1 and coarse_solver = 1");
    if (strategy == 4 && c->PZ != c->P)
      throw SemError(SEM_EUNSUPPORTED, "strategy III (4): isotropic orders only");
    condense_destroy(c);   // the interior factorisations follow the geometry (re-formed on the next condensed solve)
    const int p = c->P, Nf = n_prism(p, c->PZ), E = c->E;
    std::vector<double> X(node_xyz, node_xyz + (size_t)E * Nf * 3);
    Scratch sc;
    const double* d_X = sc.put(X);
    const int nlev = (strategy == 1) ? 1 : (int)c->L.size();   // 2, 4: every level's operator
    for (int li = 0; li < nlev; ++li) {
      DeviceLevel& L = c->L[li];
      Scratch s2;
      const double* d_gm = s2.put(geometry_matrix(p, L.p, c->PZ, L.q));
      const double* d_w = s2.put(L.ref.wq);
      if (launch_geometry(c, li, d_X, d_gm, Nf, d_w)) throw SemError(SEM_EBADELEM, "detJ <= 0 at a cubature point");
      if (L.Gw) build_g_tiles(c, li);
      if (L.Ae1) {
        const double* d_D = s2.put(L.ref.Dfull);
        build_p1_matrices(c, li, d_D);
      }
      level_xyz(L, p, X, L.conn_host, L.owner_host, E, false, c->PZ);
    }
    if (strategy == 4 && c->L.size() > 1) {  // III: every smoother and the coarse preconditioner too
      for (size_t li = 0; li + 1 < c->L.size(); ++li) fdm_refresh_vertical(c, (int)li, d_X);
      coarse_refresh_lines(c);
    }
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
  } catch (const SemError& e) {
    return fail(e);
  }
  return SEM_OK;
}

int laplace_solve_guess(sem_ctx* c, const double* rhs, const double* phiD, double tol, double* phi, sem_report* rep) {
  if (!c) return SEM_EINVAL;
  if (c->dist) return SEM_EUNSUPPORTED;
  DeviceGuard guard(c->device);
  try {
    return do_solve(c, rhs, phiD, tol, phi, rep, 1);
  } catch (const SemError& e) {
    return fail(e);
  }
}

int laplace_solve_host(sem_ctx* c, const double* rhs_host, const double* phiD_host, double tol, double* phi_host,
                       sem_report* rep) {
  if (!c || !phiD_host || !phi_host) return SEM_EINVAL;
  DeviceGuard guard(c->device);
  try {
    sem_info inf;
    sem_get_info(c, &inf);
    const int64_t n = inf.n_dof;
    if (c->dist && !c->host_in) {
      c->host_in = dalloc<double>(c, n);
      c->host_in2 = dalloc<double>(c, n);
      c->host_out = dalloc<double>(c, n);
    }
    if (rhs_host)
      CUDA_CHECK(cudaMemcpyAsync(c->host_in2, rhs_host, n * 8, cudaMemcpyHostToDevice, c->stream));
    CUDA_CHECK(cudaMemcpyAsync(c->host_in, phiD_host, n * 8, cudaMemcpyHostToDevice, c->stream));
    int st = c->dist ? dist_solve(c, rhs_host ? c->host_in2 : nullptr, c->host_in, tol, c->host_out, rep)
                     : do_solve(c, rhs_host ? c->host_in2 : nullptr, c->host_in, tol, c->host_out, rep);
    CUDA_CHECK(cudaMemcpyAsync(phi_host, c->host_out, n * 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
    return st;
  } catch (const SemError& e) {
    return fail(e);
  }
}

int sem_prolong(sem_ctx* c, int level, const double* uc, double* uf) {
  if (c && c->dist) return SEM_EUNSUPPORTED;
  if (!c || !uc || !uf || level < 0 || level + 1 >= (int)c->L.size()) return SEM_EINVAL;
  DeviceGuard guard(c->device);
  try {
    launch_prolong(c, level, uc, uf);
  } catch (const SemError& e) {
    return fail(e);
  }
  return SEM_OK;
}

int sem_restrict(sem_ctx* c, int level, const double* rf, double* rc) {
  if (c && c->dist) return SEM_EUNSUPPORTED;
  if (!c || !rf || !rc || level < 0 || level + 1 >= (int)c->L.size()) return SEM_EINVAL;
  DeviceGuard guard(c->device);
  try {
    launch_restrict(c, level, rf, rc);
  } catch (const SemError& e) {
    return fail(e);
  }
  return SEM_OK;
}

int sem_schwarz(sem_ctx* c, int level, const double* r, double* u, int transpose) {
  if (c && c->dist) return SEM_EUNSUPPORTED;
  if (!c || !r || !u || level < 0 || level + 1 >= (int)c->L.size()) return SEM_EINVAL;
  DeviceGuard guard(c->device);
  try {
    launch_schwarz(c, level, r, u, transpose);
  } catch (const SemError& e) {
    return fail(e);
  }
  return SEM_OK;
}

int sem_coarse_solve(sem_ctx* c, const double* r, double* z) {
  if (c && c->dist) return SEM_EUNSUPPORTED;
  if (!c || !r || !z) return SEM_EINVAL;
  DeviceGuard guard(c->device);
  try {
    coarse_solve(c, r, z);
  } catch (const SemError& e) {
    return fail(e);
  }
  return SEM_OK;
}

int sem_bench_kernel(sem_ctx* c, int kernel, int level, int reps, double* mean_us, double* alg_bytes) {
  if (!c || reps < 1 || kernel < 0 || kernel > 2) return SEM_EINVAL;
  DeviceGuard guard(c->device);
  try {
    sem_ctx* t = c->dist ? dist_part0(c) : c;
    if (kernel == 2) level = (int)t->L.size() - 1;
    if (kernel == 2 && !t->C.Apack && !t->C.Apack32) return SEM_EINVAL;
    if (level < 0 || level >= (int)t->L.size()) return SEM_EINVAL;
    if (kernel == 0 && level + 1 >= (int)t->L.size()) return SEM_EINVAL;
    DeviceLevel& L = t->L[level];
    CUDA_CHECK(cudaMemsetAsync(L.f, 0, sizeof(double) * L.n, t->stream));
    CUDA_CHECK(cudaMemsetAsync(L.u, 0, sizeof(double) * L.n, t->stream));
    auto run = [&]() {
      if (kernel == 0) launch_schwarz(t, level, L.f, L.u, 0);
      else if (kernel == 2) launch_coarse(t, L.f, L.u);
      else launch_apply(t, level, L.f, L.u, 0);
    };
    for (int i = 0; i < 3; ++i) run();
    CUDA_CHECK(cudaEventRecord(t->ev0, t->stream));
    for (int i = 0; i < reps; ++i) run();
    CUDA_CHECK(cudaEventRecord(t->ev1, t->stream));
    CUDA_CHECK(cudaEventSynchronize(t->ev1));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, t->ev0, t->ev1));
    if (mean_us) *mean_us = 1e3 * ms / reps;
    if (alg_bytes) {
      const int64_t nc = t->C.nc, T = (nc + 63) / 64;
      if (kernel == 2)  // packed lower tiles of the inverse + x, index, z
        *alg_bytes = (t->C.Apack ? 8.0 : 4.0) * 4096.0 * (double)(T * (T + 1) / 2) + 28.0 * nc;
      else if (kernel == 0 && L.fdm)
        *alg_bytes = (double)L.f_bytes + (L.tiles32 ? 4.0 : 8.0) * L.packed + 32.0 * L.n +
                     (L.nsub ? 4.0 * L.nk_sum : 0.0);
      else if (kernel == 0)
        *alg_bytes = (L.tiles32 ? 4.0 : 8.0) * L.packed + 4.0 * L.nk_sum + 32.0 * L.n;
      else if (L.Ae1 && (t->opts.apply_kernel == 0 || t->opts.apply_kernel >= 3))  // element-matrix path (p <= 2)
        *alg_bytes = (double)t->E_own * (8.0 * L.N * (L.N + 1) / 2 + 4.0 * L.N) + 16.0 * L.n;
      else
        *alg_bytes = (double)t->E_own * (48.0 * L.Q + 4.0 * L.N) + 16.0 * L.n;
    }
  } catch (const SemError& e) {
    return fail(e);
  }
  return SEM_OK;
}

int sem_fnpf_init(sem_ctx* c, const double* node_xyz, int strategy, int64_t* n_surface) {
  if (!c || !node_xyz) return SEM_EINVAL;
  DeviceGuard guard(c->device);
  try {
    fnpf_init(c, node_xyz, strategy);
    if (n_surface) *n_surface = fnpf_surface(c, nullptr);
  } catch (const SemError& e) {
    return fail(e);
  }
  return SEM_OK;
}

int sem_fnpf_surface_nodes(const sem_ctx* c, int32_t* node_ids) {
  if (!c || !node_ids || !c->fnpf) return SEM_EINVAL;
  fnpf_surface(c, node_ids);
  return SEM_OK;
}

int fnpf_rhs(sem_ctx* c, const double* eta, const double* phis, double* deta, double* dphis, double* w, double tol,
             int linear, sem_report* rep) {
  if (!c || !c->fnpf || !eta || !phis || !deta || !dphis || !(tol >= 0.0)) return SEM_EINVAL;
  DeviceGuard guard(c->device);
  try {
    sem_report R;
    fnpf_stage(c, eta, phis, deta, dphis, w, tol, linear, &R);
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
    if (rep) *rep = R;
    return R.converged ? SEM_OK : SEM_ENOTCONV;
  } catch (const SemError& e) {
    return fail(e);
  }
}

int fnpf_erk4_step(sem_ctx* c, double* eta, double* phis, double dt, double tol, int linear, int* iters) {
  if (!c || !c->fnpf || !eta || !phis || !(tol >= 0.0)) return SEM_EINVAL;
  DeviceGuard guard(c->device);
  try {
    fnpf_erk4(c, eta, phis, dt, tol, linear, iters);
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
  } catch (const SemError& e) {
    return fail(e);
  }
  return SEM_OK;
}

int sem_nccl_unique_id(void* id_out) {
  if (!id_out) return SEM_EINVAL;
  try {
    nccl_unique_id(id_out);
  } catch (const SemError& e) {
    return fail(e);
  }
  return SEM_OK;
}

int64_t sem_launch_count(const sem_ctx* c, int reset) {
  if (!c) return -1;
  if (c->dist) return dist_launches(c, reset) + c->launches;
  int64_t v = c->launches;
  if (reset) const_cast<sem_ctx*>(c)->launches = 0;
  return v;
}

void sem_destroy(sem_ctx* c) {
  if (!c) return;
  DeviceGuard guard(c->device);
  cudaDeviceSynchronize();
  dist_destroy(c);
  for (int i = 0; i < 2; ++i)
    if (c->vc_graph[i]) cudaGraphExecDestroy(c->vc_graph[i]);
  coarse_destroy(c);
  fnpf_destroy(c);
  condense_destroy(c);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  for (void* p : c->allocs) cudaFree(p);
  if (c->hscal) cudaFreeHost(c->hscal);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  delete c;
}

// ---------------------------------------------------------------- host diagnostics
static HostMesh host_mesh_of(const sem_mesh* mesh) {
  if (!mesh || !mesh->prism || !mesh->face_tag || mesh->n_prism <= 0) throw SemError(SEM_EINVAL, "mesh arrays missing");
  HostMesh hm;
  hm.nv = mesh->n_vert;
  hm.E = mesh->n_prism;
  hm.prism.assign(mesh->prism, mesh->prism + (size_t)hm.E * 6);
  hm.tag.assign(mesh->face_tag, mesh->face_tag + (size_t)hm.E * 5);
  for (auto v : hm.prism)
    if (v < 0 || v >= hm.nv) throw SemError(SEM_EINVAL, "prism vertex index out of range");
  return hm;
}

int sem_host_numbering(const sem_mesh* mesh, int p, int64_t* n_dof, int64_t* n_free, int32_t* conn,
                       uint8_t* dirichlet, uint8_t* owner) {
  if (p < 1 || p > 8) return SEM_EINVAL;
  try {
    HostMesh hm = host_mesh_of(mesh);
    Entities ent;
    if (p >= 2) ent = build_entities(hm);
    LevelTopo T = number_level(hm, ent, p);
    if (n_dof) *n_dof = T.n;
    if (n_free) *n_free = T.nfree;
    if (conn) std::copy(T.conn.begin(), T.conn.end(), conn);
    if (dirichlet) std::copy(T.dir.begin(), T.dir.end(), dirichlet);
    if (owner) std::copy(T.owner.begin(), T.owner.end(), owner);
  } catch (const SemError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SEM_EINVAL;
  }
  return SEM_OK;
}

int sem_host_schwarz(const sem_mesh* mesh, int p, int overlap, int64_t* total, int64_t* off, int32_t* idx,
                     double* W) {
  if (p < 1 || p > 8 || overlap < 0) return SEM_EINVAL;
  try {
    HostMesh hm = host_mesh_of(mesh);
    Entities ent;
    if (p >= 2) ent = build_entities(hm);
    LevelTopo T = number_level(hm, ent, p);
    SchwarzTopo S = schwarz_topology(T, hm.E, overlap, std::min(32, std::max(1, omp_get_max_threads())));
    if (total) *total = S.off[hm.E];
    if (off) std::copy(S.off.begin(), S.off.end(), off);
    if (idx) std::copy(S.idx.begin(), S.idx.end(), idx);
    if (W) std::copy(S.W.begin(), S.W.end(), W);
  } catch (const SemError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SEM_EINVAL;
  }
  return SEM_OK;
}

int sem_host_partition(const sem_mesh* mesh, int p, int nranks, int rank, int level, int64_t* sizes,
                       int32_t* elems, int32_t* gid, uint8_t* owned, int32_t* nbr, int64_t* xoff, int32_t* xidx) {
  if (p < 2 || p > 8 || nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks || !sizes) return SEM_EINVAL;
  try {
    sem_opts o;
    sem_default_opts(&o);
    o.nranks = nranks;
    GlobalModel gm;
    prepare_global(mesh, p, o, gm);
    if (level < 0 || level >= (int)gm.sched.size()) return SEM_EINVAL;
    std::vector<int> epart;
    std::vector<SchwarzTopo> sch;
    compute_partition(gm, o, epart, sch);
    LocalPart P = extract_part(gm.topo, sch, epart, rank, nranks);
    const LocalLevel& L = P.L[level];
    int64_t nx = 0;
    for (auto& v : L.xidx) nx += (int64_t)v.size();
    sizes[0] = (int64_t)P.elems.size();
    sizes[1] = P.E_own;
    sizes[2] = L.n;
    sizes[3] = (int64_t)L.nbr.size();
    sizes[4] = nx;
    if (elems) std::copy(P.elems.begin(), P.elems.end(), elems);
    if (gid) std::copy(L.gid.begin(), L.gid.end(), gid);
    if (owned) std::copy(L.owned.begin(), L.owned.end(), owned);
    if (nbr) std::copy(L.nbr.begin(), L.nbr.end(), nbr);
    if (xoff || xidx) {
      int64_t o2 = 0;
      if (xoff) xoff[0] = 0;
      for (size_t j = 0; j < L.xidx.size(); ++j) {
        if (xidx) std::copy(L.xidx[j].begin(), L.xidx[j].end(), xidx + o2);
        o2 += (int64_t)L.xidx[j].size();
        if (xoff) xoff[j + 1] = o2;
      }
    }
  } catch (const SemError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SEM_EINVAL;
  }
  return SEM_OK;
}

int sem_host_fdm(const sem_mesh* mesh, int p, int overlap, int64_t* total, int64_t* off, int32_t* idx, double* W) {
  if (p < 1 || p > 8 || overlap < 0) return SEM_EINVAL;
  try {
    sem_opts o;
    sem_default_opts(&o);
    int lv[1] = {p};
    if (p == 1) { o.levels = lv; o.n_levels = 1; }
    GlobalModel gm;
    prepare_global(mesh, p, o, gm);
    FdmTopo F = fdm_topology(gm.hm, gm.topo[0], gm.X, p, overlap);
    const int E = gm.hm.E;
    SchwarzTopo S;
    bool hybrid = false;
    for (uint8_t r : F.regular) hybrid |= !r;
    if (hybrid) S = schwarz_topology(gm.topo[0], E, overlap, std::min(32, std::max(1, omp_get_max_threads())));
    std::vector<int64_t> o2(E + 1, 0);
    std::vector<int32_t> all;
    std::vector<double> cnt(gm.topo[0].n, 0.0);
    for (int e = 0; e < E; ++e) {
      std::vector<int32_t> s;
      if (F.regular[e]) {
        for (int64_t t = F.ioff[e]; t < F.ioff[e + 1]; ++t)
          if (F.idx[t] >= 0) s.push_back(F.idx[t]);
      } else {  // reading O35: exact local inverse on the O15 set
        s.assign(S.idx.begin() + S.off[e], S.idx.begin() + S.off[e + 1]);
      }
      std::sort(s.begin(), s.end());
      for (int32_t g : s) cnt[g] += 1.0;
      all.insert(all.end(), s.begin(), s.end());
      o2[e + 1] = (int64_t)all.size();
    }
    for (int64_t i = 0; i < gm.topo[0].n; ++i) F.W[i] = gm.topo[0].dir[i] ? 0.0 : 1.0 / cnt[i];
    if (total) *total = (int64_t)all.size();
    if (off) std::copy(o2.begin(), o2.end(), off);
    if (idx) std::copy(all.begin(), all.end(), idx);
    if (W) std::copy(F.W.begin(), F.W.end(), W);
  } catch (const SemError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SEM_EINVAL;
  }
  return SEM_OK;
}

int sem_host_reference(int p, double* B0, double* Br, double* Bs, double* Bt, double* Dt, double* w) {
  if (p < 1 || p > 8) return SEM_EINVAL;
  LevelRef R = make_level_ref(p);
  if (B0) std::copy(R.B0.begin(), R.B0.end(), B0);
  if (Br) std::copy(R.Br.begin(), R.Br.end(), Br);
  if (Bs) std::copy(R.Bs.begin(), R.Bs.end(), Bs);
  if (Bt) std::copy(R.Bt.begin(), R.Bt.end(), Bt);
  if (Dt) std::copy(R.Dt.begin(), R.Dt.end(), Dt);
  if (w) std::copy(R.wq.begin(), R.wq.end(), w);
  return SEM_OK;
}

const char* sem_strerror(int code) {
  switch (code) {
    case SEM_OK: return "success";
    case SEM_EINVAL: return "invalid argument";
    case SEM_EBADELEM: return "invalid element (detJ <= 0)";
    case SEM_ENOMEM: return "out of device memory";
    case SEM_ESINGULAR: return "singular Schwarz block or coarse matrix";
    case SEM_ENOTCONV: return "not converged within imax iterations";
    case SEM_EBREAKDOWN: return "PCG breakdown (p^T A p <= 0)";
    case SEM_ECUDA: return "CUDA / cuSOLVER / cuBLAS error";
    case SEM_ENCCL: return "communication error";
    case SEM_EUNSUPPORTED: return "unsupported option combination";
    default: return "unknown error";
  }
}

const char* sem_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"
