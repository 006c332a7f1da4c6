// Iterative P=1 coarse solve ("A^-1"; reading O9): preconditioned CG on the
// matrix-free P=1 operator to ||r|| <= coarse_rtol ||b||, for coarse problems too
// large for the stored dense inverse.
//
// Preconditioner: vertical-line block Jacobi.  The P=1 nodes of a layered prism mesh
// form vertical lines (a prism's top vertex v3+m sits above its bottom vertex v0+m);
// the coarse operator restricted to one line is tridiagonal (the lines' own vertical
// edges), and it carries the strong coupling of thin layers (config 4: d_xy / d_z = 4,
// so the vertical couplings are ~16x the horizontal ones).  Each line is solved
// exactly by the Thomas algorithm with factors precomputed at setup; on meshes whose
// prisms do not stack consistently every line is a single node (point Jacobi).
//
// Two-level correction (reading O44): the line solves leave the smooth horizontal error, so
// the preconditioner adds an exact solve on a coarse space of piecewise constants over
// aggregates of whole lines (recursive coordinate bisection of the lines' (x, y)):
//   z = T^-1 r + P_a A_a^-1 P_a^T r,   A_a = P_a^T A P_a (dense inverse, formed at setup).
// Both terms are SPD, so CG stays CG.  Restriction P_a^T r is fused into the line kernel
// (one atomic per line), A_a^-1 is one small dense GEMV, and the prolongation is folded into
// the search-direction update p = (T^-1 r + P_a z_a) + beta p.
//
// The whole solve runs on the device: the stop test is a CUDA-graph WHILE node whose
// condition a one-thread kernel sets after every iteration, so no host round trip
// happens inside the solve and the V-cycle that contains it can itself be captured
// and replayed from a CUDA graph (capi.cu vcycle_pcg).  Outside a capture the solve
// is replayed from a cached graph of its own.
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "internal.h"
#include "partition.h"
#include "setup_util.h"

namespace sem {

// device scalar slots of the coarse solve (C.cs)
// (k_line_solve writes z.r and r.r to two consecutive slots: CS_ZR_NEW, CS_RR_DUP)
enum : int { CS_PQ = 0, CS_RR = 1, CS_ZR_OLD = 2, CS_ZR_NEW = 3, CS_RR_DUP = 4, CS_THR2 = 6, CS_IT = 7,
             CS_TOTAL = 8, CS_GO = 9, CS_N = 16 };
static_assert(CS_RR_DUP == CS_ZR_NEW + 1, "line solve output slots");

static int cgrid(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  return (int)std::max<int64_t>(g, 1);
}

// off[i] += A_e[m][m+3] for the vertical edge (i = bottom m, j = top m) of every P=1 prism (setup)
__global__ void k_offdiag_accum(int64_t E, const int32_t* __restrict__ conn, const double* __restrict__ Ae,
                                double* __restrict__ off) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= E * 3) return;
  const int64_t e = idx / 3;
  const int m = (int)(idx % 3);
  const int32_t i = conn[e * 6 + m], j = conn[e * 6 + m + 3];
  if (i >= 0 && j >= 0) atomicAdd(off + i, Ae[(e * 6 + m) * 6 + m + 3]);
}

// z = T^-1 r on every line (Thomas algorithm with precomputed factors), out[0] += z.r, out[1] += r.r
__global__ void k_line_solve(int nlines, const int64_t* __restrict__ loff, const int32_t* __restrict__ lnode,
                             const double* __restrict__ ta, const double* __restrict__ tinv,
                             const double* __restrict__ tc, const double* __restrict__ r, double* __restrict__ z,
                             double* out, double* part) {
  double s0 = 0.0, s1 = 0.0;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nlines; l += gridDim.x * blockDim.x) {
    const int64_t b = loff[l], e = loff[l + 1];
    double d = 0.0;
    for (int64_t t = b; t < e; ++t) {  // forward elimination: d'_t = (r_t - a_t d'_{t-1}) / den_t
      d = (r[lnode[t]] - ta[t] * d) * tinv[t];
      z[lnode[t]] = d;
    }
    double x = 0.0;
    for (int64_t t = e - 1; t >= b; --t) {  // back substitution: x_t = d'_t - c'_t x_{t+1}
      const int32_t g = lnode[t];
      x = z[g] - tc[t] * x;
      z[g] = x;
      const double rg = r[g];
      s0 = fma(x, rg, s0);
      s1 = fma(rg, rg, s1);
    }
  }
  // block reduction + one atomic per block
  __shared__ double sh0[32], sh1[32];
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    sh0[w] = s0;
    sh1[w] = s1;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    s0 = lane < nw ? sh0[lane] : 0.0;
    s1 = lane < nw ? sh1[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (lane == 0) {
      if (part) {  // deterministic mode: fixed-order sum in det_finalize
        part[2 * blockIdx.x] = s0;
        part[2 * blockIdx.x + 1] = s1;
      } else {
        atomicAdd(out, s0);
        atomicAdd(out + 1, s1);
      }
    }
  }
}

__global__ void k_zero_slots(double* cs, int a, int b, int c2, int d) {
  cs[a] = 0.0;
  cs[b] = 0.0;
  if (c2 >= 0) cs[c2] = 0.0;
  if (d >= 0) cs[d] = 0.0;
}

// after the prologue: thr^2 = rtol^2 ||b||^2 (||b||^2 = r.r of the initial residual), loop iff b != 0
__global__ void k_coarse_start(double* cs, double rtol2, cudaGraphConditionalHandle h, int use_h) {
  cs[CS_THR2] = rtol2 * cs[CS_RR_DUP];
  cs[CS_IT] = 0.0;
  cs[CS_ZR_OLD] = cs[CS_ZR_NEW];
  const unsigned go = cs[CS_RR_DUP] > 0.0 ? 1u : 0u;
  cs[CS_PQ] = 0.0;
  cs[CS_RR] = 0.0;
  cs[CS_ZR_NEW] = 0.0;
  cs[CS_RR_DUP] = 0.0;
  cs[CS_GO] = go;
  if (use_h) cudaGraphSetConditional(h, go);
}

// end of one CG iteration: beta used, shift z.r, count, stop test ||r||^2 <= thr^2 or maxit,
// zero the reduction slots of the next iteration
__global__ void k_coarse_next(double* cs, double maxit, cudaGraphConditionalHandle h, int use_h) {
  const double rr = cs[CS_RR];
  cs[CS_ZR_OLD] = cs[CS_ZR_NEW];
  cs[CS_IT] += 1.0;
  cs[CS_TOTAL] += 1.0;
  const unsigned go = (rr > cs[CS_THR2] && cs[CS_IT] < maxit) ? 1u : 0u;
  cs[CS_PQ] = 0.0;
  cs[CS_RR] = 0.0;
  cs[CS_ZR_NEW] = 0.0;
  cs[CS_RR_DUP] = 0.0;
  cudaGraphSetConditional(h, go);
}

// ---- fused iteration (P = 1 element matrices available, default mode): three kernels per CG iteration
__device__ __forceinline__ double cw_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// q = A_FF p (packed P = 1 element matrices, one thread per element) and p^T A p = sum_e p_e^T A_e p_e
// (p = 0 on Dirichlet nodes, so the element energies sum to p^T q)
__global__ void __launch_bounds__(128) k_coarse_apply_pq(int E, const int32_t* __restrict__ conn,
                                                         const double* __restrict__ Aem, const double* __restrict__ p,
                                                         double* __restrict__ q, double* pq) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  double en = 0.0;
  if (e < E) {
    int g[6];
    double x[6], acc[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      g[i] = __ldg(conn + (size_t)e * 6 + i);
      x[i] = g[i] >= 0 ? __ldg(p + g[i]) : 0.0;
      acc[i] = 0.0;
    }
    int k = 0;
#pragma unroll
    for (int r = 0; r < 6; ++r)
#pragma unroll
      for (int c2 = 0; c2 <= r; ++c2) {
        const double a = __ldg(Aem + (size_t)(k++) * E + e);
        acc[r] = fma(a, x[c2], acc[r]);
        if (c2 != r) acc[c2] = fma(a, x[r], acc[c2]);
      }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      en = fma(x[i], acc[i], en);
      if (g[i] >= 0) atomicAdd(q + g[i], acc[i]);
    }
  }
  __shared__ double sh[4];
  en = cw_sum(en);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = en;
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(pq, sh[0] + sh[1] + sh[2] + sh[3]);
}

// per line: x += alpha p, r -= alpha q (alpha = z.r / p.q), then z = T^-1 r; ||r||^2 and z.r
__global__ void k_line_axpy_solve(int nlines, const int64_t* __restrict__ loff, const int32_t* __restrict__ lnode,
                                  const double* __restrict__ ta, const double* __restrict__ tinv,
                                  const double* __restrict__ tc, double* __restrict__ x, double* __restrict__ r,
                                  const double* __restrict__ p, const double* __restrict__ q, double* __restrict__ z,
                                  double* cs, const int32_t* __restrict__ aggl, double* __restrict__ rc) {
  const double alpha = cs[CS_ZR_OLD] / cs[CS_PQ];
  double s0 = 0.0, s1 = 0.0;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nlines; l += gridDim.x * blockDim.x) {
    const int64_t b = loff[l], e = loff[l + 1];
    double d = 0.0, rsum = 0.0;
    for (int64_t t = b; t < e; ++t) {
      const int32_t g = lnode[t];
      x[g] = fma(alpha, p[g], x[g]);
      const double rg = fma(-alpha, q[g], r[g]);
      r[g] = rg;
      s1 = fma(rg, rg, s1);
      rsum += rg;
      d = (rg - ta[t] * d) * tinv[t];
      z[g] = d;
    }
    if (aggl) atomicAdd(rc + aggl[l], rsum);   // P_a^T r
    double xx = 0.0;
    for (int64_t t = e - 1; t >= b; --t) {
      const int32_t g = lnode[t];
      xx = z[g] - tc[t] * xx;
      z[g] = xx;
      s0 = fma(xx, r[g], s0);
    }
  }
  __shared__ double sh0[32], sh1[32];
  s0 = cw_sum(s0);
  s1 = cw_sum(s1);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    sh0[w] = s0;
    sh1[w] = s1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      a += sh0[i];
      b += sh1[i];
    }
    atomicAdd(cs + CS_ZR_NEW, a);
    atomicAdd(cs + CS_RR, b);
  }
}

// p = z + beta p (beta = z.r_new / z.r_old), q = 0 for the next apply; the last block to finish
// shifts z.r, counts the iteration, zeroes the reduction slots and sets the WHILE condition
__global__ void k_coarse_update(int64_t n, double* __restrict__ p, const double* __restrict__ z,
                                double* __restrict__ q, double* cs, unsigned int* done, double maxit,
                                cudaGraphConditionalHandle h, int use_h, const int32_t* __restrict__ aggn,
                                const double* __restrict__ zc, double* __restrict__ rc, int nagg) {
  const double beta = cs[CS_ZR_NEW] / cs[CS_ZR_OLD];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double zi = z[i];
    if (aggn) {   // z = T^-1 r + P_a z_a
      const int32_t a = aggn[i];
      if (a >= 0) zi += zc[a];
      if (i < nagg) rc[i] = 0.0;   // the next iteration's restriction accumulates from 0
    }
    p[i] = fma(beta, p[i], zi);
    q[i] = 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done, 1u) == gridDim.x - 1) {  // every block has read beta
      __threadfence();
      const double rr = cs[CS_RR];
      cs[CS_ZR_OLD] = cs[CS_ZR_NEW];
      cs[CS_IT] += 1.0;
      cs[CS_TOTAL] += 1.0;
      const unsigned go = (rr > cs[CS_THR2] && cs[CS_IT] < maxit) ? 1u : 0u;
      cs[CS_PQ] = 0.0;
      cs[CS_RR] = 0.0;
      cs[CS_ZR_NEW] = 0.0;
      cs[CS_RR_DUP] = 0.0;
      *done = 0u;
      cs[CS_GO] = go;
      if (use_h) cudaGraphSetConditional(h, go);
    }
  }
}

// ---- two-level correction kernels
// rc[aggn[i]] += r[i] (free nodes)
__global__ void k_agg_restrict(int64_t n, const int32_t* __restrict__ aggn, const double* __restrict__ r,
                               double* __restrict__ rc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = aggn[i];
    if (a >= 0) atomicAdd(rc + a, r[i]);
  }
}

// zc = A_a^-1 rc (one warp per row of the symmetric inverse); zr += zc . rc
__global__ void k_agg_solve(int na, const double* __restrict__ Ainv, const double* __restrict__ rc,
                            double* __restrict__ zc, double* zr) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= na) return;
  const double* a = Ainv + (int64_t)row * na;
  double s = 0.0;
  for (int j = lane; j < na; j += 32) s = fma(a[j], rc[j], s);
  s = cw_sum(s);
  if (lane == 0) {
    zc[row] = s;
    atomicAdd(zr, s * rc[row]);
  }
}

// z[i] += zc[aggn[i]]
__global__ void k_agg_prolong_add(int64_t n, const int32_t* __restrict__ aggn, const double* __restrict__ zc,
                                  double* __restrict__ z) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = aggn[i];
    if (a >= 0) z[i] += zc[a];
  }
}

// A_a[aggn[i]][aggn[j]] += A_e[i][j] for the free nodes of P = 1 elements e0 .. e0+ne (setup)
__global__ void k_agg_assemble(int ne, const int32_t* __restrict__ conn, const double* __restrict__ Ae,
                               const int32_t* __restrict__ aggn, int na, double* __restrict__ Aa) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)ne * 36) return;
  const int64_t e = idx / 36;
  const int i = (int)(idx % 36) / 6, j = (int)(idx % 6);
  const int32_t gi = conn[e * 6 + i], gj = conn[e * 6 + j];
  if (gi < 0 || gj < 0) return;
  atomicAdd(Aa + (int64_t)aggn[gi] * na + aggn[gj], Ae[idx]);
}

// z += P_a A_a^-1 P_a^T r and zr += (P_a^T r) . (A_a^-1 P_a^T r); leaves rc = 0
static void agg_correct(sem_ctx* c, const double* r, double* z, double* zr) {
  Coarse& C = c->C;
  const int64_t n = c->L.back().n;
  k_agg_restrict<<<cgrid(n, 256), 256, 0, c->stream>>>(n, C.aggn, r, C.rc);
  k_agg_solve<<<(C.nagg + 7) / 8, 256, 0, c->stream>>>(C.nagg, C.Aagg_inv, C.rc, C.zc, zr);
  k_agg_prolong_add<<<cgrid(n, 256), 256, 0, c->stream>>>(n, C.aggn, C.zc, z);
  CUDA_CHECK(cudaGetLastError());
  CUDA_CHECK(cudaMemsetAsync(C.rc, 0, sizeof(double) * C.nagg, c->stream));
  c->launches += 3;
}

static void line_solve(sem_ctx* c, const double* r, double* z, double* out2) {
  Coarse& C = c->C;
  const int gb = cgrid(C.nlines, 128);
  k_line_solve<<<gb, 128, 0, c->stream>>>(C.nlines, C.loff, C.lnode, C.ta, C.tinv, C.tc, r, z, out2, c->det.part);
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
  if (c->det.part) det_finalize(c, gb, out2, out2 + 1);
}

// ---------------------------------------------------------------- setup
// Lines of the P=1 level (host) and their Thomas factors from the assembled diagonal and
// vertical off-diagonals.  conn: [E][6] level ids; dir: Dirichlet mask; diag, off on the device.
void setup_coarse_lines(sem_ctx* c, const std::vector<int32_t>& conn, const std::vector<uint8_t>& dir,
                        const double* d_diag, const double* d_off) {
  Coarse& C = c->C;
  const int64_t n = (int64_t)dir.size();
  const int64_t E = (int64_t)conn.size() / 6;
  std::vector<int32_t> up(n, -1), down(n, -1);
  bool consistent = true;
  for (int64_t e = 0; e < E && consistent; ++e)
    for (int m = 0; m < 3; ++m) {
      const int32_t i = conn[e * 6 + m], j = conn[e * 6 + m + 3];
      if (dir[i] || dir[j]) continue;
      if ((up[i] >= 0 && up[i] != j) || (down[j] >= 0 && down[j] != i)) {
        consistent = false;
        break;
      }
      up[i] = j;
      down[j] = i;
    }
  std::vector<double> diag(n), off(n);
  CUDA_CHECK(cudaMemcpy(diag.data(), d_diag, n * 8, cudaMemcpyDeviceToHost));
  CUDA_CHECK(cudaMemcpy(off.data(), d_off, n * 8, cudaMemcpyDeviceToHost));
  std::vector<int64_t> loff{0};
  std::vector<int32_t> lnode;
  std::vector<double> ta, tinv, tc;
  lnode.reserve(n);
  for (int64_t s = 0; s < n; ++s) {
    if (dir[s] || (consistent && down[s] >= 0)) continue;  // line starts: free nodes with nothing below
    double cprev = 0.0, aprev = 0.0;
    int64_t t0 = (int64_t)lnode.size();
    for (int32_t g = (int32_t)s; g >= 0; g = consistent ? up[g] : -1) {
      const bool first = (int64_t)lnode.size() == t0;
      const double a = first ? 0.0 : aprev;               // A[g][below]
      const double den = diag[g] - a * cprev;
      if (!(den > 0.0)) throw SemError(SEM_ESINGULAR, "coarse line block is not SPD");
      const int32_t nx = consistent ? up[g] : -1;
      const double cg = nx >= 0 ? off[g] : 0.0;            // A[g][above]
      lnode.push_back(g);
      ta.push_back(a);
      tinv.push_back(1.0 / den);
      tc.push_back(cg / den);
      cprev = cg / den;
      aprev = cg;
    }
    loff.push_back((int64_t)lnode.size());
  }
  int64_t nfree = 0;
  for (int64_t i = 0; i < n; ++i) nfree += !dir[i];
  if ((int64_t)lnode.size() != nfree) throw SemError(SEM_EINVAL, "coarse lines do not cover the free nodes");
  C.nlines = (int)(loff.size() - 1);
  C.line_max = 0;
  for (int l = 0; l < C.nlines; ++l) C.line_max = std::max<int64_t>(C.line_max, loff[l + 1] - loff[l]);
  C.loff = upload(c, loff);
  C.lnode = upload(c, lnode);
  C.ta = upload(c, ta);
  C.tinv = upload(c, tinv);
  C.tc = upload(c, tc);
  // aggregates of the two-level correction (reading O44): RCB of the lines' (x, y)
  C.nagg = 0;
  const int want = c->opts.coarse_agg < 0 ? (C.nlines >= 4096 ? std::min(1024, C.nlines / 32) : 0)
                                          : std::min(c->opts.coarse_agg, C.nlines);
  const std::vector<double>& xyz = c->L.back().xyz;
  if (want > 0 && !c->opts.deterministic && (int64_t)xyz.size() == 3 * n) {
    std::vector<double> lx(C.nlines), ly(C.nlines);
    for (int l = 0; l < C.nlines; ++l) {
      const int32_t g = lnode[loff[l]];
      lx[l] = xyz[3 * (size_t)g];
      ly[l] = xyz[3 * (size_t)g + 1];
    }
    std::vector<int> al = partition_columns(lx, ly, want);   // equal-(x, y) lines stay together
    std::vector<int> used(want, -1);
    int na = 0;
    for (int& a : al) {   // compact (an RCB part can be empty when lines share (x, y))
      if (used[a] < 0) used[a] = na++;
      a = used[a];
    }
    std::vector<int32_t> aggl(al.begin(), al.end()), aggn(n, -1);
    for (int l = 0; l < C.nlines; ++l)
      for (int64_t t = loff[l]; t < loff[l + 1]; ++t) aggn[lnode[t]] = aggl[l];
    C.nagg = na;
    C.aggl = upload(c, aggl);
    C.aggn = upload(c, aggn);
    C.rc = dalloc<double>(c, na);
    C.zc = dalloc<double>(c, na);
    CUDA_CHECK(cudaMemset(C.rc, 0, na * sizeof(double)));
  }
  C.cs = dalloc<double>(c, CS_N);
  CUDA_CHECK(cudaMemset(C.cs, 0, CS_N * sizeof(double)));
  C.done = dalloc<unsigned int>(c, 1);
  CUDA_CHECK(cudaMemset(C.done, 0, sizeof(unsigned int)));
  CUDA_CHECK(cudaMemset(C.z, 0, n * sizeof(double)));
}

int coarse_agg_count(const sem_ctx* c) { return c->C.nagg; }

// A_a = P_a^T A P_a from the P = 1 element matrices and its dense inverse (cuSOLVER, setup only)
void setup_coarse_agg(sem_ctx* c, const double* d_D, void* cusolver_handle) {
  Coarse& C = c->C;
  if (!C.nagg) return;
  cusolverDnHandle_t sol = (cusolverDnHandle_t)cusolver_handle;
  const int li = (int)c->L.size() - 1;
  DeviceLevel& L = c->L[li];
  const int na = C.nagg, E = c->E;
  C.Aagg_inv = dalloc<double>(c, (size_t)na * na);
  CUDA_CHECK(cudaMemsetAsync(C.Aagg_inv, 0, (size_t)na * na * 8, c->stream));
  Scratch sc;
  const int64_t chunk = std::min<int64_t>(E, 1 << 20);
  double* Ae = sc.get<double>((size_t)chunk * 36);
  for (int64_t e0 = 0; e0 < E; e0 += chunk) {
    const int ne = (int)std::min<int64_t>(chunk, E - e0);
    launch_elem_matrices(c, li, d_D, Ae, (int)e0, ne);
    k_agg_assemble<<<(int)((ne * 36 + 255) / 256), 256, 0, c->stream>>>(ne, L.conn + (size_t)e0 * 6, Ae, C.aggn, na,
                                                                          C.Aagg_inv);
    CUDA_CHECK(cudaGetLastError());
  }
  int lwork = 0, lwork2 = 0;
  if (cusolverDnDpotrf_bufferSize(sol, CUBLAS_FILL_MODE_LOWER, na, C.Aagg_inv, na, &lwork) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDpotri_bufferSize(sol, CUBLAS_FILL_MODE_LOWER, na, C.Aagg_inv, na, &lwork2) != CUSOLVER_STATUS_SUCCESS)
    throw SemError(SEM_ECUDA, "cusolverDn buffer size (aggregate coarse space)");
  double* work = sc.get<double>(std::max(lwork, lwork2));
  int* dinfo = sc.get<int>(1);
  int hinfo = 0;
  if (cusolverDnDpotrf(sol, CUBLAS_FILL_MODE_LOWER, na, C.Aagg_inv, na, work, lwork, dinfo) != CUSOLVER_STATUS_SUCCESS)
    throw SemError(SEM_ECUDA, "cusolverDnDpotrf (aggregate coarse space)");
  CUDA_CHECK(cudaMemcpyAsync(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
  if (hinfo != 0) throw SemError(SEM_ESINGULAR, "aggregate coarse matrix is not SPD (info " + std::to_string(hinfo) + ")");
  if (cusolverDnDpotri(sol, CUBLAS_FILL_MODE_LOWER, na, C.Aagg_inv, na, work, lwork2, dinfo) != CUSOLVER_STATUS_SUCCESS)
    throw SemError(SEM_ECUDA, "cusolverDnDpotri (aggregate coarse space)");
  CUDA_CHECK(cudaMemcpyAsync(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
  if (hinfo != 0) throw SemError(SEM_ESINGULAR, "aggregate coarse inverse failed (info " + std::to_string(hinfo) + ")");
  launch_symmetrize(c, C.Aagg_inv, na);
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
}

void launch_offdiag_accum(sem_ctx* c, const int32_t* conn, int ne, const double* Ae, double* off) {
  const int64_t tot = (int64_t)ne * 3;
  k_offdiag_accum<<<(int)((tot + 255) / 256), 256, 0, c->stream>>>(ne, conn, Ae, off);
  CUDA_CHECK(cudaGetLastError());
}

// ---------------------------------------------------------------- solve
// prologue: x = 0, r = b (free nodes), z = T^-1 r, p = z; ||b||^2, z.r; the stop threshold and the
// first loop condition (graph handle h when use_h, and cs[CS_GO] always)
static void coarse_prologue(sem_ctx* c, const double* b, double* x, cudaGraphConditionalHandle h, int use_h) {
  const int li = (int)c->L.size() - 1;
  const DeviceLevel& L = c->L[li];
  Coarse& C = c->C;
  double* cs = C.cs;
  k_zero_slots<<<1, 1, 0, c->stream>>>(cs, CS_ZR_NEW, CS_RR_DUP, -1, -1);
  launch_init_masked(c, li, nullptr, x, 1);
  launch_init_masked(c, li, b, C.r, 1);
  line_solve(c, C.r, C.z, cs + CS_ZR_NEW);  // [ZR_NEW] = z.r, [RR_DUP] = r.r
  if (C.nagg) agg_correct(c, C.r, C.z, cs + CS_ZR_NEW);
  launch_xpby(c, L.n, C.p, C.z, nullptr, nullptr, 1);
  launch_init_masked(c, li, nullptr, C.q, 1);   // q = 0 (the fused body re-zeroes it every iteration)
  const double rt = c->opts.coarse_rtol;
  k_coarse_start<<<1, 1, 0, c->stream>>>(cs, rt * rt, h, use_h);
  CUDA_CHECK(cudaGetLastError());
  c->launches += 2;
}

// one CG iteration; the last kernel sets the loop condition
static void coarse_body(sem_ctx* c, double* x, cudaGraphConditionalHandle h, int use_h) {
  const int li = (int)c->L.size() - 1;
  const DeviceLevel& L = c->L[li];
  Coarse& C = c->C;
  const int64_t n = L.n;
  double* cs = C.cs;
  const double maxit = (double)c->opts.coarse_maxit;
  if (L.Ae1 && !c->det.on && L.N == 6) {
    // fused: [q = A p, p.q] -> [x, r update, z = T^-1 r, ||r||^2, z.r] -> [p = z + beta p, q = 0, stop test]
    const int E = c->E;
    k_coarse_apply_pq<<<(E + 127) / 128, 128, 0, c->stream>>>(E, L.conn, L.Ae1, C.p, C.q, cs + CS_PQ);
    k_line_axpy_solve<<<cgrid(C.nlines, 128), 128, 0, c->stream>>>(C.nlines, C.loff, C.lnode, C.ta, C.tinv, C.tc,
                                                                   x, C.r, C.p, C.q, C.z, cs, C.aggl, C.rc);
    if (C.nagg)   // z_a = A_a^-1 P_a^T r (rc accumulated by the line kernel), z.r += z_a . rc
      k_agg_solve<<<(C.nagg + 7) / 8, 256, 0, c->stream>>>(C.nagg, C.Aagg_inv, C.rc, C.zc, cs + CS_ZR_NEW);
    k_coarse_update<<<cgrid(n, 256), 256, 0, c->stream>>>(n, C.p, C.z, C.q, cs, C.done, maxit, h, use_h, C.aggn,
                                                          C.zc, C.rc, C.nagg);
    CUDA_CHECK(cudaGetLastError());
    c->launches += C.nagg ? 4 : 3;
    return;
  }
  // q = A p; p.q; x += alpha p, r -= alpha q (||r||^2); z = T^-1 r (z.r); p = z + beta p; stop test
  launch_init_masked(c, li, nullptr, C.q, 1);
  launch_apply(c, li, C.p, C.q, 0);
  launch_dot2(c, n, C.p, C.q, nullptr, nullptr, nullptr, cs + CS_PQ, false);
  launch_axpy_pcg(c, n, x, C.r, C.p, C.q, cs + CS_ZR_OLD, cs + CS_PQ, cs + CS_RR, nullptr, false);
  line_solve(c, C.r, C.z, cs + CS_ZR_NEW);
  if (C.nagg) agg_correct(c, C.r, C.z, cs + CS_ZR_NEW);
  launch_xpby(c, n, C.p, C.z, cs + CS_ZR_NEW, cs + CS_ZR_OLD, 0);
  k_coarse_next<<<1, 1, 0, c->stream>>>(cs, maxit, h, use_h);
  CUDA_CHECK(cudaGetLastError());
  c->launches++;
}

// Enqueue the whole PCG on c->stream, which must be capturing: prologue, then a conditional
// WHILE node whose body (one CG iteration) is captured through a second stream.  x = A_1^-1 b
// from x = 0.  The body's kernels are counted per executed iteration (coarse_count_launches).
static void emit_coarse_pcg(sem_ctx* c, const double* b, double* x) {
  Coarse& C = c->C;
  cudaStreamCaptureStatus st;
  cudaGraph_t graph = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  CUDA_CHECK(cudaStreamGetCaptureInfo(c->stream, &st, nullptr, &graph, &deps, &ndeps));
  if (st != cudaStreamCaptureStatusActive) throw SemError(SEM_ECUDA, "coarse PCG emitted outside a capture");
  cudaGraphConditionalHandle h;
  CUDA_CHECK(cudaGraphConditionalHandleCreate(&h, graph, 0, cudaGraphCondAssignDefault));
  coarse_prologue(c, b, x, h, 1);
  CUDA_CHECK(cudaStreamGetCaptureInfo(c->stream, &st, nullptr, &graph, &deps, &ndeps));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CUDA_CHECK(cudaGraphAddNode(&node, graph, deps, ndeps, &cp));
  CUDA_CHECK(cudaStreamUpdateCaptureDependencies(c->stream, &node, 1, cudaStreamSetCaptureDependencies));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  if (!C.body_stream) CUDA_CHECK(cudaStreamCreateWithFlags(&C.body_stream, cudaStreamNonBlocking));
  CUDA_CHECK(cudaStreamBeginCaptureToGraph(C.body_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  cudaStream_t keep = c->stream;
  c->stream = C.body_stream;
  const int64_t l0 = c->launches;
  try {
    coarse_body(c, x, h, 1);
  } catch (...) {
    c->stream = keep;
    cudaGraph_t g2;
    cudaStreamEndCapture(C.body_stream, &g2);
    throw;
  }
  C.body_launches = c->launches - l0;
  c->launches = l0;
  c->stream = keep;
  cudaGraph_t g2 = nullptr;
  CUDA_CHECK(cudaStreamEndCapture(C.body_stream, &g2));
}

static bool no_graphs() {
  static const int off = [] {
    const char* e = getenv("SEM_NO_GRAPHS");
    return (e && atoi(e)) ? 1 : 0;
  }();
  return off != 0;
}

void coarse_pcg(sem_ctx* c, const double* b, double* x) {
  Coarse& C = c->C;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  CUDA_CHECK(cudaStreamIsCapturing(c->stream, &st));
  if (st == cudaStreamCaptureStatusActive) {
    emit_coarse_pcg(c, b, x);
    return;
  }
  if (no_graphs()) {  // SEM_NO_GRAPHS=1 (profiling): host-driven loop, one condition read per iteration
    coarse_prologue(c, b, x, 0, 0);
    for (;;) {
      double go = 0.0;
      CUDA_CHECK(cudaMemcpyAsync(&go, C.cs + CS_GO, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CUDA_CHECK(cudaStreamSynchronize(c->stream));
      if (go == 0.0) break;
      coarse_body(c, x, 0, 0);
    }
    return;
  }
  // eager: replay the solve's own graph on the coarsest level's buffers
  const int li = (int)c->L.size() - 1;
  DeviceLevel& L = c->L[li];
  if (!C.exec) {
    if (!C.cap_stream) CUDA_CHECK(cudaStreamCreateWithFlags(&C.cap_stream, cudaStreamNonBlocking));
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
    cudaStream_t keep = c->stream;
    c->stream = C.cap_stream;
    const int64_t l0 = c->launches;
    cudaGraph_t g = nullptr;
    CUDA_CHECK(cudaStreamBeginCapture(C.cap_stream, cudaStreamCaptureModeThreadLocal));
    try {
      emit_coarse_pcg(c, L.f, L.u);
    } catch (...) {
      cudaStreamEndCapture(C.cap_stream, &g);
      if (g) cudaGraphDestroy(g);
      c->stream = keep;
      throw;
    }
    CUDA_CHECK(cudaStreamEndCapture(C.cap_stream, &g));
    c->stream = keep;
    C.exec_launches = c->launches - l0;
    c->launches = l0;
    CUDA_CHECK(cudaGraphInstantiate(&C.exec, g, 0));
    CUDA_CHECK(cudaGraphDestroy(g));
  }
  if (b != L.f) CUDA_CHECK(cudaMemcpyAsync(L.f, b, L.n * 8, cudaMemcpyDeviceToDevice, c->stream));
  CUDA_CHECK(cudaGraphLaunch(C.exec, c->stream));
  c->launches += C.exec_launches;
  if (x != L.u) CUDA_CHECK(cudaMemcpyAsync(x, L.u, L.n * 8, cudaMemcpyDeviceToDevice, c->stream));
}

// graph-replayed WHILE bodies: add the kernels of the `iters` executed iterations to the count
void coarse_count_launches(sem_ctx* c, int64_t iters) {
  if (c->C.iterative && !no_graphs()) c->launches += iters * c->C.body_launches;
}

// total inner iterations since the last reset (synchronises the stream)
int64_t coarse_iters(sem_ctx* c, bool reset) {
  if (!c->C.iterative || !c->C.cs) return 0;
  double v = 0.0;
  CUDA_CHECK(cudaMemcpyAsync(&v, c->C.cs + CS_TOTAL, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
  if (reset) CUDA_CHECK(cudaMemsetAsync(c->C.cs + CS_TOTAL, 0, sizeof(double), c->stream));
  return (int64_t)v;
}

void coarse_reset_iters(sem_ctx* c) {
  if (c->C.iterative && c->C.cs) CUDA_CHECK(cudaMemsetAsync(c->C.cs + CS_TOTAL, 0, sizeof(double), c->stream));
}

void coarse_destroy(sem_ctx* c) {
  Coarse& C = c->C;
  if (C.exec) cudaGraphExecDestroy(C.exec);
  if (C.cap_stream) cudaStreamDestroy(C.cap_stream);
  if (C.body_stream) cudaStreamDestroy(C.body_stream);
  C.exec = nullptr;
  C.cap_stream = C.body_stream = nullptr;
}

}  // namespace sem
