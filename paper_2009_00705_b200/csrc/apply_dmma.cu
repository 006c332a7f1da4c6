// Operator apply on FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64) for sm_100a.
//
// Same mathematics as k_apply<P> in kernels.cu (eq 3.8: y (+/-)=
// sum_e Q_e^T D^T (G (.) D Q_e u) with D = [B_r (x) B_t ; B_s (x) B_t ; B_0 (x) D_t]),
// reorganised as four batched small GEMMs per batch of NE elements:
//
//   stage 1  U_c  [a][j]   = sum_m  B_c[a][m] u[m][j]          (j = e*N1 + l)
//   stage 2  g_c^T[q][a]   = sum_l  M_c[q][l] U_c[a][e*N1+l]   (M = B_t for r,s; D_t for t)
//   stage 3  w = G g        pointwise, in the stage-2 accumulator registers
//   stage 4  V_c^T[l][a]   = sum_q  M_c[q][l] w_c[q][a]
//   stage 5  y_c  [m][j]   = sum_a  B_c[a][m] V_c[a][j],   y = y_r + y_s + y_0
//
// The geometric factors of the batch (NE * 6 * Q doubles, contiguous) are staged
// into shared memory with one TMA bulk copy (cp.async.bulk + mbarrier) issued at
// kernel entry, overlapping the gather and stages 1-2.  Reference-matrix operands
// are pre-arranged on the host in fragment order ([...][lane]) and live in
// registers.  Fragment layouts (PTX ISA, mma.m8n8k4 .f64):
//   A (8x4):  a0 = A[lane>>2][lane&3]
//   B (4x8):  b0 = B[lane&3][lane>>2]
//   C (8x8):  c_i = C[lane>>2][2*(lane&3)+i]
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>

#include "internal.h"

namespace sem {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__host__ __device__ constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }
// smallest y >= x with y % 8 == 4: rows of a fragment read (4 rows x 4 columns per half-warp)
// then start in distinct 8-word bank groups
__host__ __device__ constexpr int pad4(int x) { return x + ((4 - x % 8) + 8) % 8; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

// tuning: elements per batch NE_, warps per CTA W_, reference fragments in shared memory FS_
template <int P, int NE_ = 0, int W_ = 16, int FS_ = -1>
struct MD {
  static constexpr int N1 = P + 1, NT = N1 * (N1 + 1) / 2, N = NT * N1, QT = N1 * N1, QV = N1, Q = QT * QV;
  static constexpr int NE = NE_ ? NE_ : ((P == 1) ? 16 : (P <= 3 ? 8 : (P <= 5 ? 4 : 2)));
  static constexpr bool FS = FS_ >= 0 ? (FS_ == 1) : (P <= 5);
  static constexpr int JW = N1 * NE;                    // stage-1/5 columns (e, l)
  static constexpr int NJT = cdiv(JW, 8);               // n-tiles over j
  static constexpr int MT1 = cdiv(QT, 8);               // m-tiles over a (stage 1), n-tiles over a (2, 4)
  static constexpr int KT1 = cdiv(NT, 4);               // k-steps over m (stage 1)
  static constexpr int MTV = cdiv(QV, 8);               // m-tiles over q (stage 2)
  static constexpr int KTV = cdiv(N1, 4);               // k-steps over l (stage 2)
  static constexpr int MT4 = cdiv(N1, 8);               // m-tiles over l (stage 4)
  static constexpr int KT4 = cdiv(QV, 4);               // k-steps over q (stage 4)
  static constexpr int MT5 = cdiv(NT, 8);               // m-tiles over m (stage 5)
  static constexpr int KT5 = cdiv(QT, 4);               // k-steps over a per component (stage 5)
  // shared-memory strides (doubles); row counts padded for fragment reads
  static constexpr int SU = pad4(8 * NJT);                               // su [4*KT1][SU]
  static constexpr int SUO = pad4(cmax(8 * NJT, (NE - 1) * N1 + 4 * KTV)); // sU [3][8*MT1][SUO]
  static constexpr int SA = pad4(8 * MT1);                               // sW [3][NE][RW][SA]
  static constexpr int RW = cmax(8 * MTV, 4 * KT4);                      // rows q of sW
  static constexpr int RV = cmax(4 * KT5, 8 * MT1);                      // rows a of sV
  static constexpr int SV = pad4(cmax(8 * NJT, (NE - 1) * N1 + 8 * MT4)); // sV [3][RV][SV], sY [3][8*MT5][SV]
  static constexpr int SZ_U = 4 * KT1 * SU;
  static constexpr int SZ_UO = 3 * 8 * MT1 * SUO;
  static constexpr int SZ_V = 3 * RV * SV;
  static constexpr int SZ_Y = 3 * 8 * MT5 * SV;
  static constexpr int SZ_W = 3 * NE * RW * SA;
  static constexpr int SZ_G = NE * 6 * Q;
  // regions: [su][X = sU | sV][Wr = sW | sY][G]
  static constexpr int SZ_X = cmax(SZ_UO, SZ_V);
  static constexpr int SZ_WR = cmax(SZ_W, SZ_Y);
  static constexpr int WARPS = W_, T = 32 * WARPS;
  // fragment arrays (doubles): F1 [3][MT1][KT1][32], FV [2][MTV][KTV][32], F4 [2][MT4][KT4][32], F5 [3][MT5][KT5][32]
  static constexpr int OFF_F1 = 0;
  static constexpr int OFF_FV = OFF_F1 + 3 * MT1 * KT1 * 32;
  static constexpr int OFF_F4 = OFF_FV + 2 * MTV * KTV * 32;
  static constexpr int OFF_F5 = OFF_F4 + 2 * MT4 * KT4 * 32;
  static constexpr int FRAG_DOUBLES = OFF_F5 + 3 * MT5 * KT5 * 32;
  // persistent layout: [fragments if FS][su][X][Wr][G][mbarrier]
  static constexpr int SMEM = ((FS ? FRAG_DOUBLES : 0) + SZ_U + SZ_X + SZ_WR + SZ_G) * 8 + 16;
  static_assert(SMEM <= 227 * 1024, "apply_dmma shared memory exceeds 227 KB");
};

// host: fragment-ordered reference operands for order p
std::vector<double> dmma_fragments(const LevelRef& R) {
  const int p = R.p;
  auto run = [&](auto tag) {
    using D = MD<decltype(tag)::value, 1, 8, 0>;  // fragment layout does not depend on NE/W/FS
    std::vector<double> f(D::FRAG_DOUBLES, 0.0);
    const double* Bc[3] = {R.Br.data(), R.Bs.data(), R.B0.data()};  // [qt][nt]
    for (int c = 0; c < 3; ++c)
      for (int mt = 0; mt < D::MT1; ++mt)
        for (int kt = 0; kt < D::KT1; ++kt)
          for (int ln = 0; ln < 32; ++ln) {
            int a = 8 * mt + (ln >> 2), m = 4 * kt + (ln & 3);
            f[D::OFF_F1 + ((c * D::MT1 + mt) * D::KT1 + kt) * 32 + ln] =
                (a < D::QT && m < D::NT) ? Bc[c][a * D::NT + m] : 0.0;
          }
    const double* Mv[2] = {R.Bt.data(), R.Dt.data()};  // [qv][n1]
    for (int v = 0; v < 2; ++v) {
      for (int mt = 0; mt < D::MTV; ++mt)
        for (int kt = 0; kt < D::KTV; ++kt)
          for (int ln = 0; ln < 32; ++ln) {  // A = M[q][l]
            int q = 8 * mt + (ln >> 2), l = 4 * kt + (ln & 3);
            f[D::OFF_FV + ((v * D::MTV + mt) * D::KTV + kt) * 32 + ln] =
                (q < D::QV && l < D::N1) ? Mv[v][q * D::N1 + l] : 0.0;
          }
      for (int mt = 0; mt < D::MT4; ++mt)
        for (int kt = 0; kt < D::KT4; ++kt)
          for (int ln = 0; ln < 32; ++ln) {  // A = M^T[l][q]
            int l = 8 * mt + (ln >> 2), q = 4 * kt + (ln & 3);
            f[D::OFF_F4 + ((v * D::MT4 + mt) * D::KT4 + kt) * 32 + ln] =
                (q < D::QV && l < D::N1) ? Mv[v][q * D::N1 + l] : 0.0;
          }
    }
    for (int c = 0; c < 3; ++c)
      for (int mt = 0; mt < D::MT5; ++mt)
        for (int kt = 0; kt < D::KT5; ++kt)
          for (int ln = 0; ln < 32; ++ln) {  // A = B_c^T[m][a]
            int m = 8 * mt + (ln >> 2), a = 4 * kt + (ln & 3);
            f[D::OFF_F5 + ((c * D::MT5 + mt) * D::KT5 + kt) * 32 + ln] =
                (a < D::QT && m < D::NT) ? Bc[c][a * D::NT + m] : 0.0;
          }
    return f;
  };
  switch (p) {
    case 1: return run(std::integral_constant<int, 1>{});
    case 2: return run(std::integral_constant<int, 2>{});
    case 3: return run(std::integral_constant<int, 3>{});
    case 4: return run(std::integral_constant<int, 4>{});
    case 5: return run(std::integral_constant<int, 5>{});
    case 6: return run(std::integral_constant<int, 6>{});
    case 7: return run(std::integral_constant<int, 7>{});
    case 8: return run(std::integral_constant<int, 8>{});
  }
  return {};
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int P, int NE_, int W_, int FS_>
__global__ void __launch_bounds__(32 * W_, 1) k_apply_dmma(int E, int nbatch, const int32_t* __restrict__ conn,
                                                           const double* __restrict__ G,
                                                           const double* __restrict__ frag,
                                                           const double* __restrict__ u, double* __restrict__ y,
                                                           int flags) {
  using D = MD<P, NE_, W_, FS_>;
  extern __shared__ __align__(128) double sm[];
  // persistent single-buffer pipeline: [F][su][X][Wr][G][mbar].  su is refilled
  // (cp.async gather) as soon as stage 1 has consumed it, G (TMA bulk copy) as
  // soon as stage 3 has consumed it, so both loads overlap the remaining stages.
  double* sF = sm;
  double* su = sF + (D::FS ? D::FRAG_DOUBLES : 0);
  double* sX = su + D::SZ_U;
  double* sWr = sX + D::SZ_X;
  double* sG = sWr + D::SZ_WR;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sG + D::SZ_G);
  const double* F = D::FS ? sF : frag;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int IT = (D::NE * D::N + D::T - 1) / D::T;  // gather/scatter items per thread

  if (D::FS)
    for (int i = tid; i < D::FRAG_DOUBLES; i += D::T) sF[i] = __ldg(frag + i);
  for (int i = tid; i < D::SZ_U + D::SZ_X + D::SZ_WR; i += D::T) su[i] = 0.0;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue_G = [&](int b) {  // one thread: TMA bulk copy of batch b's geometric factors
    const int e0 = b * D::NE, ne = min(D::NE, E - e0);
    const uint32_t bytes = (uint32_t)ne * 6u * D::Q * 8u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(mbar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(sG)),
        "l"(G + (size_t)e0 * 6 * D::Q), "r"(bytes), "r"(smem_addr(mbar))
        : "memory");
  };
  auto load_conn = [&](int b, int* cn) {
    const int e0 = b * D::NE, ne = min(D::NE, E - e0);
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int i = tid + k * D::T;
      cn[k] = (i < D::NE * D::N && i / D::N < ne) ? __ldg(conn + (size_t)e0 * D::N + i) : INT_MIN;
    }
  };
  auto issue_gather = [&](const int* cn) {  // cp.async u[conn] -> su
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int i = tid + k * D::T;
      if (i >= D::NE * D::N) continue;
      const int e = i / D::N, n = i % D::N, m = n % D::NT, l = n / D::NT;
      double* dst = su + m * D::SU + e * D::N1 + l;
      const int c = cn[k];
      if (c >= 0 || (c != INT_MIN && (flags & AP_GATHER_ALL))) {
        const double* s = u + (c >= 0 ? c : ~c);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(s) : "memory");
      } else {
        *dst = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  int b = blockIdx.x;
  uint32_t ph = 0;
  int cn[IT], cnn[IT];
  if (b < nbatch) {
    if (tid == 0) issue_G(b);
    load_conn(b, cn);
    issue_gather(cn);
  }
  const double sgn = (flags & AP_NEGATE) ? -1.0 : 1.0;
  for (; b < nbatch; b += gridDim.x) {
    const int bn = b + gridDim.x;
    const int ne = min(D::NE, E - b * D::NE);
    if (bn < nbatch) load_conn(bn, cnn);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    // ---- stage 1: U_c[a][j] = sum_m B_c[a][m] u[m][j]; job = (c, mt), NJT independent chains
    for (int job = warp; job < 3 * D::MT1; job += D::WARPS) {
      const int c = job / D::MT1, mt = job % D::MT1;
      const double* fa = F + D::OFF_F1 + ((c * D::MT1 + mt) * D::KT1) * 32 + lane;
      double acc[D::NJT][2];
#pragma unroll
      for (int nt = 0; nt < D::NJT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
      for (int kt = 0; kt < D::KT1; ++kt) {
        const double a = fa[kt * 32];
        const double* bs = su + (4 * kt + (lane & 3)) * D::SU + (lane >> 2);
#pragma unroll
        for (int nt = 0; nt < D::NJT; ++nt) dmma(acc[nt][0], acc[nt][1], a, bs[8 * nt]);
      }
      double* out = sX + (c * 8 * D::MT1 + 8 * mt + (lane >> 2)) * D::SUO + 2 * (lane & 3);
#pragma unroll
      for (int nt = 0; nt < D::NJT; ++nt)
        *reinterpret_cast<double2*>(out + 8 * nt) = make_double2(acc[nt][0], acc[nt][1]);
    }
    __syncthreads();
    if (bn < nbatch) issue_gather(cnn);  // su is free: next batch's gather overlaps stages 2-5
    {
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_addr(mbar)), "r"(ph)
            : "memory");
      }
      ph ^= 1;
    }
    // ---- stages 2+3: g_c^T[q][a] = sum_l M_c[q][l] U_c[a][e*N1+l]; w = G g; job = (e, nt over a)
    for (int job = warp; job < D::NE * D::MT1; job += D::WARPS) {
      const int e = job / D::MT1, nt = job % D::MT1;
#pragma unroll
      for (int mv = 0; mv < D::MTV; ++mv) {
        double g[3][2];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          g[c][0] = 0.0;
          g[c][1] = 0.0;
          const double* src = sX + (c * 8 * D::MT1 + 8 * nt + (lane >> 2)) * D::SUO + e * D::N1 + (lane & 3);
          const int v = (c < 2) ? 0 : 1;
#pragma unroll
          for (int kt = 0; kt < D::KTV; ++kt)
            dmma(g[c][0], g[c][1], F[D::OFF_FV + ((v * D::MTV + mv) * D::KTV + kt) * 32 + lane], src[4 * kt]);
        }
        const int q = 8 * mv + (lane >> 2);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int a = 8 * nt + 2 * (lane & 3) + i;
          if (q < D::QV && a < D::QT) {
            double w0 = 0.0, w1 = 0.0, w2 = 0.0;
            if (e < ne) {
              const double* gg = sG + (size_t)e * 6 * D::Q + a + D::QT * q;
              const double gxx = gg[0], gxy = gg[D::Q], gxz = gg[2 * D::Q], gyy = gg[3 * D::Q],
                           gyz = gg[4 * D::Q], gzz = gg[5 * D::Q];
              w0 = gxx * g[0][i] + gxy * g[1][i] + gxz * g[2][i];
              w1 = gxy * g[0][i] + gyy * g[1][i] + gyz * g[2][i];
              w2 = gxz * g[0][i] + gyz * g[1][i] + gzz * g[2][i];
            }
            sWr[((0 * D::NE + e) * D::RW + q) * D::SA + a] = w0;
            sWr[((1 * D::NE + e) * D::RW + q) * D::SA + a] = w1;
            sWr[((2 * D::NE + e) * D::RW + q) * D::SA + a] = w2;
          }
        }
      }
    }
    __syncthreads();
    if (bn < nbatch && tid == 0) issue_G(bn);  // sG is free: next batch's TMA overlaps stages 4-5
    // ---- stage 4: V_c^T[l][a] = sum_q M_c[q][l] w_c[q][a] -> sV[c][a][e*N1+l]; job = (c, e, nt over a)
    for (int job = warp; job < 3 * D::NE * D::MT1; job += D::WARPS) {
      const int c = job / (D::NE * D::MT1), rem = job % (D::NE * D::MT1), e = rem / D::MT1, nt = rem % D::MT1;
      const int v = (c < 2) ? 0 : 1;
      const double* src = sWr + ((c * D::NE + e) * D::RW + (lane & 3)) * D::SA + 8 * nt + (lane >> 2);
#pragma unroll
      for (int m4 = 0; m4 < D::MT4; ++m4) {
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int kt = 0; kt < D::KT4; ++kt)
          dmma(c0, c1, F[D::OFF_F4 + ((v * D::MT4 + m4) * D::KT4 + kt) * 32 + lane], src[4 * kt * D::SA]);
        const int l = 8 * m4 + (lane >> 2);
        const int a = 8 * nt + 2 * (lane & 3);
        if (l < D::N1) {
          double* o = sX + (c * D::RV + a) * D::SV + e * D::N1 + l;
          if (a < D::QT) o[0] = c0;
          if (a + 1 < D::QT) o[D::SV] = c1;
        }
      }
    }
    __syncthreads();
    // ---- stage 5: y[m][j] = sum_c sum_a B_c[a][m] V_c[a][j]; job = (mt5, nt), two accumulator chains
    for (int job = warp; job < D::MT5 * D::NJT; job += D::WARPS) {
      const int mt = job / D::NJT, nt = job % D::NJT;
      double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double* fa = F + D::OFF_F5 + ((c * D::MT5 + mt) * D::KT5) * 32 + lane;
        const double* src = sX + (c * D::RV + (lane & 3)) * D::SV + 8 * nt + (lane >> 2);
#pragma unroll
        for (int kt = 0; kt < D::KT5; ++kt) {
          if (kt & 1) dmma(d0, d1, fa[kt * 32], src[4 * kt * D::SV]);
          else dmma(c0, c1, fa[kt * 32], src[4 * kt * D::SV]);
        }
      }
      double* o = sWr + (8 * mt + (lane >> 2)) * D::SV + 8 * nt + 2 * (lane & 3);
      *reinterpret_cast<double2*>(o) = make_double2(c0 + d0, c1 + d1);
    }
    __syncthreads();
    // ---- scatter-add y = Q_e^T y_e (connectivity still in registers)
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int i = tid + k * D::T;
      const int c = cn[k];
      if (i >= D::NE * D::N || c == INT_MIN) continue;
      const int e = i / D::N, n = i % D::N, m = n % D::NT, l = n / D::NT;
      const double v = sWr[m * D::SV + e * D::N1 + l];
      if (c >= 0) atomicAdd(y + c, sgn * v);
      else if (flags & AP_SCATTER_ALL) atomicAdd(y + ~c, sgn * v);
    }
#pragma unroll
    for (int k = 0; k < IT; ++k) cn[k] = cnn[k];
    (void)ne;
  }
}

template <int P, int NE_ = 0, int W_ = 16, int FS_ = -1>
static void apply_dmma_P(sem_ctx* c, const DeviceLevel& L, const double* u, double* y, int flags) {
  using D = MD<P, NE_, W_, FS_>;
  constexpr int ne = D::NE, w = D::WARPS, fs = D::FS ? 1 : 0;
  auto kern = k_apply_dmma<P, ne, w, fs>;
  static int grid_maxes[kMaxDev] = {0};
  const int dev = cur_device();
  int& grid_max = grid_maxes[dev];
  if (!grid_max) {
    CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, D::SMEM));
    int per_sm = 0, sms = 0;
    CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, D::T, D::SMEM));
    grid_max = sms * (per_sm > 0 ? per_sm : 1);
  }
  if (c->E_own == 0) return;
  const int nbatch = (c->E_own + D::NE - 1) / D::NE;
  const int grid = nbatch < grid_max ? nbatch : grid_max;
  kern<<<grid, D::T, D::SMEM, c->stream>>>(c->E_own, nbatch, L.conn, L.G, L.frag, u, y, flags);
  CUDA_CHECK(cudaGetLastError());
}

// variant table for tuning sweeps (SEM_DMMA_VARIANT=<k>); 0 = default per order
static int dmma_variant() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("SEM_DMMA_VARIANT");
    v = s ? atoi(s) : 0;
  }
  return v;
}

void launch_apply_dmma(sem_ctx* c, int level, const double* u, double* y, int flags) {
  const DeviceLevel& L = c->L[level];
  switch (L.p) {
    case 1: apply_dmma_P<1>(c, L, u, y, flags); break;
    case 2: apply_dmma_P<2>(c, L, u, y, flags); break;
    case 3: apply_dmma_P<3>(c, L, u, y, flags); break;
    case 4:
      switch (dmma_variant()) {
        case 1: apply_dmma_P<4, 4, 8, 1>(c, L, u, y, flags); break;
        case 2: apply_dmma_P<4, 8, 16, 0>(c, L, u, y, flags); break;
        case 3: apply_dmma_P<4, 2, 8, 1>(c, L, u, y, flags); break;
        default: apply_dmma_P<4>(c, L, u, y, flags);
      }
      break;
    case 5:
      switch (dmma_variant()) {
        case 1: apply_dmma_P<5, 4, 16, 1>(c, L, u, y, flags); break;
        case 2: apply_dmma_P<5, 2, 8, 1>(c, L, u, y, flags); break;
        case 3: apply_dmma_P<5, 2, 4, 0>(c, L, u, y, flags); break;
        case 4: apply_dmma_P<5, 4, 8, 1>(c, L, u, y, flags); break;
        // r1 sweep on config 3 (tools/sweep_dmma.sh): (NE,W,FS) = (4,8,0) 446 us,
        // (4,16,1) 503 us, (2,8,1) 506 us, (2,4,0) 544 us, (4,8,1) 562 us
        default: apply_dmma_P<5, 4, 8, 0>(c, L, u, y, flags);
      }
      break;
    case 6: apply_dmma_P<6>(c, L, u, y, flags); break;
    case 7: apply_dmma_P<7>(c, L, u, y, flags); break;
    case 8:
      switch (dmma_variant()) {
        case 1: apply_dmma_P<8, 1, 8, 0>(c, L, u, y, flags); break;
        default: apply_dmma_P<8>(c, L, u, y, flags);
      }
      break;
    default: throw SemError(SEM_EINVAL, "order out of range");
  }
  c->launches++;
}

}  // namespace sem
