// Operator apply, one warp per element, on FP64 tensor cores (sm_100a DMMA).
//
// Same mathematics as k_apply<P> / k_apply_dmma<P> (eq 3.8, P:153-161:
// y (+/-)= sum_e Q_e^T D^T (G (.) D Q_e u), D = [B_r (x) B_t ; B_s (x) B_t ;
// B_0 (x) D_t]), sum-factorised vertical-first so that every stage is a small
// GEMM on mma.sync.m8n8k4.f64 with the element's data in registers:
//
//   A   Ut[m][q]  = sum_l u[m][l] Bt[q][l],   Udt[m][q] = sum_l u[m][l] Dt[q][l]
//   B   g_r[a][q] = sum_m Br[a][m] Ut[m][q],  g_s (Bs, Ut),  g_t (B0, Udt)   per a-tile
//   G   w = G g  at every cubature point (a, q)                              per a-tile
//   B^T Vt[m][q] += sum_a Br[a][m] w_r[a][q] + Bs[a][m] w_s[a][q],
//       Vdt[m][q] += sum_a B0[a][m] w_t[a][q]                                per a-tile
//   A^T y[m][l]   = sum_q Vt[m][q] Bt[q][l] + Vdt[m][q] Dt[q][l]
//
// (m: triangle node, l: vertical node, a: triangle cubature point, q: vertical
// Gauss point).  Fragment layouts of m8n8k4: A a0 = A[r4][c4], B b0 = B[c4][r4],
// C c_i = C[r4][2 c4 + i] with r4 = lane >> 2, c4 = lane & 3.  C fragments are
// re-laid out as A or B fragments of the next stage with two shuffles.
//
// Data movement: the element's geometric factors (6 Q doubles, contiguous) are
// stored a-tile-major (k_g_tiles) and streamed through a 3-slot ring per warp,
// one TMA bulk copy (cp.async.bulk + mbarrier) per a-tile issued two tiles
// ahead (across element boundaries); u is gathered into registers through
// the connectivity, y scattered with FP64 atomics.  Persistent CTAs, no CTA
// barrier after the prologue.
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>

#include "internal.h"

namespace sem {

#ifndef AW_W_SMALL
#define AW_W_SMALL 16   // warps per CTA for p <= 5
#endif
#ifndef AW_MA_UNROLL
#define AW_MA_UNROLL 1  // unroll of the a-tile loop
#endif
#define AW_PRAGMA_(x) _Pragma(#x)
#define AW_PRAGMA(x) AW_PRAGMA_(x)

namespace aw {
__host__ __device__ constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }
}  // namespace aw

template <int P>
struct AW {
  static constexpr int N1 = P + 1, NT = N1 * (N1 + 1) / 2, QT = N1 * N1, QV = N1, Q = QT * QV, N = NT * N1;
  static constexpr int MTM = aw::cdiv(NT, 8);   // m-tiles over triangle nodes
  static constexpr int KM = 2 * MTM;            // k-steps over triangle nodes (padded to 8 MTM)
  static constexpr int MTA = aw::cdiv(QT, 8);   // a-tiles over triangle cubature points
  static constexpr int NQ = aw::cdiv(QV, 8);    // n-tiles over vertical points
  static constexpr int KL = aw::cdiv(N1, 4);    // k-steps over vertical nodes
  static constexpr int NL = aw::cdiv(N1, 8);    // n-tiles over vertical nodes
  static constexpr int KQ = aw::cdiv(QV, 4);    // k-steps over vertical points
  static constexpr int LDM = 8 * MTM + 4;       // row stride of Bm (= 4 mod 8: conflict-free both ways)
  static constexpr int ROWSA = 8 * MTA;
  static constexpr int BM = 3 * ROWSA * LDM;    // doubles of Bm [3][ROWSA][LDM] (Br, Bs, B0)
  static constexpr int W = (P <= 5) ? AW_W_SMALL : 12;  // warps per CTA
  static constexpr int GSZ = 6 * Q;             // doubles of one element's G
  static constexpr bool WHOLE = (P <= 3);       // small elements: one TMA copy per element, else per a-tile
  static constexpr int R = WHOLE ? 2 : 3;       // slots per warp (TMA ring)
  static constexpr int TS = WHOLE ? 6 * Q : 6 * QV * 8;   // doubles of one slot
  static constexpr int TPE = WHOLE ? 1 : MTA;   // TMA copies per element
  static constexpr int NALAST = QT - 8 * (MTA - 1);
  static constexpr int QE = (QV + 1) / 2;       // even vertical points first in a tile (bank spread)
  static constexpr int SMEM = (BM + W * R * TS) * 8 + W * R * 8;
  static_assert(SMEM <= 227 * 1024, "apply_warp shared memory");
};

// host: Bm [3][ROWSA][LDM] (Br, Bs, B0 at [a][m], zero padded) followed by Bt, Dt [QV][N1]
std::vector<double> warp_apply_mats(const LevelRef& R) {
  auto run = [&](auto tag) {
    using D = AW<decltype(tag)::value>;
    std::vector<double> v(D::BM + 2 * D::QV * D::N1, 0.0);
    const double* B[3] = {R.Br.data(), R.Bs.data(), R.B0.data()};
    for (int c = 0; c < 3; ++c)
      for (int a = 0; a < D::QT; ++a)
        for (int m = 0; m < D::NT; ++m) v[(c * D::ROWSA + a) * D::LDM + m] = B[c][a * D::NT + m];
    for (int i = 0; i < D::QV * D::N1; ++i) {
      v[D::BM + i] = R.Bt[i];
      v[D::BM + D::QV * D::N1 + i] = R.Dt[i];
    }
    return v;
  };
  switch (R.p) {
    case 1: return run(std::integral_constant<int, 1>{});
    case 2: return run(std::integral_constant<int, 2>{});
    case 3: return run(std::integral_constant<int, 3>{});
    case 4: return run(std::integral_constant<int, 4>{});
    case 5: return run(std::integral_constant<int, 5>{});
    case 6: return run(std::integral_constant<int, 6>{});
  }
  return {};
}

__device__ __forceinline__ void aw_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t aw_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// B fragment (k row = 4 ks + c4 of an 8-row tile, n col = r4) of a tile held as C fragments
__device__ __forceinline__ double aw_c_to_b(double c0, double c1, int ks, int lane) {
  const int src = ((((ks & 1) << 2) + (lane & 3)) << 2) | ((lane >> 2) >> 1);
  const double x0 = __shfl_sync(0xffffffffu, c0, src);
  const double x1 = __shfl_sync(0xffffffffu, c1, src);
  return ((lane >> 2) & 1) ? x1 : x0;
}
// A fragment (row r4, k col = 4 ks + c4 of an 8-col tile) of a tile held as C fragments
__device__ __forceinline__ double aw_c_to_a(double c0, double c1, int ks, int lane) {
  const int src = (lane & ~3) | (((ks & 1) << 1) + ((lane & 3) >> 1));
  const double x0 = __shfl_sync(0xffffffffu, c0, src);
  const double x1 = __shfl_sync(0xffffffffu, c1, src);
  return (lane & 1) ? x1 : x0;
}

template <int P>
__global__ void __launch_bounds__(32 * AW<P>::W, 1) k_apply_warp(int E, const int32_t* __restrict__ conn,
                                                                 const double* __restrict__ G,
                                                                 const double* __restrict__ mats,
                                                                 const double* __restrict__ u, double* __restrict__ y,
                                                                 int flags, const int32_t* __restrict__ elist) {
  // E = element slots; slot s is element elist[s] (a subset, e.g. the interface elements of a
  // partition, dist.cu) or s itself when elist is null
  using D = AW<P>;
  extern __shared__ __align__(128) double sm[];
  double* Bm = sm;                          // [3][ROWSA][LDM]
  double* Gs = sm + D::BM;                  // [W][R][TS]  a-tile ring of every warp
  uint64_t* mbar = reinterpret_cast<uint64_t*>(Gs + D::W * D::R * D::TS);  // [W][R]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r4 = lane >> 2, c4 = lane & 3;
  for (int i = tid; i < D::BM; i += 32 * D::W) Bm[i] = __ldg(mats + i);
  if (lane == 0) {
    for (int b = 0; b < D::R; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(aw_smem(mbar + D::R * warp + b)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // constant B fragments of the vertical stages
  const double* Bt = mats + D::BM;        // [q][l]
  const double* Dt = Bt + D::QV * D::N1;
  double fBt[D::KL][D::NQ], fDt[D::KL][D::NQ];   // stage A:  B[k=l][n=q] = Bt[q][l]
#pragma unroll
  for (int kl = 0; kl < D::KL; ++kl)
#pragma unroll
    for (int nq = 0; nq < D::NQ; ++nq) {
      const int l = kl * 4 + c4, q = nq * 8 + r4;
      const bool ok = l < D::N1 && q < D::QV;
      fBt[kl][nq] = ok ? __ldg(Bt + q * D::N1 + l) : 0.0;
      fDt[kl][nq] = ok ? __ldg(Dt + q * D::N1 + l) : 0.0;
    }
  double gBt[D::KQ][D::NL], gDt[D::KQ][D::NL];   // stage A^T:  B[k=q][n=l] = Bt[q][l]
#pragma unroll
  for (int kq = 0; kq < D::KQ; ++kq)
#pragma unroll
    for (int nl = 0; nl < D::NL; ++nl) {
      const int q = kq * 4 + c4, l = nl * 8 + r4;
      const bool ok = l < D::N1 && q < D::QV;
      gBt[kq][nl] = ok ? __ldg(Bt + q * D::N1 + l) : 0.0;
      gDt[kq][nl] = ok ? __ldg(Dt + q * D::N1 + l) : 0.0;
    }
  const double sgn = (flags & AP_NEGATE) ? -1.0 : 1.0;
  const int stride = gridDim.x * D::W;
  int e = blockIdx.x * D::W + warp;
  const int e0 = e;
  double* ring = Gs + warp * D::R * D::TS;
  // copy t of this warp's stream: element e0 + (t / TPE) stride, a-tile ma = t % TPE (or the whole
  // element), slot t % R
  auto eid = [&](int sl) { return elist ? __ldg(elist + sl) : sl; };
  auto issue_tile = [&](int t) {
    const int sl = e0 + (t / D::TPE) * stride, ma = t % D::TPE;
    if (sl >= E || lane != 0) return;
    const int el = eid(sl);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of the slot
    const uint32_t bytes =
        D::WHOLE ? (uint32_t)D::GSZ * 8u : (uint32_t)(6 * D::QV * (ma < D::MTA - 1 ? 8 : D::NALAST)) * 8u;
    const uint32_t mb = aw_smem(mbar + D::R * warp + t % D::R);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            aw_smem(ring + (t % D::R) * D::TS)),
        "l"(G + (size_t)el * D::GSZ + (size_t)ma * D::TS), "r"(bytes), "r"(mb)
        : "memory");
  };
  // connectivity of the A-fragment positions (m = 8 mm + r4, l = 4 kl + c4) and gather of u
  auto load_conn_a = [&](int el, int (&cA)[D::MTM][D::KL]) {
    const int32_t* ce = conn + (size_t)el * D::N;
#pragma unroll
    for (int mm = 0; mm < D::MTM; ++mm)
#pragma unroll
      for (int kl = 0; kl < D::KL; ++kl) {
        const int m = mm * 8 + r4, l = kl * 4 + c4;
        cA[mm][kl] = (m < D::NT && l < D::N1) ? __ldg(ce + m + D::NT * l) : INT_MIN;
      }
  };
  auto gather_u = [&](const int (&cA)[D::MTM][D::KL], double (&ua)[D::MTM][D::KL]) {
#pragma unroll
    for (int mm = 0; mm < D::MTM; ++mm)
#pragma unroll
      for (int kl = 0; kl < D::KL; ++kl) {
        const int g = cA[mm][kl];
        ua[mm][kl] = (g >= 0 || (g != INT_MIN && (flags & AP_GATHER_ALL))) ? __ldg(u + (g >= 0 ? g : ~g)) : 0.0;
      }
  };
  int cA[D::MTM][D::KL];
  double ua[D::MTM][D::KL];
  if (e < E) {
    for (int t = 0; t < D::R; ++t) issue_tile(t);
    load_conn_a(eid(e), cA);
    gather_u(cA, ua);
  }
  int tk = 0;  // first copy index of the current element
  while (e < E) {
    const int en = e + stride;
    const int32_t* ce = conn + (size_t)eid(e) * D::N;
    // connectivity of this element's output positions (m = 8 mm + r4, l = 8 nl + 2 c4 + i), used at the end
    int cY[D::MTM][D::NL][2];
#pragma unroll
    for (int mm = 0; mm < D::MTM; ++mm)
#pragma unroll
      for (int nl = 0; nl < D::NL; ++nl)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int m = mm * 8 + r4, l = nl * 8 + 2 * c4 + i;
          cY[mm][nl][i] = (m < D::NT && l < D::N1) ? __ldg(ce + m + D::NT * l) : INT_MIN;
        }
    if (en < E) load_conn_a(eid(en), cA);   // next element's gather positions (in flight during stage A)
    // ---- stage A: Ut, Udt [m][q]
    double Ut[D::MTM][D::NQ][2], Udt[D::MTM][D::NQ][2];
#pragma unroll
    for (int mm = 0; mm < D::MTM; ++mm)
#pragma unroll
      for (int nq = 0; nq < D::NQ; ++nq) {
        Ut[mm][nq][0] = Ut[mm][nq][1] = Udt[mm][nq][0] = Udt[mm][nq][1] = 0.0;
#pragma unroll
        for (int kl = 0; kl < D::KL; ++kl) {
          aw_dmma(Ut[mm][nq][0], Ut[mm][nq][1], ua[mm][kl], fBt[kl][nq]);
          aw_dmma(Udt[mm][nq][0], Udt[mm][nq][1], ua[mm][kl], fDt[kl][nq]);
        }
      }
    // ---- next element's u (in flight during stages B, G, B^T)
    double un[D::MTM][D::KL];
    if (en < E) gather_u(cA, un);
    // ---- B fragments of Ut, Udt for stage B: B[k=m][n=q]
    double bU[D::KM][D::NQ], bD[D::KM][D::NQ];
#pragma unroll
    for (int km = 0; km < D::KM; ++km)
#pragma unroll
      for (int nq = 0; nq < D::NQ; ++nq) {
        bU[km][nq] = aw_c_to_b(Ut[km >> 1][nq][0], Ut[km >> 1][nq][1], km, lane);
        bD[km][nq] = aw_c_to_b(Udt[km >> 1][nq][0], Udt[km >> 1][nq][1], km, lane);
      }
    double Vt[D::MTM][D::NQ][2], Vdt[D::MTM][D::NQ][2];
#pragma unroll
    for (int mm = 0; mm < D::MTM; ++mm)
#pragma unroll
      for (int nq = 0; nq < D::NQ; ++nq) Vt[mm][nq][0] = Vt[mm][nq][1] = Vdt[mm][nq][0] = Vdt[mm][nq][1] = 0.0;
    AW_PRAGMA(unroll AW_MA_UNROLL)
    for (int ma = 0; ma < D::MTA; ++ma) {
      const int t = D::WHOLE ? tk : tk + ma;
      if (!D::WHOLE || ma == 0) {  // wait for copy t of G
        const uint32_t mb = aw_smem(mbar + D::R * warp + t % D::R);
        const uint32_t par = (uint32_t)(t / D::R) & 1u;
        uint32_t done = 0;
        while (!done)
          asm volatile(
              "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
              : "=r"(done)
              : "r"(mb), "r"(par)
              : "memory");
      }
      const double* Gt = ring + (t % D::R) * D::TS + (D::WHOLE ? ma * 48 * D::QV : 0);
      const int na = (ma < D::MTA - 1) ? 8 : D::NALAST;
      // ---- stage B for a-tile ma
      double g[3][D::NQ][2];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int nq = 0; nq < D::NQ; ++nq) g[c][nq][0] = g[c][nq][1] = 0.0;
#pragma unroll
      for (int km = 0; km < D::KM; ++km) {
        const int off = (ma * 8 + r4) * D::LDM + km * 4 + c4;
        const double ar = Bm[off], as = Bm[D::ROWSA * D::LDM + off], a0 = Bm[2 * D::ROWSA * D::LDM + off];
#pragma unroll
        for (int nq = 0; nq < D::NQ; ++nq) {
          aw_dmma(g[0][nq][0], g[0][nq][1], ar, bU[km][nq]);
          aw_dmma(g[1][nq][0], g[1][nq][1], as, bU[km][nq]);
          aw_dmma(g[2][nq][0], g[2][nq][1], a0, bD[km][nq]);
        }
      }
      // ---- w = G g at the points (a, q) of the C fragments
#pragma unroll
      for (int nq = 0; nq < D::NQ; ++nq)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int a = ma * 8 + r4, q = nq * 8 + 2 * c4 + i;
          double w0 = 0.0, w1 = 0.0, w2 = 0.0;
          if (a < D::QT && q < D::QV) {
            const int qp = (q & 1) ? D::QE + (q >> 1) : (q >> 1);   // tile row of q
            const double* gp = Gt + qp * na + r4;
            const int cs = D::QV * na;                               // component stride in the tile
            const double gxx = gp[0], gxy = gp[cs], gxz = gp[2 * cs], gyy = gp[3 * cs], gyz = gp[4 * cs],
                         gzz = gp[5 * cs];
            const double x0 = g[0][nq][i], x1 = g[1][nq][i], x2 = g[2][nq][i];
            w0 = gxx * x0 + gxy * x1 + gxz * x2;
            w1 = gxy * x0 + gyy * x1 + gyz * x2;
            w2 = gxz * x0 + gyz * x1 + gzz * x2;
          }
          g[0][nq][i] = w0;
          g[1][nq][i] = w1;
          g[2][nq][i] = w2;
        }
      // ---- stage B^T: Vt += Br^T w_r + Bs^T w_s, Vdt += B0^T w_t over this a-tile (k = a)
#pragma unroll
      for (int ka = 0; ka < 2; ++ka) {
        double bw[3][D::NQ];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int nq = 0; nq < D::NQ; ++nq) bw[c][nq] = aw_c_to_b(g[c][nq][0], g[c][nq][1], ka, lane);
#pragma unroll
        for (int mm = 0; mm < D::MTM; ++mm) {
          const int off = (ma * 8 + ka * 4 + c4) * D::LDM + mm * 8 + r4;   // A[m][a] = B[a][m]
          const double ar = Bm[off], as = Bm[D::ROWSA * D::LDM + off], a0 = Bm[2 * D::ROWSA * D::LDM + off];
#pragma unroll
          for (int nq = 0; nq < D::NQ; ++nq) {
            aw_dmma(Vt[mm][nq][0], Vt[mm][nq][1], ar, bw[0][nq]);
            aw_dmma(Vt[mm][nq][0], Vt[mm][nq][1], as, bw[1][nq]);
            aw_dmma(Vdt[mm][nq][0], Vdt[mm][nq][1], a0, bw[2][nq]);
          }
        }
      }
      if (!D::WHOLE || ma == D::MTA - 1) {
        __syncwarp();  // every lane is done with this slot before it is refilled
        issue_tile(t + D::R);
      }
    }
    // ---- stage A^T: y[m][l] = Vt Bt + Vdt Dt (k = q), scatter
#pragma unroll
    for (int mm = 0; mm < D::MTM; ++mm) {
      double yc[D::NL][2];
#pragma unroll
      for (int nl = 0; nl < D::NL; ++nl) yc[nl][0] = yc[nl][1] = 0.0;
#pragma unroll
      for (int kq = 0; kq < D::KQ; ++kq) {
        const double at = aw_c_to_a(Vt[mm][kq >> 1][0], Vt[mm][kq >> 1][1], kq, lane);
        const double ad = aw_c_to_a(Vdt[mm][kq >> 1][0], Vdt[mm][kq >> 1][1], kq, lane);
#pragma unroll
        for (int nl = 0; nl < D::NL; ++nl) {
          aw_dmma(yc[nl][0], yc[nl][1], at, gBt[kq][nl]);
          aw_dmma(yc[nl][0], yc[nl][1], ad, gDt[kq][nl]);
        }
      }
#pragma unroll
      for (int nl = 0; nl < D::NL; ++nl)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int g = cY[mm][nl][i];
          if (g >= 0) atomicAdd(y + g, sgn * yc[nl][i]);
          else if (g != INT_MIN && (flags & AP_SCATTER_ALL)) atomicAdd(y + ~g, sgn * yc[nl][i]);
        }
    }
    if (en < E) {
#pragma unroll
      for (int mm = 0; mm < D::MTM; ++mm)
#pragma unroll
        for (int kl = 0; kl < D::KL; ++kl) ua[mm][kl] = un[mm][kl];
    }
    tk += D::TPE;
    e = en;
  }
}

// G [E][6][Q] (point a + QT q) -> a-tile-major copy for k_apply_warp: per element, tile ma
// (8 points a, the last one QT - 8(MTA-1)) at offset 48 QV ma, inside [comp][qpos][a_local]
// with the even vertical points first (qpos spreads a fragment's 4 q-rows over both bank halves)
__global__ void k_g_tiles(int64_t E, int QT, int QV, const double* __restrict__ G, double* __restrict__ Gw) {
  const int Q = QT * QV, MTA = (QT + 7) / 8, QE = (QV + 1) / 2;
  const int64_t tot = E * 6 * Q;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / (6 * Q);
    const int r = (int)(i % (6 * Q)), c = r / Q, pt = r % Q, a = pt % QT, q = pt / QT;
    const int ma = a / 8, na = (ma < MTA - 1) ? 8 : QT - 8 * (MTA - 1);
    const int qp = (q & 1) ? QE + (q >> 1) : (q >> 1);
    Gw[e * 6 * Q + (int64_t)48 * QV * ma + (c * QV + qp) * na + (a - 8 * ma)] = G[i];
  }
}

void build_g_tiles(sem_ctx* c, int level) {
  DeviceLevel& L = c->L[level];
  const int QT = L.ref.qt, QV = L.ref.qv;
  if (L.p > 6 || (c->opts.apply_kernel != 0 && c->opts.apply_kernel != 3 && c->opts.apply_kernel != 4)) return;
  if (!L.Gw) {  // refreshed in place by sem_update_geometry
    CUDA_CHECK(cudaMalloc(&L.Gw, (size_t)c->E * 6 * L.Q * sizeof(double)));
    c->allocs.push_back(L.Gw);
    c->device_bytes += (int64_t)c->E * 6 * L.Q * 8;
  }
  k_g_tiles<<<148 * 16, 256, 0, c->stream>>>(c->E, QT, QV, L.G, L.Gw);
  CUDA_CHECK(cudaGetLastError());
}

template <int P>
static void apply_warp_P(sem_ctx* c, const DeviceLevel& L, const double* u, double* y, int flags,
                         const int32_t* elist, int ne) {
  using D = AW<P>;
  static int grid_maxes[kMaxDev] = {0};
  const int dev = cur_device();
  int& grid_max = grid_maxes[dev];
  if (!grid_max) {
    CUDA_CHECK(cudaFuncSetAttribute(k_apply_warp<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, D::SMEM));
    int per_sm = 0, sms = 0;
    CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_apply_warp<P>, 32 * D::W, D::SMEM));
    grid_max = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int E = elist ? ne : c->E_own;
  if (E == 0) return;
  const int need = (E + D::W - 1) / D::W;
  const int grid = need < grid_max ? need : grid_max;
  k_apply_warp<P><<<grid, 32 * D::W, D::SMEM, c->stream>>>(E, L.conn, L.Gw, L.wmats, u, y, flags, elist);
  CUDA_CHECK(cudaGetLastError());
}

bool launch_apply_warp(sem_ctx* c, int level, const double* u, double* y, int flags, const int32_t* elist, int ne) {
  const DeviceLevel& L = c->L[level];
  if (!L.wmats || !L.Gw) return false;
  switch (L.p) {
    case 1: apply_warp_P<1>(c, L, u, y, flags, elist, ne); break;
    case 2: apply_warp_P<2>(c, L, u, y, flags, elist, ne); break;
    case 3: apply_warp_P<3>(c, L, u, y, flags, elist, ne); break;
    case 4: apply_warp_P<4>(c, L, u, y, flags, elist, ne); break;
    case 5: apply_warp_P<5>(c, L, u, y, flags, elist, ne); break;
    case 6: apply_warp_P<6>(c, L, u, y, flags, elist, ne); break;
    default: return false;
  }
  c->launches++;
  return true;
}

}  // namespace sem
