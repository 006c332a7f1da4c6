// Operator apply, FOUR elements per warp, FP64 tensor cores (sm_100a DMMA) for the
// triangle stages and FP64 FMA for the vertical stages.
//
// The same operator as k_apply_warp / k_apply (eq 3.8): y (+/-)= sum_e
// Q_e^T D^T (G (.) D Q_e u), sum-factorised vertical-first:
//
//   A    Ut[m][q] = sum_l u[m][l] Bt[q][l],  Udt[m][q] = sum_l u[m][l] Dt[q][l]      (FMA)
//   B    g_c[a][q] = sum_m B_c[a][m] U_c[m][q]   (c = r, s on Ut; c = 0 on Udt)    (DMMA)
//   G    w = G g at every cubature point (a, q)                                     (FMA)
//   B^T  Vt[m][q] = sum_a Br[a][m] w_r + Bs[a][m] w_s,  Vdt[m][q] = sum_a B0[a][m] w_0 (DMMA)
//   A^T  y[m][l] = sum_q Vt[m][q] Bt[q][l] + Vdt[m][q] Dt[q][l]                    (FMA)
//
// Why four elements: the triangle stages carry ~85 % of the flops.  With one element
// per warp (k_apply_warp) their DMMA tiles are padded along the vertical points (p+1 =
// 6 of 8 columns at p = 5).  Here the M dimension of both triangle GEMMs is the pair
// (vertical point q, element e) of four elements, row = 8 mt + r4 with e = r4 & 3 and
// q = 2 mt + (r4 >> 2): (p+1) x 4 rows fill whole 8-row tiles (p = 3, 5), and every
// lane only ever holds data of ONE element (e = (lane >> 2) & 3).  Consequences:
//   * stage A's outputs are computed by each lane directly in the A-fragment layout
//     of stage B (FMA, no padding along the 6-point vertical dimension);
//   * stage B's C fragment (row, a = 8 na + 2 c4 + i) is stage B^T's A fragment
//     without any shuffle: the contraction index a of stage B^T is enumerated as
//     k-step i <-> a = 8 na + 2 c4 + i (a permutation of k, applied to the B operand
//     read from shared memory as well);
//   * stage A^T is again per lane (FMA) over the lane's own three q values, then one
//     xor-16 shuffle adds the partner lane's other three.
// DMMA per element at p = 5: 135 (k_apply_warp: 195).
//
// Data movement: the geometric factors of the four elements' current a-tile are
// staged by four TMA bulk copies (cp.async.bulk + mbarrier) into a per-warp ring of
// 2 slots (the a-tile-major layout of k_g_tiles, shared with k_apply_warp); u is
// gathered through the connectivity into registers, y scattered with FP64 atomics.
// Persistent CTAs of 8 warps.
#include <cuda_runtime.h>

#include <climits>

#include "internal.h"

namespace sem {

namespace aq {
__host__ __device__ constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }
}  // namespace aq

// P: triangle order, PZ: vertical order (anisotropic P_P x P_PZ levels of SURVEY NEXT-2; PZ = P
// for the isotropic kernels): N1 = P + 1 triangle-edge nodes, NV = PZ + 1 vertical nodes and points
template <int P, int PZ = P>
struct AQ {
  static constexpr int N1 = P + 1, NT = N1 * (N1 + 1) / 2, QT = N1 * N1, NV = PZ + 1, QV = NV, Q = QT * QV,
                       N = NT * NV;
  static constexpr int MTQ = aq::cdiv(QV, 2);   // row tiles over (q, e)
  static constexpr int KM = aq::cdiv(NT, 4);    // k-steps over triangle nodes (stage B)
  static constexpr int MTA = aq::cdiv(QT, 8);   // a-tiles
  static constexpr int NM = aq::cdiv(NT, 8);    // n-tiles over triangle nodes (stage B^T)
  static constexpr int NALAST = QT - 8 * (MTA - 1);
  static constexpr int QE = (QV + 1) / 2;       // k_g_tiles' q permutation: even points first
  static constexpr int LDM = 8 * aq::cdiv(NT, 8) + 4;   // row stride of Bm (= 4 mod 8)
  static constexpr int ROWSA = 8 * MTA;
  static constexpr int BM = 3 * ROWSA * LDM;    // Br, Bs, B0 [a][m], zero padded (stage B operands)
  // stage B^T operands, transposed: [3][8 NM][LDA] = B_c[a][m] at [m][a]; LDA = 8 mod 16 so that the
  // 16-byte loads of the (a, a+1) pairs of a quarter-warp (two m rows x four a pairs) hit distinct banks
  static constexpr int LDA = 8 * MTA + ((8 * MTA) % 16 == 0 ? 8 : 0);
  static constexpr int BMT = 3 * 8 * NM * LDA;
  static constexpr int BT = 2 * QV * NV;        // Bt, Dt [q][l]
  static constexpr int W = 8;                   // warps per CTA
  static constexpr int R = 2;                   // ring slots per warp
  static constexpr int TSE0 = 6 * QV * 8;       // doubles of one element's a-tile (full tile)
  static constexpr int TSE = TSE0 + 8;          // slot stride per element: = 8 mod 16 (bank spread of the 4 elements)
  static constexpr int TS = 4 * TSE;            // doubles of one slot (four elements)
  static constexpr int NYL = aq::cdiv(NV, 2);   // vertical output nodes scattered per lane
  // next quad's gather staged in shared memory by cp.async: u [4][UST] (UST = 4 mod 16: the four
  // elements' rows in distinct banks) and the connectivity [4 N]
  static constexpr int UST = (N + 11) / 16 * 16 + 4;
  static constexpr int SU = 4 * UST, SC = 4 * N;
  static constexpr int SMEM = (BMT + BT + W * R * TS + W * SU) * 8 + W * SC * 4 + W * R * 8;
  static_assert(TSE % 16 == 8 && LDA % 16 == 8, "bank layout");
};

// host: Bm [3][ROWSA][LDM] (Br, Bs, B0 at [a][m]), BmT [3][8 NM][LDA] (the same at [m][a]),
// then Bt, Dt [q][l]
std::vector<double> quad_apply_mats(const LevelRef& R) {
  auto run = [&](auto tp, auto tq) {
    using D = AQ<decltype(tp)::value, decltype(tq)::value>;
    std::vector<double> v(D::BM + D::BMT + D::BT, 0.0);
    const double* B[3] = {R.Br.data(), R.Bs.data(), R.B0.data()};
    for (int c = 0; c < 3; ++c)
      for (int a = 0; a < D::QT; ++a)
        for (int m = 0; m < D::NT; ++m) {
          v[(c * D::ROWSA + a) * D::LDM + m] = B[c][a * D::NT + m];
          v[D::BM + (c * 8 * D::NM + m) * D::LDA + a] = B[c][a * D::NT + m];
        }
    for (int i = 0; i < D::QV * D::NV; ++i) {
      v[D::BM + D::BMT + i] = R.Bt[i];
      v[D::BM + D::BMT + D::QV * D::NV + i] = R.Dt[i];
    }
    return v;
  };
  using std::integral_constant;
#define AQ_CASE(P_, Q_) \
  if (R.p == P_ && R.q == Q_) return run(integral_constant<int, P_>{}, integral_constant<int, Q_>{});
  AQ_CASE(3, 3) AQ_CASE(4, 4) AQ_CASE(5, 5) AQ_CASE(6, 6)
  AQ_CASE(3, 1) AQ_CASE(3, 2) AQ_CASE(3, 4) AQ_CASE(3, 5)
  AQ_CASE(4, 1) AQ_CASE(4, 2) AQ_CASE(4, 3) AQ_CASE(4, 5)
  AQ_CASE(5, 1) AQ_CASE(5, 2) AQ_CASE(5, 3) AQ_CASE(5, 4)
#undef AQ_CASE
  return {};
}

__device__ __forceinline__ void aq_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t aq_smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int P>
__global__ void __launch_bounds__(32 * AQ<P>::W, 1)
    k_apply_quad(int E, const int32_t* __restrict__ conn, const double* __restrict__ Gw,
                 const double* __restrict__ mats, const double* __restrict__ u, double* __restrict__ y, int flags) {
  using D = AQ<P>;
  static_assert(D::SMEM <= 227 * 1024, "apply_quad shared memory");
  extern __shared__ __align__(128) double sm[];
  double* BmT = sm;                       // [3][8 NM][LDA]  B_c[a][m] at [m][a] (both triangle stages)
  double* sBt = BmT + D::BMT;             // [QV][N1]
  double* sDt = sBt + D::QV * D::N1;
  double* ringall = sBt + D::BT;          // [W][R][4][TSE]
  double* suall = ringall + D::W * D::R * D::TS;      // [W][4][UST]
  int32_t* scall = reinterpret_cast<int32_t*>(suall + D::W * D::SU);   // [W][4 N]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(scall + D::W * D::SC);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r4 = lane >> 2, c4 = lane & 3, el = r4 & 3, h = r4 >> 2;
  for (int i = tid; i < D::BMT + D::BT; i += 32 * D::W) sm[i] = __ldg(mats + D::BM + i);
  if (lane == 0) {
    for (int b = 0; b < D::R; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(aq_smem(mbar + D::R * warp + b)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const double sgn = (flags & AP_NEGATE) ? -1.0 : 1.0;
  const int nquad = (E + 3) >> 2;
  const int qstride = gridDim.x * D::W;
  const int q0 = blockIdx.x * D::W + warp;
  double* ring = ringall + warp * D::R * D::TS;
  // copy t of this warp: quad q0 + (t / MTA) qstride, a-tile t % MTA, slot t % R: four bulk copies
  auto issue = [&](int t) {
    const int qd = q0 + (t / D::MTA) * qstride, ma = t % D::MTA;
    if (qd >= nquad || lane != 0) return;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int ne = min(4, E - 4 * qd);
    const uint32_t one = (uint32_t)(6 * D::QV * (ma < D::MTA - 1 ? 8 : D::NALAST)) * 8u;
    const uint32_t mb = aq_smem(mbar + D::R * warp + t % D::R);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(one * ne) : "memory");
    for (int k = 0; k < ne; ++k)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              aq_smem(ring + (t % D::R) * D::TS + k * D::TSE)),
          "l"(Gw + (size_t)(4 * qd + k) * 6 * D::Q + (size_t)ma * 48 * D::QV), "r"(one), "r"(mb)
          : "memory");
  };
  double* su = suall + warp * D::SU;
  int32_t* scn = scall + warp * D::SC;
  // gather staging of quad qd: (1) its connectivity, 16-byte cp.async; (2) u through it, 8-byte
  // cp.async (zero-filled where absent / Dirichlet); consumed after cp.async.wait_group 0
  auto stage_conn = [&](int qd) {
    const int64_t base = (int64_t)4 * qd * D::N;
    const int nval = min(4, E - 4 * qd) * D::N;   // ints of the quad's existing elements
    for (int i = lane; i < D::SC / 4; i += 32) {
      const int cnt = min(4, max(0, nval - 4 * i));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(aq_smem(scn + 4 * i)),
                   "l"(conn + base + 4 * i), "r"(4 * cnt)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto stage_u = [&](int qd) {
    const int nval = min(4, E - 4 * qd) * D::N;
    for (int i = lane; i < D::SC; i += 32) {
      const int g = i < nval ? scn[i] : INT_MIN;
      const bool take = g >= 0 || (g != INT_MIN && (flags & AP_GATHER_ALL));
      const double* src = u + (take ? (g >= 0 ? g : ~g) : 0);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(aq_smem(su + (i / D::N) * D::UST + i % D::N)),
                   "l"(src), "r"(take ? 8 : 0)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (q0 < nquad) {
    for (int t = 0; t < D::R; ++t) issue(t);
    stage_conn(q0);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    stage_u(q0);
  }
  int tk = 0;
  for (int qd = q0; qd < nquad; qd += qstride, tk += D::MTA) {
    const int e = 4 * qd + el;
    const bool ev = e < E;
    const int32_t* ce = conn + (size_t)(ev ? e : 0) * D::N;
    // ---- stage A (FMA): lane's A fragments of stage B, m = 4 ks + c4, q = 2 mt + h
    double Ua[D::MTQ][D::KM], Ud[D::MTQ][D::KM];
    asm volatile("cp.async.wait_group 0;" ::: "memory");   // this quad's u (staged during the previous one)
    __syncwarp();
    {
      double uu[D::KM][D::N1];
#pragma unroll
      for (int ks = 0; ks < D::KM; ++ks)
#pragma unroll
        for (int l = 0; l < D::N1; ++l) {
          const int m = 4 * ks + c4;
          uu[ks][l] = (ev && m < D::NT) ? su[el * D::UST + m + D::NT * l] : 0.0;
        }
#pragma unroll
      for (int mt = 0; mt < D::MTQ; ++mt) {
        const int q = 2 * mt + h;
#pragma unroll
        for (int ks = 0; ks < D::KM; ++ks) Ua[mt][ks] = Ud[mt][ks] = 0.0;
        if (q < D::QV) {
#pragma unroll
          for (int l = 0; l < D::N1; ++l) {
            const double bt = sBt[q * D::N1 + l], dt = sDt[q * D::N1 + l];
#pragma unroll
            for (int ks = 0; ks < D::KM; ++ks) {
              Ua[mt][ks] = fma(uu[ks][l], bt, Ua[mt][ks]);
              Ud[mt][ks] = fma(uu[ks][l], dt, Ud[mt][ks]);
            }
          }
        }
      }
    }
    double Vt[D::MTQ][D::NM][2], Vd[D::MTQ][D::NM][2];
#pragma unroll
    for (int mt = 0; mt < D::MTQ; ++mt)
#pragma unroll
      for (int nm = 0; nm < D::NM; ++nm) Vt[mt][nm][0] = Vt[mt][nm][1] = Vd[mt][nm][0] = Vd[mt][nm][1] = 0.0;
    // next quad's gather staged in shared memory during this quad (only 2 warps per scheduler:
    // the connectivity -> u dependent loads of a quad start would otherwise stall the warp)
    const int qn = qd + qstride;
#pragma unroll 1
    for (int na = 0; na < D::MTA; ++na) {
      const int t = tk + na;
      if (na == 0 && qn < nquad) {
        __syncwarp();   // every lane has read this quad's u from su
        stage_conn(qn);
      }
      if (na == 1 && qn < nquad) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        stage_u(qn);
      }
      {  // wait for copy t
        const uint32_t mb = aq_smem(mbar + D::R * warp + t % D::R);
        const uint32_t par = (uint32_t)(t / D::R) & 1u;
        uint32_t done = 0;
        while (!done)
          asm volatile(
              "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
              : "=r"(done)
              : "r"(mb), "r"(par)
              : "memory");
      }
      // ---- stage B: g_c^T[(q,e)][a] for this a-tile, B operand = B_c[a = 8 na + r4][m = 4 ks + c4]
      double g[3][D::MTQ][2];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int mt = 0; mt < D::MTQ; ++mt) g[c][mt][0] = g[c][mt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < D::KM; ++ks) {
        const int off = (4 * ks + c4) * D::LDA + 8 * na + r4;    // B_c[a = 8 na + r4][m = 4 ks + c4]
        const double br = BmT[off], bs = BmT[8 * D::NM * D::LDA + off], b0 = BmT[16 * D::NM * D::LDA + off];
#pragma unroll
        for (int mt = 0; mt < D::MTQ; ++mt) {
          aq_dmma(g[0][mt][0], g[0][mt][1], Ua[mt][ks], br);
          aq_dmma(g[1][mt][0], g[1][mt][1], Ua[mt][ks], bs);
          aq_dmma(g[2][mt][0], g[2][mt][1], Ud[mt][ks], b0);
        }
      }
      // ---- w = G g at the lane's points (a = 8 na + 2 c4 + i, q = 2 mt + h) of element el
      const int nat = (na < D::MTA - 1) ? 8 : D::NALAST;
      const double* Gt = ring + (t % D::R) * D::TS + el * D::TSE;
      const int cs = D::QV * nat;   // component stride in the tile
#pragma unroll
      for (int mt = 0; mt < D::MTQ; ++mt) {
        const int q = 2 * mt + h;
        const int qp = (q & 1) ? D::QE + (q >> 1) : (q >> 1);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int al = 2 * c4 + i;
          double w0 = 0.0, w1 = 0.0, w2 = 0.0;
          if (ev && q < D::QV && al < nat) {
            const double* gp = Gt + qp * nat + al;
            double gxx, gxy, gxz, gyy, gyz, gzz;
            if ((D::NALAST & 1) == 0 || na < D::MTA - 1) {  // the pair (al, al + 1): one 16-byte load per component
              const double2 v0 = *reinterpret_cast<const double2*>(gp - i);
              const double2 v1 = *reinterpret_cast<const double2*>(gp - i + cs);
              const double2 v2 = *reinterpret_cast<const double2*>(gp - i + 2 * cs);
              const double2 v3 = *reinterpret_cast<const double2*>(gp - i + 3 * cs);
              const double2 v4 = *reinterpret_cast<const double2*>(gp - i + 4 * cs);
              const double2 v5 = *reinterpret_cast<const double2*>(gp - i + 5 * cs);
              gxx = i ? v0.y : v0.x;
              gxy = i ? v1.y : v1.x;
              gxz = i ? v2.y : v2.x;
              gyy = i ? v3.y : v3.x;
              gyz = i ? v4.y : v4.x;
              gzz = i ? v5.y : v5.x;
            } else {
              gxx = gp[0];
              gxy = gp[cs];
              gxz = gp[2 * cs];
              gyy = gp[3 * cs];
              gyz = gp[4 * cs];
              gzz = gp[5 * cs];
            }
            const double x0 = g[0][mt][i], x1 = g[1][mt][i], x2 = g[2][mt][i];
            w0 = gxx * x0 + gxy * x1 + gxz * x2;
            w1 = gxy * x0 + gyy * x1 + gyz * x2;
            w2 = gxz * x0 + gyz * x1 + gzz * x2;
          }
          g[0][mt][i] = w0;
          g[1][mt][i] = w1;
          g[2][mt][i] = w2;
        }
      }
      __syncwarp();  // every lane is done with this slot before it is refilled
      issue(t + D::R);
      // ---- stage B^T: V^T[(q,e)][m] += w^T[(q,e)][a] B_c[a][m]; k-step i <-> a = 8 na + 2 c4 + i
      // B^T operands of both k-steps (a = 8 na + 2 c4 + {0, 1}) in one 16-byte load per component;
      // the DMMAs then sweep all (mt, nm) accumulators per operand, so that two updates of one
      // accumulator are MTQ x NM instructions apart (no back-to-back dependent DMMA)
      double2 bo[3][D::NM];
#pragma unroll
      for (int nm = 0; nm < D::NM; ++nm) {
        const int off = (8 * nm + r4) * D::LDA + 8 * na + 2 * c4;
#pragma unroll
        for (int c = 0; c < 3; ++c) bo[c][nm] = *reinterpret_cast<const double2*>(BmT + 8 * c * D::NM * D::LDA + off);
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int mt = 0; mt < D::MTQ; ++mt)
#pragma unroll
            for (int nm = 0; nm < D::NM; ++nm) {
              const double b = i ? bo[c][nm].y : bo[c][nm].x;
              if (c < 2) aq_dmma(Vt[mt][nm][0], Vt[mt][nm][1], g[c][mt][i], b);
              else aq_dmma(Vd[mt][nm][0], Vd[mt][nm][1], g[2][mt][i], b);
            }
    }
    // ---- stage A^T (FMA): y[m][l] over the lane's q = 2 mt + h, partner lane (h ^ 1) adds the rest
    double yp[D::NM][2][D::N1];
#pragma unroll
    for (int nm = 0; nm < D::NM; ++nm)
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int l = 0; l < D::N1; ++l) yp[nm][i][l] = 0.0;
#pragma unroll
    for (int mt = 0; mt < D::MTQ; ++mt) {
      const int q = 2 * mt + h;
      if (q < D::QV) {
#pragma unroll
        for (int l = 0; l < D::N1; ++l) {
          const double bt = sBt[q * D::N1 + l], dt = sDt[q * D::N1 + l];
#pragma unroll
          for (int nm = 0; nm < D::NM; ++nm)
#pragma unroll
            for (int i = 0; i < 2; ++i)
              yp[nm][i][l] = fma(Vt[mt][nm][i], bt, fma(Vd[mt][nm][i], dt, yp[nm][i][l]));
        }
      }
    }
#pragma unroll
    for (int nm = 0; nm < D::NM; ++nm)
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int l = 0; l < D::N1; ++l) yp[nm][i][l] += __shfl_xor_sync(0xffffffffu, yp[nm][i][l], 16);
    if (ev) {
#pragma unroll
      for (int nm = 0; nm < D::NM; ++nm)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int m = 8 * nm + 2 * c4 + i;
          if (m < D::NT) {
#pragma unroll
            for (int l = 0; l < D::N1; ++l) {
              if ((l < D::NYL) != (h == 0)) continue;   // lane h = 0 scatters the lower l, h = 1 the upper
              const int gq = __ldg(ce + m + D::NT * l);
              if (gq >= 0) atomicAdd(y + gq, sgn * yp[nm][i][l]);
              else if (flags & AP_SCATTER_ALL) atomicAdd(y + ~gq, sgn * yp[nm][i][l]);
            }
          }
        }
    }
  }
}

template <int P>
static void apply_quad_P(sem_ctx* c, const DeviceLevel& L, const double* u, double* y, int flags) {
  using D = AQ<P>;
  static int grid_maxes[kMaxDev] = {0};
  const int dev = cur_device();
  int& grid_max = grid_maxes[dev];
  if (!grid_max) {
    CUDA_CHECK(cudaFuncSetAttribute(k_apply_quad<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, D::SMEM));
    int per_sm = 0, sms = 0;
    CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_apply_quad<P>, 32 * D::W, D::SMEM));
    grid_max = sms * (per_sm > 0 ? per_sm : 1);
  }
  if (c->E_own == 0) return;
  const int nquad = (c->E_own + 3) / 4;
  const int need = (nquad + D::W - 1) / D::W;
  const int grid = need < grid_max ? need : grid_max;
  k_apply_quad<P><<<grid, 32 * D::W, D::SMEM, c->stream>>>(c->E_own, L.conn, L.Gw, L.qmats, u, y, flags);
  CUDA_CHECK(cudaGetLastError());
}

bool launch_apply_quad(sem_ctx* c, int level, const double* u, double* y, int flags) {
  const DeviceLevel& L = c->L[level];
  if (!L.qmats || !L.Gw) return false;
  switch (L.p) {
    case 3: apply_quad_P<3>(c, L, u, y, flags); break;
    case 4: apply_quad_P<4>(c, L, u, y, flags); break;
    case 5: apply_quad_P<5>(c, L, u, y, flags); break;
    default: return false;
  }
  c->launches++;
  return true;
}


// ---------------------------------------------------------------------------------------------
// k_apply_qs<P>: the same four-element quad, split over MTQ warps (one per row tile mt of the
// (q, e) rows, i.e. vertical points q = 2 mt, 2 mt + 1).  Same arithmetic as k_apply_quad per row
// tile; what changes is the register footprint: a warp holds only its tile's stage-A fragments
// and stage-B^T accumulators (~130 registers instead of 242), so 15-16 warps fit per SM (4 per
// scheduler instead of 2) and the DMMA / shared-memory latencies of one warp hide behind the
// others.  The quad's data are shared by its group of warps:
//   * u gathered once per quad into shared memory (cp.async, all the group's threads);
//   * the geometric factors of the quad's current a-tile: one ring of R slots per group, filled
//     by four TMA bulk copies (one per element) issued by the group's first warp, "full" mbarrier
//     (tx bytes) waited on by every warp, "empty" mbarrier (one arrival per warp) waited on by the
//     producer before it refills a slot;
//   * stage A^T writes each warp's partial y (its two q values summed by one xor-16 shuffle) to a
//     per-warp shared buffer; after a group barrier the group sums the MTQ partials in a fixed
//     order and scatters with FP64 atomics, element-major (coalesced connectivity reads).
// Group barriers are named barriers (bar.sync 1 + group, 32 MTQ threads).
template <int P, int PZ = P>
struct AS {
  using B = AQ<P, PZ>;
  static constexpr int N1 = B::N1, NV = B::NV, NT = B::NT, QT = B::QT, QV = B::QV, Q = B::Q, N = B::N;
  static constexpr int MW = B::MTQ;             // warps per quad group (row tiles)
  static constexpr int R = 2;
  static constexpr int KM = B::KM, MTA = B::MTA, NM = B::NM, NALAST = B::NALAST, QE = B::QE, LDA = B::LDA;
  static constexpr int TSE = B::TSE, TS = B::TS, UST = B::UST, NYL = B::NYL;
  static constexpr int BT = B::BT, BM = B::BM;
  // B_c[a][m] at [m][a] in shared memory with row offsets ro(m) = m LDB + 4 ((m >> 1) & 1), LDB = 8 mod 16:
  // conflict-free for both the 8-byte stage-B loads (half-warp: m = 4 ks + c4, a = 8 na + r4) and the
  // 16-byte stage-B^T loads (quarter-warp: m = 8 nm + r4, a pair 8 na + 2 c4)
  static constexpr int LDB = ((8 * MTA + 4 + 7) / 16) * 16 + 8;
  static constexpr int CSB = 8 * NM * LDB + 8;  // component stride
  static constexpr int BMT = 3 * CSB;
  static constexpr int SU = 4 * UST, SY = MW * 4 * N, SC = 4 * N;
  static constexpr int NGQ = (4 * N + 32 * MW - 1) / (32 * MW);   // scatter entries per thread
  static constexpr int GD = R * TS + SU + SY;   // doubles per group
  // groups per CTA: measured for the isotropic orders; anisotropic levels take as many as fit in
  // 227 KB of shared memory and 16 warps (<= 128 registers per thread)
  static constexpr int GB = GD * 8 + SC * 4 + 2 * R * 8;
  static constexpr int NGS = (227 * 1024 - (BMT + BT) * 8) / GB, NGW = 16 / MW;
  static constexpr int NG = P == PZ ? (P == 3 ? 8 : P == 6 ? 3 : 5) : (NGS < NGW ? (NGS < 8 ? NGS : 8) : (NGW < 8 ? NGW : 8));
  static constexpr int W = MW * NG;
  static constexpr int SMEM = (BMT + BT + NG * GD) * 8 + NG * SC * 4 + NG * 2 * R * 8;
  static_assert(LDB % 16 == 8 && LDB >= 8 * MTA + 4, "qs operand layout");
  static_assert(SMEM <= 227 * 1024, "apply_qs shared memory");
};

__device__ __forceinline__ void qs_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void qs_wait(uint32_t mb, uint32_t par) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(mb), "r"(par)
        : "memory");
}

template <int P, int PZ>
__global__ void __launch_bounds__(32 * AS<P, PZ>::W, 1)
    k_apply_qs(int E, const int32_t* __restrict__ conn, const double* __restrict__ Gw,
               const double* __restrict__ mats, const double* __restrict__ u, double* __restrict__ y, int flags,
               const int32_t* __restrict__ elist) {
  using D = AS<P, PZ>;
  extern __shared__ __align__(128) double sm[];
  double* BmT = sm;
  double* sBt = BmT + D::BMT;
  double* sDt = sBt + D::QV * D::NV;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = warp / D::MW, mt = warp % D::MW, gt = tid - grp * 32 * D::MW;
  const int r4 = lane >> 2, c4 = lane & 3, el = r4 & 3, h = r4 >> 2, q = 2 * mt + h;
  double* gbase = sBt + D::BT + grp * D::GD;
  double* ring = gbase;                       // [R][4][TSE]
  double* su = ring + D::R * D::TS;           // [4][UST]
  double* yb = su + D::SU;                    // [MW][4][N]
  int32_t* scn = reinterpret_cast<int32_t*>(sBt + D::BT + D::NG * D::GD) + grp * D::SC;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(reinterpret_cast<int32_t*>(sBt + D::BT + D::NG * D::GD) +
                                               D::NG * D::SC) + grp * 2 * D::R;   // full[R], empty[R]
  {  // BmT (global: [3][8 NM][LDA]) -> shared rows at ro(m); then Bt, Dt
    constexpr int RW = 8 * D::MTA, CW = 8 * D::NM * RW;
    for (int i = tid; i < 3 * CW; i += 32 * D::W) {
      const int c = i / CW, m = (i - c * CW) / RW, a = i - c * CW - m * RW;
      sm[c * D::CSB + m * D::LDB + 4 * ((m >> 1) & 1) + a] = __ldg(mats + D::BM + (c * 8 * D::NM + m) * D::LDA + a);
    }
    for (int i = tid; i < D::BT; i += 32 * D::W) sBt[i] = __ldg(mats + D::BM + AQ<P, PZ>::BMT + i);
  }
  if (gt == 0) {
    for (int b = 0; b < D::R; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(aq_smem(mbar + b)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(aq_smem(mbar + D::R + b)), "r"(D::MW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int gbar = 1 + grp, gthr = 32 * D::MW;
  const double sgn = (flags & AP_NEGATE) ? -1.0 : 1.0;
  const int nquad = (E + 3) >> 2;
  const int qstride = gridDim.x * D::NG;
  const int q0 = blockIdx.x * D::NG + grp;
  auto elem = [&](int i) { return elist ? __ldg(elist + i) : i; };
  // copy t of this group: quad q0 + (t / MTA) qstride, a-tile t % MTA, slot t % R
  auto issue = [&](int t) {
    const int qd = q0 + (t / D::MTA) * qstride, ma = t % D::MTA;
    if (qd >= nquad) return;
    if (t >= D::R) qs_wait(aq_smem(mbar + D::R + t % D::R), (uint32_t)((t / D::R) - 1) & 1u);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int ne = min(4, E - 4 * qd);
    const uint32_t one = (uint32_t)(6 * D::QV * (ma < D::MTA - 1 ? 8 : D::NALAST)) * 8u;
    const uint32_t mb = aq_smem(mbar + t % D::R);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(one * ne) : "memory");
    for (int k = 0; k < ne; ++k)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              aq_smem(ring + (t % D::R) * D::TS + k * D::TSE)),
          "l"(Gw + (size_t)elem(4 * qd + k) * 6 * D::Q + (size_t)ma * 48 * D::QV), "r"(one), "r"(mb)
          : "memory");
  };
  // the gather of the next quad is staged by the group's last warp alone (its own cp.async
  // groups and __syncwarp: no group barrier), the producer of the G ring is the first warp
  const bool stager = mt == D::MW - 1;
  auto stage_conn = [&](int qd) {
    const int ne = min(4, E - 4 * qd);
    for (int i = lane; i < ne * D::N; i += 32) {
      const int k = i / D::N;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(aq_smem(scn + i)),
                   "l"(conn + (size_t)elem(4 * qd + k) * D::N + (i - k * D::N))
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto stage_u = [&](int qd) {
    const int nval = min(4, E - 4 * qd) * D::N;
    for (int i = lane; i < D::SC; i += 32) {
      const int g = i < nval ? scn[i] : INT_MIN;
      const bool take = g >= 0 || (g != INT_MIN && (flags & AP_GATHER_ALL));
      const double* src = u + (take ? (g >= 0 ? g : ~g) : 0);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(aq_smem(su + (i / D::N) * D::UST + i % D::N)),
                   "l"(src), "r"(take ? 8 : 0)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (q0 < nquad) {
    if (gt == 0)
      for (int t = 0; t < D::R; ++t) issue(t);
    if (stager) {
      stage_conn(q0);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      stage_u(q0);
    }
  }
  int tk = 0;
  for (int qd = q0; qd < nquad; qd += qstride, tk += D::MTA) {
    const bool ev = 4 * qd + el < E;
    // ---- stage A (FMA): this warp's A fragments, m = 4 ks + c4, q = 2 mt + h
    double Ua[D::KM], Ud[D::KM];
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    qs_bar(gbar, gthr);   // u of this quad visible; the previous quad's yb consumed
    const int ne = min(4, E - 4 * qd);
    int gq[D::NGQ];       // scatter targets of this thread (scn is refilled for the next quad below)
#pragma unroll
    for (int k = 0; k < D::NGQ; ++k) {
      const int i = gt + k * gthr;
      gq[k] = i < ne * D::N ? scn[i] : INT_MIN;
    }
#pragma unroll
    for (int ks = 0; ks < D::KM; ++ks) Ua[ks] = Ud[ks] = 0.0;
    if (q < D::QV) {
#pragma unroll
      for (int l = 0; l < D::NV; ++l) {
        const double bt = sBt[q * D::NV + l], dt = sDt[q * D::NV + l];
#pragma unroll
        for (int ks = 0; ks < D::KM; ++ks) {
          const int m = 4 * ks + c4;
          const double uu = (ev && m < D::NT) ? su[el * D::UST + m + D::NT * l] : 0.0;
          Ua[ks] = fma(uu, bt, Ua[ks]);
          Ud[ks] = fma(uu, dt, Ud[ks]);
        }
      }
    }
    qs_bar(gbar, gthr);   // su and scn free
    const int qn = qd + qstride;
    if (stager && qn < nquad) stage_conn(qn);
    double Vt[D::NM][2], Vd[D::NM][2];
#pragma unroll
    for (int nm = 0; nm < D::NM; ++nm) Vt[nm][0] = Vt[nm][1] = Vd[nm][0] = Vd[nm][1] = 0.0;
#pragma unroll 1
    for (int na = 0; na < D::MTA; ++na) {
      const int t = tk + na;
      if (stager && na == D::MTA / 2 && qn < nquad) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        stage_u(qn);
      }
      qs_wait(aq_smem(mbar + t % D::R), (uint32_t)(t / D::R) & 1u);
      // ---- stage B: g_c^T[(q,e)][a] of this warp's row tile
      double g[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int ks = 0; ks < D::KM; ++ks) {
        const int m = 4 * ks + c4, off = m * D::LDB + 4 * ((m >> 1) & 1) + 8 * na + r4;
        const double br = BmT[off], bs = BmT[D::CSB + off], b0 = BmT[2 * D::CSB + off];
        aq_dmma(g[0][0], g[0][1], Ua[ks], br);
        aq_dmma(g[1][0], g[1][1], Ua[ks], bs);
        aq_dmma(g[2][0], g[2][1], Ud[ks], b0);
      }
      // ---- w = G g at (a = 8 na + 2 c4 + i, q)
      const int nat = (na < D::MTA - 1) ? 8 : D::NALAST;
      const double* Gt = ring + (t % D::R) * D::TS + el * D::TSE;
      const int cs = D::QV * nat;
      const int qp = (q & 1) ? D::QE + (q >> 1) : (q >> 1);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int al = 2 * c4 + i;
        double w0 = 0.0, w1 = 0.0, w2 = 0.0;
        if (ev && q < D::QV && al < nat) {
          const double* gp = Gt + qp * nat + al;
          double gxx, gxy, gxz, gyy, gyz, gzz;
          if ((D::NALAST & 1) == 0 || na < D::MTA - 1) {
            const double2 v0 = *reinterpret_cast<const double2*>(gp - i);
            const double2 v1 = *reinterpret_cast<const double2*>(gp - i + cs);
            const double2 v2 = *reinterpret_cast<const double2*>(gp - i + 2 * cs);
            const double2 v3 = *reinterpret_cast<const double2*>(gp - i + 3 * cs);
            const double2 v4 = *reinterpret_cast<const double2*>(gp - i + 4 * cs);
            const double2 v5 = *reinterpret_cast<const double2*>(gp - i + 5 * cs);
            gxx = i ? v0.y : v0.x;
            gxy = i ? v1.y : v1.x;
            gxz = i ? v2.y : v2.x;
            gyy = i ? v3.y : v3.x;
            gyz = i ? v4.y : v4.x;
            gzz = i ? v5.y : v5.x;
          } else {
            gxx = gp[0];
            gxy = gp[cs];
            gxz = gp[2 * cs];
            gyy = gp[3 * cs];
            gyz = gp[4 * cs];
            gzz = gp[5 * cs];
          }
          const double x0 = g[0][i], x1 = g[1][i], x2 = g[2][i];
          w0 = gxx * x0 + gxy * x1 + gxz * x2;
          w1 = gxy * x0 + gyy * x1 + gyz * x2;
          w2 = gxz * x0 + gyz * x1 + gzz * x2;
        }
        g[0][i] = w0;
        g[1][i] = w1;
        g[2][i] = w2;
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(aq_smem(mbar + D::R + t % D::R)) : "memory");
      if (mt == 0 && lane == 0) issue(t + D::R);
      // ---- stage B^T: V^T[(q,e)][m] += w^T[(q,e)][a] B_c[a][m]; k-step i <-> a = 8 na + 2 c4 + i
      double2 bo[3][D::NM];
#pragma unroll
      for (int nm = 0; nm < D::NM; ++nm) {
        const int m = 8 * nm + r4, off = m * D::LDB + 4 * ((m >> 1) & 1) + 8 * na + 2 * c4;
#pragma unroll
        for (int c = 0; c < 3; ++c) bo[c][nm] = *reinterpret_cast<const double2*>(BmT + c * D::CSB + off);
      }
      // component order r, 0, s: the two updates of a Vt accumulator per k-step are 2 NM apart
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
#pragma unroll
          for (int nm = 0; nm < D::NM; ++nm) {
            const int c = cc == 0 ? 0 : (cc == 1 ? 2 : 1);
            const double b = i ? bo[c][nm].y : bo[c][nm].x;
            if (c < 2) aq_dmma(Vt[nm][0], Vt[nm][1], g[c][i], b);
            else aq_dmma(Vd[nm][0], Vd[nm][1], g[2][i], b);
          }
    }
    // ---- stage A^T (FMA): partial y of this warp's two q values -> yb[mt]
    double* ybw = yb + mt * 4 * D::N + el * D::N;
#pragma unroll
    for (int l = 0; l < D::NV; ++l) {
      const double bt = q < D::QV ? sBt[q * D::NV + l] : 0.0, dt = q < D::QV ? sDt[q * D::NV + l] : 0.0;
      double yl[D::NM][2];
#pragma unroll
      for (int nm = 0; nm < D::NM; ++nm)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const double v = fma(Vt[nm][i], bt, Vd[nm][i] * dt);
          yl[nm][i] = v + __shfl_xor_sync(0xffffffffu, v, 16);
        }
      if ((l < D::NYL) == (h == 0)) {
#pragma unroll
        for (int nm = 0; nm < D::NM; ++nm)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int m = 8 * nm + 2 * c4 + i;
            if (m < D::NT) ybw[m + D::NT * l] = yl[nm][i];
          }
      }
    }
    qs_bar(gbar, gthr);
    // ---- sum the MW partials (fixed order) and scatter, element-major
#pragma unroll
    for (int k = 0; k < D::NGQ; ++k) {
      const int i = gt + k * gthr, g = gq[k];
      if (g == INT_MIN) continue;
      double acc = yb[i];
#pragma unroll
      for (int w = 1; w < D::MW; ++w) acc += yb[w * 4 * D::N + i];
      if (g >= 0) atomicAdd(y + g, sgn * acc);
      else if (flags & AP_SCATTER_ALL) atomicAdd(y + ~g, sgn * acc);
    }
  }
}

template <int P, int PZ>
static void apply_qs_P(sem_ctx* c, const DeviceLevel& L, const double* u, double* y, int flags,
                       const int32_t* elist, int ne) {
  using D = AS<P, PZ>;
  static int grid_maxes[kMaxDev] = {0};
  const int dev = cur_device();
  int& grid_max = grid_maxes[dev];
  if (!grid_max) {
    CUDA_CHECK(cudaFuncSetAttribute(k_apply_qs<P, PZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, D::SMEM));
    int per_sm = 0, sms = 0;
    CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_apply_qs<P, PZ>, 32 * D::W, D::SMEM));
    grid_max = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int E = elist ? ne : c->E_own;
  if (E == 0) return;
  const int nquad = (E + 3) / 4;
  const int need = (nquad + D::NG - 1) / D::NG;
  const int grid = need < grid_max ? need : grid_max;
  k_apply_qs<P, PZ><<<grid, 32 * D::W, D::SMEM, c->stream>>>(E, L.conn, L.Gw, L.qmats, u, y, flags, elist);
  CUDA_CHECK(cudaGetLastError());
}

bool launch_apply_qs(sem_ctx* c, int level, const double* u, double* y, int flags, const int32_t* elist, int ne) {
  const DeviceLevel& L = c->L[level];
  if (!L.qmats || !L.Gw) return false;
#define QS_CASE(P_, Q_) \
  else if (L.p == P_ && L.q == Q_) apply_qs_P<P_, Q_>(c, L, u, y, flags, elist, ne);
  if (false) {
  }
  QS_CASE(3, 3) QS_CASE(4, 4) QS_CASE(5, 5) QS_CASE(6, 6)
  QS_CASE(3, 1) QS_CASE(3, 2) QS_CASE(3, 4) QS_CASE(3, 5)
  QS_CASE(4, 1) QS_CASE(4, 2) QS_CASE(4, 3) QS_CASE(4, 5)
  QS_CASE(5, 1) QS_CASE(5, 2) QS_CASE(5, 3) QS_CASE(5, 4)
  else return false;
#undef QS_CASE
  c->launches++;
  return true;
}

}  // namespace sem
