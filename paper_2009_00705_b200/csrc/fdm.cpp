// Host topology and operators of the FDM local solves (reading O33; fdm.h).
// Independent of oracle/ (which finds vertical lines by coordinates): here the
// lines come from the prism stacking (a prism's top triangle is the bottom
// triangle of the prism above) and the global numbering.
#include "fdm.h"

#include <omp.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <string>

#include "internal.h"
#include "refelem.h"

namespace sem {

namespace {
[[noreturn]] void unsupported(const std::string& s) {
  throw SemError(SEM_EUNSUPPORTED, "FDM local solves need a layered prism mesh: " + s);
}
}  // namespace

FdmTopo fdm_topology(const HostMesh& m, const LevelTopo& L, const std::vector<double>& X, int pg, int overlap,
                     int qg) {
  FdmTopo F;
  // p: horizontal order (triangle patches, 2D operators); q: vertical order (node lines, 1D operators)
  const int p = L.p, q = L.q > 0 ? L.q : L.p, Nt = n_tri(p), N = L.N, E = m.E;
  if (qg < 0) qg = pg;
  F.p = p;
  F.q = q;
  F.overlap = overlap;
  // ---- 1. stacking: columns and layers
  struct KE {
    std::array<int32_t, 3> k;
    int32_t e;
  };
  auto tri_key = [&](int e, int f) {
    std::array<int32_t, 3> s = {m.prism[(size_t)e * 6 + 3 * f], m.prism[(size_t)e * 6 + 3 * f + 1],
                                m.prism[(size_t)e * 6 + 3 * f + 2]};
    std::sort(s.begin(), s.end());
    return s;
  };
  std::vector<KE> bot(E);
  for (int e = 0; e < E; ++e) bot[e] = {tri_key(e, 0), e};
  std::sort(bot.begin(), bot.end(), [](const KE& a, const KE& b) { return a.k < b.k; });
  for (int i = 1; i < E; ++i)
    if (bot[i].k == bot[i - 1].k) unsupported("two prisms share a bottom triangle");
  std::vector<int32_t> above(E, -1), below(E, -1);
  for (int e = 0; e < E; ++e) {
    const auto t = tri_key(e, 1);
    auto it = std::lower_bound(bot.begin(), bot.end(), t, [](const KE& a, const std::array<int32_t, 3>& k) {
      return a.k < k;
    });
    if (it != bot.end() && it->k == t) {
      above[e] = it->e;
      below[it->e] = e;
    }
  }
  F.col.assign(E, -1);
  F.layer.assign(E, -1);
  std::vector<int32_t> colbot, nlay;
  for (int e = 0; e < E; ++e) {
    if (below[e] != -1) continue;
    const int c = (int)colbot.size();
    colbot.push_back(e);
    int j = 0;
    for (int x = e; x != -1; x = above[x]) {
      if (F.col[x] != -1) unsupported("cyclic stacking");
      F.col[x] = c;
      F.layer[x] = j++;
    }
    nlay.push_back(j);
  }
  for (int e = 0; e < E; ++e)
    if (F.col[e] == -1) unsupported("cyclic stacking");
  const int ncol = (int)colbot.size();
  F.ncol = ncol;
  // ---- 2. 2D node ids: the bottom-level nodes of every column, carried up the stack
  std::vector<int32_t> h2(L.n, -1), eh((size_t)E * Nt);
  int32_t nh2 = 0;
  for (int c = 0; c < ncol; ++c) {
    const int e0 = colbot[c];
    for (int mm = 0; mm < Nt; ++mm) {
      const int32_t g = L.conn[(size_t)e0 * N + mm];
      if (h2[g] < 0) h2[g] = nh2++;
      eh[(size_t)e0 * Nt + mm] = h2[g];
    }
    for (int x = e0; above[x] != -1; x = above[x]) {
      const int y = above[x];
      for (int mm = 0; mm < Nt; ++mm) {
        const int32_t g = L.conn[(size_t)y * N + mm];
        int found = -1;
        for (int m2 = 0; m2 < Nt; ++m2)
          if (L.conn[(size_t)x * N + m2 + (size_t)Nt * q] == g) found = m2;
        if (found < 0) unsupported("stacked prisms do not share their nodes");
        eh[(size_t)y * Nt + mm] = eh[(size_t)x * Nt + found];
      }
    }
  }
  // ---- 3. vertical lines: node (h, z) with z = layer * q + l
  std::vector<int32_t> linelen(nh2, 0);
  for (int e = 0; e < E; ++e)
    for (int mm = 0; mm < Nt; ++mm) {
      int32_t& ll = linelen[eh[(size_t)e * Nt + mm]];
      ll = std::max(ll, (F.layer[e] + 1) * q + 1);
    }
  std::vector<int64_t> lineoff(nh2 + 1, 0);
  for (int h = 0; h < nh2; ++h) lineoff[h + 1] = lineoff[h] + linelen[h];
  std::vector<int32_t> vline(lineoff[nh2], -1);
  std::vector<int64_t> pos(L.n, -1);
  for (int e = 0; e < E; ++e)
    for (int n = 0; n < N; ++n) {
      const int mm = n % Nt, l = n / Nt;
      const int64_t s = lineoff[eh[(size_t)e * Nt + mm]] + F.layer[e] * q + l;
      const int32_t g = L.conn[(size_t)e * N + n];
      if ((vline[s] != -1 && vline[s] != g) || (pos[g] != -1 && pos[g] != s)) unsupported("nodes off their lines");
      vline[s] = g;
      pos[g] = s;
    }
  // ---- 4. 2D lattice graph (O15 on one level) and node -> column incidence
  std::vector<int> li, lj;
  for (int j = 0; j <= p; ++j)
    for (int i = 0; i <= p - j; ++i) { li.push_back(i); lj.push_back(j); }
  std::vector<std::pair<int, int>> steps;
  for (int a = 0; a < Nt; ++a)
    for (int b = 0; b < Nt; ++b) {
      const int di = li[a] - li[b], dj = lj[a] - lj[b], dk = -(di + dj);
      if (std::abs(di) + std::abs(dj) + std::abs(dk) == 2) steps.push_back({a, b});
    }
  std::vector<int64_t> aoff(nh2 + 1, 0), coff(nh2 + 1, 0);
  for (int c = 0; c < ncol; ++c) {
    const int32_t* t = &eh[(size_t)colbot[c] * Nt];
    for (auto& st : steps) aoff[t[st.first] + 1]++;
    for (int mm = 0; mm < Nt; ++mm) coff[t[mm] + 1]++;
  }
  for (int h = 0; h < nh2; ++h) { aoff[h + 1] += aoff[h]; coff[h + 1] += coff[h]; }
  std::vector<int32_t> adj(aoff[nh2]), cinc(coff[nh2]);
  {
    std::vector<int64_t> fa(aoff.begin(), aoff.end() - 1), fc(coff.begin(), coff.end() - 1);
    for (int c = 0; c < ncol; ++c) {
      const int32_t* t = &eh[(size_t)colbot[c] * Nt];
      for (auto& st : steps) adj[fa[t[st.first]]++] = t[st.second];
      for (int mm = 0; mm < Nt; ++mm) cinc[fc[t[mm]]++] = c;
    }
  }
  // ---- 5. reference data: 2D collapsed cubature, 1D GLL operators
  const LevelRef R = make_level_ref(p, q);
  std::vector<double> wt(R.qt, 0.0);
  for (int a = 0; a < R.qt; ++a)
    for (int k = 0; k < R.qv; ++k) wt[a] += R.wq[a + R.qt * k];
  for (auto& w : wt) w *= 0.5;  // sum of the vertical GL weights is 2
  const Rule1D gv = gauss_legendre_rule(q + 1);
  std::vector<double> Kref(R.n1 * R.n1, 0.0), Mref(R.n1 * R.n1, 0.0);
  for (int a = 0; a < R.n1; ++a)
    for (int b = 0; b < R.n1; ++b)
      for (int k = 0; k < R.qv; ++k) {
        Kref[a * R.n1 + b] += gv.w[k] * R.Dt[k * R.n1 + a] * R.Dt[k * R.n1 + b];
        Mref[a * R.n1 + b] += gv.w[k] * R.Bt[k * R.n1 + a] * R.Bt[k * R.n1 + b];
      }
  const int Ntg = n_tri(pg), Ng = Ntg * (qg + 1);
  const int corner[3] = {0, pg, Ntg - 1};  // lattice (0,0), (pg,0), (0,pg) = v0, v1, v2
  auto xyz = [&](int e, int n, int i) { return X[((size_t)e * Ng + n) * 3 + i]; };
  // 2D element operators of every column [ncol][Nt][Nt]
  std::vector<double> Kt((size_t)ncol * Nt * Nt), Mt((size_t)ncol * Nt * Nt);
#pragma omp parallel for schedule(static)
  for (int c = 0; c < ncol; ++c) {
    const int e0 = colbot[c];
    const double x0 = xyz(e0, corner[0], 0), y0 = xyz(e0, corner[0], 1);
    const double J00 = 0.5 * (xyz(e0, corner[1], 0) - x0), J01 = 0.5 * (xyz(e0, corner[2], 0) - x0);
    const double J10 = 0.5 * (xyz(e0, corner[1], 1) - y0), J11 = 0.5 * (xyz(e0, corner[2], 1) - y0);
    const double det = J00 * J11 - J01 * J10;
    const double i00 = J11 / det, i01 = -J01 / det, i10 = -J10 / det, i11 = J00 / det;  // d(r,s)/d(x,y)
    double* K = &Kt[(size_t)c * Nt * Nt];
    double* M = &Mt[(size_t)c * Nt * Nt];
    std::fill(K, K + Nt * Nt, 0.0);
    std::fill(M, M + Nt * Nt, 0.0);
    for (int a = 0; a < R.qt; ++a) {
      const double w = wt[a] * std::fabs(det);
      const double* B0 = &R.B0[a * Nt];
      const double* Br = &R.Br[a * Nt];
      const double* Bs = &R.Bs[a * Nt];
      for (int i = 0; i < Nt; ++i) {
        const double xi = Br[i] * i00 + Bs[i] * i10, yi = Br[i] * i01 + Bs[i] * i11;
        for (int j = 0; j < Nt; ++j) {
          const double xj = Br[j] * i00 + Bs[j] * i10, yj = Br[j] * i01 + Bs[j] * i11;
          K[i * Nt + j] += w * (xi * xj + yi * yj);
          M[i * Nt + j] += w * B0[i] * B0[j];
        }
      }
    }
  }
  // ---- 6. horizontal patches and their operators (per column)
  std::vector<std::vector<int32_t>> patch(ncol);
  std::vector<std::vector<double>> pK(ncol), pM(ncol);
#pragma omp parallel
  {
    std::vector<int32_t> stamp(nh2, -1), cstamp(ncol, -1), cur, nxt;
#pragma omp for schedule(dynamic, 64)
    for (int c = 0; c < ncol; ++c) {
      std::vector<int32_t>& H = patch[c];
      H.clear();
      cur.clear();
      const int32_t* t = &eh[(size_t)colbot[c] * Nt];
      for (int mm = 0; mm < Nt; ++mm)
        if (stamp[t[mm]] != c) { stamp[t[mm]] = c; cur.push_back(t[mm]); H.push_back(t[mm]); }
      for (int d = 0; d < overlap; ++d) {
        nxt.clear();
        for (int32_t h : cur)
          for (int64_t s = aoff[h]; s < aoff[h + 1]; ++s)
            if (stamp[adj[s]] != c) { stamp[adj[s]] = c; nxt.push_back(adj[s]); H.push_back(adj[s]); }
        cur.swap(nxt);
      }
      std::sort(H.begin(), H.end());
      const int nh = (int)H.size();
      auto where = [&](int32_t h) {
        auto it = std::lower_bound(H.begin(), H.end(), h);
        return (it != H.end() && *it == h) ? (int)(it - H.begin()) : -1;
      };
      pK[c].assign((size_t)nh * nh, 0.0);
      pM[c].assign((size_t)nh * nh, 0.0);
      for (int32_t h : H)
        for (int64_t s = coff[h]; s < coff[h + 1]; ++s) {
          const int t2 = cinc[s];
          if (cstamp[t2] == c) continue;
          cstamp[t2] = c;
          const int32_t* tt = &eh[(size_t)colbot[t2] * Nt];
          int loc[64];
          for (int mm = 0; mm < Nt; ++mm) loc[mm] = where(tt[mm]);
          for (int a = 0; a < Nt; ++a) {
            if (loc[a] < 0) continue;
            for (int b = 0; b < Nt; ++b) {
              if (loc[b] < 0) continue;
              pK[c][(size_t)loc[a] * nh + loc[b]] += Kt[((size_t)t2 * Nt + a) * Nt + b];
              pM[c][(size_t)loc[a] * nh + loc[b]] += Mt[((size_t)t2 * Nt + a) * Nt + b];
            }
          }
        }
    }
  }
  F.hoff.assign(ncol + 1, 0);
  F.moff.assign(ncol + 1, 0);
  for (int c = 0; c < ncol; ++c) {
    const int64_t nh = (int64_t)patch[c].size();
    F.hoff[c + 1] = F.hoff[c] + nh;
    F.moff[c + 1] = F.moff[c] + nh * nh;
    F.nh_max = std::max<int>(F.nh_max, (int)nh);
  }
  F.hnode.resize(F.hoff[ncol]);
  F.Kh.resize(F.moff[ncol]);
  F.Mh.resize(F.moff[ncol]);
  for (int c = 0; c < ncol; ++c) {
    std::copy(patch[c].begin(), patch[c].end(), F.hnode.begin() + F.hoff[c]);
    std::copy(pK[c].begin(), pK[c].end(), F.Kh.begin() + F.moff[c]);
    std::copy(pM[c].begin(), pM[c].end(), F.Mh.begin() + F.moff[c]);
  }
  // ---- 7. vertical boxes and 1D operators (layer thickness = mean of the 3 vertical edges)
  std::vector<int32_t> colel((size_t)0);
  std::vector<int64_t> cfirst(ncol + 1, 0);
  for (int c = 0; c < ncol; ++c) cfirst[c + 1] = cfirst[c] + nlay[c];
  colel.resize(cfirst[ncol]);
  for (int e = 0; e < E; ++e) colel[cfirst[F.col[e]] + F.layer[e]] = e;
  F.z0.assign(E, 0);
  F.nv.assign(E, 0);
  for (int e = 0; e < E; ++e) {
    const int c = F.col[e], j = F.layer[e], Zc = nlay[c] * q;
    const int32_t* t = &eh[(size_t)colbot[c] * Nt];
    auto dlev = [&](int z) {  // z-level of the column made of Dirichlet nodes only
      for (int mm = 0; mm < Nt; ++mm)
        if (!L.dir[vline[lineoff[t[mm]] + z]]) return false;
      return true;
    };
    int lo = std::max(0, j * q - overlap), hi = std::min(Zc, j * q + q + overlap);
    while (lo <= hi && dlev(lo)) ++lo;
    while (hi >= lo && dlev(hi)) --hi;
    for (int z = lo; z <= hi; ++z)
      if (dlev(z)) unsupported("a Dirichlet level inside a column");
    if (hi < lo) unsupported("an element made of Dirichlet nodes only");
    F.z0[e] = lo;
    F.nv[e] = hi - lo + 1;
    F.nv_max = std::max(F.nv_max, F.nv[e]);
  }
  F.voff.assign(E + 1, 0);
  F.ioff.assign(E + 1, 0);
  for (int e = 0; e < E; ++e) {
    F.voff[e + 1] = F.voff[e] + (int64_t)F.nv[e] * F.nv[e];
    F.ioff[e + 1] = F.ioff[e] + (F.hoff[F.col[e] + 1] - F.hoff[F.col[e]]) * F.nv[e];
  }
  F.Kv.assign(F.voff[E], 0.0);
  F.Mv.assign(F.voff[E], 0.0);
  F.idx.resize(F.ioff[E]);
#pragma omp parallel for schedule(dynamic, 256)
  for (int e = 0; e < E; ++e) {
    const int c = F.col[e], nv = F.nv[e], lo = F.z0[e];
    double* Kv = &F.Kv[F.voff[e]];
    double* Mv = &F.Mv[F.voff[e]];
    for (int jj = 0; jj < nlay[c]; ++jj) {  // layers overlapping [lo, lo+nv)
      const int zb = jj * q;
      if (zb + q < lo || zb > lo + nv - 1) continue;
      const int x = colel[cfirst[c] + jj];
      double d = 0.0;
      for (int v = 0; v < 3; ++v)
        d += xyz(x, corner[v] + Ntg * qg, 2) - xyz(x, corner[v], 2);
      d /= 3.0;
      for (int a = 0; a <= q; ++a)
        for (int b = 0; b <= q; ++b) {
          const int za = zb + a - lo, zb2 = zb + b - lo;
          if (za < 0 || za >= nv || zb2 < 0 || zb2 >= nv) continue;
          Kv[za * nv + zb2] += (2.0 / d) * Kref[a * R.n1 + b];
          Mv[za * nv + zb2] += (d / 2.0) * Mref[a * R.n1 + b];
        }
    }
    const int64_t h0 = F.hoff[c], nh = F.hoff[c + 1] - h0;
    int32_t* out = &F.idx[F.ioff[e]];
    for (int64_t a = 0; a < nh; ++a) {
      const int32_t h = F.hnode[h0 + a];
      for (int z = 0; z < nv; ++z) {
        int32_t g = (lo + z < linelen[h]) ? vline[lineoff[h] + lo + z] : -1;
        if (g >= 0 && L.dir[g]) g = -1;
        out[a * nv + z] = g;
      }
    }
  }
  // ---- 8. column view
  F.cfirst = cfirst;
  F.colel = colel;
  F.nzc.resize(ncol);
  F.cioff.assign(ncol + 1, 0);
  for (int c = 0; c < ncol; ++c) {
    F.nzc[c] = nlay[c] * q + 1;
    F.cioff[c + 1] = F.cioff[c] + (F.hoff[c + 1] - F.hoff[c]) * F.nzc[c];
  }
  F.cidx.resize(F.cioff[ncol]);
#pragma omp parallel for schedule(static)
  for (int c = 0; c < ncol; ++c) {
    const int64_t h0 = F.hoff[c], nh = F.hoff[c + 1] - h0;
    const int nz = F.nzc[c];
    for (int64_t a = 0; a < nh; ++a) {
      const int32_t h = F.hnode[h0 + a];
      for (int z = 0; z < nz; ++z) {
        int32_t g = (z < linelen[h]) ? vline[lineoff[h] + z] : -1;
        if (g >= 0 && L.dir[g]) g = -1;
        F.cidx[F.cioff[c] + a * nz + z] = g;
      }
    }
  }
  // ---- 9. regular boxes (reading O35): every column touching the patch widened by one element
  //         ring (lattice radius overlap + p) as tall as the element's own column
  {
    std::vector<uint8_t> creg(ncol, 1);
    const int radius = overlap + p;
#pragma omp parallel
    {
      std::vector<int32_t> stamp(nh2, -1), cur, nxt, ball;
#pragma omp for schedule(dynamic, 64)
      for (int c = 0; c < ncol; ++c) {
        cur.clear();
        ball.clear();
        const int32_t* t = &eh[(size_t)colbot[c] * Nt];
        for (int mm = 0; mm < Nt; ++mm)
          if (stamp[t[mm]] != c) { stamp[t[mm]] = c; cur.push_back(t[mm]); ball.push_back(t[mm]); }
        for (int d = 0; d < radius; ++d) {
          nxt.clear();
          for (int32_t h : cur)
            for (int64_t s2 = aoff[h]; s2 < aoff[h + 1]; ++s2)
              if (stamp[adj[s2]] != c) { stamp[adj[s2]] = c; nxt.push_back(adj[s2]); ball.push_back(adj[s2]); }
          cur.swap(nxt);
        }
        for (int32_t h : ball) {
          for (int64_t s2 = coff[h]; s2 < coff[h + 1]; ++s2)
            if (nlay[cinc[s2]] != nlay[c]) { creg[c] = 0; break; }
          if (!creg[c]) break;
        }
      }
    }
    F.regular.resize(E);
    for (int e = 0; e < E; ++e) F.regular[e] = creg[F.col[e]];
  }
  // ---- 10. weights (eq 4.6) over the FDM subdomains
  std::vector<double> cnt(L.n, 0.0);
  for (int32_t g : F.idx)
    if (g >= 0) cnt[g] += 1.0;
  F.W.assign(L.n, 0.0);
  for (int64_t i = 0; i < L.n; ++i)
    if (!L.dir[i]) {
      if (cnt[i] == 0.0) unsupported("a free node outside every subdomain");
      F.W[i] = 1.0 / cnt[i];
    }
  return F;
}

FdmTopo fdm_local(const FdmTopo& G, const std::vector<int32_t>& elems, int E_own, const std::vector<int32_t>& gid,
                  int64_t n_global, const std::vector<double>& Wg) {
  FdmTopo F;
  F.p = G.p;
  F.q = G.q;
  F.overlap = G.overlap;
  std::vector<int32_t> gloc(n_global, -1);
  for (size_t i = 0; i < gid.size(); ++i) gloc[gid[i]] = (int32_t)i;
  auto lid = [&](int32_t g) {
    if (g < 0) return -1;
    const int32_t l = gloc[g];
    if (l < 0) throw SemError(SEM_EINVAL, "FDM partition: a box node is not held by the rank");
    return (int)l;
  };
  const int Eg = (int)G.col.size();
  std::vector<int32_t> eloc(Eg, -1);
  for (int k = 0; k < E_own; ++k) eloc[elems[k]] = k;
  // local columns: the owned elements' columns in ascending global column id
  std::vector<int32_t> gcols;
  for (int k = 0; k < E_own; ++k) gcols.push_back(G.col[elems[k]]);
  std::sort(gcols.begin(), gcols.end());
  gcols.erase(std::unique(gcols.begin(), gcols.end()), gcols.end());
  const int ncol = (int)gcols.size();
  F.ncol = ncol;
  std::vector<int32_t> cloc(G.ncol, -1);
  for (int q = 0; q < ncol; ++q) cloc[gcols[q]] = q;
  F.hoff.assign(ncol + 1, 0);
  F.moff.assign(ncol + 1, 0);
  F.cfirst.assign(ncol + 1, 0);
  F.cioff.assign(ncol + 1, 0);
  F.nzc.resize(ncol);
  for (int q = 0; q < ncol; ++q) {
    const int gc = gcols[q];
    const int64_t nh = G.hoff[gc + 1] - G.hoff[gc];
    F.hoff[q + 1] = F.hoff[q] + nh;
    F.moff[q + 1] = F.moff[q] + nh * nh;
    F.nh_max = std::max<int>(F.nh_max, (int)nh);
    F.hnode.insert(F.hnode.end(), G.hnode.begin() + G.hoff[gc], G.hnode.begin() + G.hoff[gc + 1]);
    F.Kh.insert(F.Kh.end(), G.Kh.begin() + G.moff[gc], G.Kh.begin() + G.moff[gc + 1]);
    F.Mh.insert(F.Mh.end(), G.Mh.begin() + G.moff[gc], G.Mh.begin() + G.moff[gc + 1]);
    for (int64_t j = G.cfirst[gc]; j < G.cfirst[gc + 1]; ++j) {
      const int k = eloc[G.colel[j]];
      if (k < 0) throw SemError(SEM_EINVAL, "FDM partition: a column split between ranks");
      F.colel.push_back(k);
    }
    F.cfirst[q + 1] = (int64_t)F.colel.size();
    F.nzc[q] = G.nzc[gc];
    for (int64_t t = G.cioff[gc]; t < G.cioff[gc + 1]; ++t) F.cidx.push_back(lid(G.cidx[t]));
    F.cioff[q + 1] = (int64_t)F.cidx.size();
  }
  F.col.resize(E_own);
  F.layer.resize(E_own);
  F.z0.resize(E_own);
  F.nv.resize(E_own);
  F.regular.resize(E_own);
  F.voff.assign(E_own + 1, 0);
  F.ioff.assign(E_own + 1, 0);
  for (int k = 0; k < E_own; ++k) {
    const int e = elems[k];
    F.col[k] = cloc[G.col[e]];
    F.layer[k] = G.layer[e];
    F.z0[k] = G.z0[e];
    F.nv[k] = G.nv[e];
    F.regular[k] = G.regular[e];
    F.nv_max = std::max(F.nv_max, F.nv[k]);
    F.Kv.insert(F.Kv.end(), G.Kv.begin() + G.voff[e], G.Kv.begin() + G.voff[e + 1]);
    F.Mv.insert(F.Mv.end(), G.Mv.begin() + G.voff[e], G.Mv.begin() + G.voff[e + 1]);
    F.voff[k + 1] = (int64_t)F.Kv.size();
    for (int64_t t = G.ioff[e]; t < G.ioff[e + 1]; ++t) F.idx.push_back(lid(G.idx[t]));
    F.ioff[k + 1] = (int64_t)F.idx.size();
  }
  F.W.resize(gid.size());
  for (size_t i = 0; i < gid.size(); ++i) F.W[i] = Wg[gid[i]];
  return F;
}

}  // namespace sem
