#include "topology.h"

#include <omp.h>

#include <algorithm>
#include <array>
#include <stdexcept>
#include <string>

namespace sem {

namespace {
struct Key3 {
  int32_t a, b, c;
  bool operator==(const Key3& o) const { return a == o.a && b == o.b && c == o.c; }
};
struct Key4 {
  int32_t a, b, c, d;
  bool operator==(const Key4& o) const { return a == o.a && b == o.b && c == o.c && d == o.d; }
};
struct H3 {
  size_t operator()(const Key3& k) const {
    uint64_t h = (uint64_t)(uint32_t)k.a * 0x9E3779B97F4A7C15ull;
    h ^= (uint64_t)(uint32_t)k.b * 0xC2B2AE3D27D4EB4Full + (h << 6) + (h >> 2);
    h ^= (uint64_t)(uint32_t)k.c * 0x165667B19E3779F9ull + (h << 6) + (h >> 2);
    return (size_t)h;
  }
};
struct H4 {
  size_t operator()(const Key4& k) const {
    H3 h3;
    uint64_t h = h3(Key3{k.a, k.b, k.c});
    h ^= (uint64_t)(uint32_t)k.d * 0x27D4EB2F165667C5ull + (h << 6) + (h >> 2);
    return (size_t)h;
  }
};
}  // namespace

Entities build_entities(const HostMesh& m) {
  Entities ent;
  const int E = m.E;
  ent.edge.resize((size_t)E * 9);
  ent.tface.resize((size_t)E * 2);
  ent.qface.resize((size_t)E * 3);
  std::unordered_map<uint64_t, int32_t> emap;
  std::unordered_map<Key3, int32_t, H3> tmap;
  std::unordered_map<Key4, int32_t, H4> qmap;
  emap.reserve((size_t)E * 4);
  tmap.reserve((size_t)E * 2);
  qmap.reserve((size_t)E * 2);
  static const int he[3][2] = {{0, 1}, {1, 2}, {2, 0}};
  for (int e = 0; e < E; ++e) {
    const int32_t* v = &m.prism[(size_t)e * 6];
    auto edge_id = [&](int32_t a, int32_t b) {
      uint64_t k = ((uint64_t)(uint32_t)std::min(a, b) << 32) | (uint32_t)std::max(a, b);
      auto it = emap.find(k);
      if (it != emap.end()) return it->second;
      int32_t id = ent.n_edge++;
      emap.emplace(k, id);
      return id;
    };
    for (int t = 0; t < 3; ++t) {
      ent.edge[(size_t)e * 9 + t] = edge_id(v[he[t][0]], v[he[t][1]]);
      ent.edge[(size_t)e * 9 + 3 + t] = edge_id(v[3 + he[t][0]], v[3 + he[t][1]]);
      ent.edge[(size_t)e * 9 + 6 + t] = edge_id(v[t], v[3 + t]);
    }
    for (int f = 0; f < 2; ++f) {
      std::array<int32_t, 3> s = {v[3 * f], v[3 * f + 1], v[3 * f + 2]};
      std::sort(s.begin(), s.end());
      Key3 k{s[0], s[1], s[2]};
      auto it = tmap.find(k);
      int32_t id;
      if (it != tmap.end()) id = it->second;
      else { id = ent.n_tface++; tmap.emplace(k, id); }
      ent.tface[(size_t)e * 2 + f] = id;
    }
    for (int t = 0; t < 3; ++t) {
      std::array<int32_t, 4> s = {v[he[t][0]], v[he[t][1]], v[3 + he[t][0]], v[3 + he[t][1]]};
      std::sort(s.begin(), s.end());
      Key4 k{s[0], s[1], s[2], s[3]};
      auto it = qmap.find(k);
      int32_t id;
      if (it != qmap.end()) id = it->second;
      else { id = ent.n_qface++; qmap.emplace(k, id); }
      ent.qface[(size_t)e * 3 + t] = id;
    }
  }
  return ent;
}

LevelTopo number_level(const HostMesh& m, const Entities& ent, int p, int qz) {
  // P_p(triangle) x P_q(t): p - 1 nodes per triangle edge, q - 1 per vertical
  // edge, (p - 1)(q - 1) per lateral quad face, nti (q - 1) per element interior
  const int q = qz < 0 ? p : qz;
  LevelTopo L;
  L.p = p;
  L.q = q;
  const int nt = (p + 1) * (p + 2) / 2, n1 = q + 1, N = nt * n1;
  L.N = N;
  const int E = m.E;
  L.conn.resize((size_t)E * N);
  L.owner.assign((size_t)E * N, 0);
  // entity bases (first touch); -1 = unassigned
  std::vector<int64_t> vbase(m.nv, -1), ebase(ent.n_edge, -1), tbase(ent.n_tface, -1), qbase(ent.n_qface, -1);
  const int ne = p - 1, nev = q - 1, nti = (p - 1) * (p - 2) / 2, nq = (p - 1) * (q - 1);
  int64_t next = 0;
  auto take = [&](std::vector<int64_t>& base, int32_t id, int cnt) {
    if (base[id] < 0) { base[id] = next; next += cnt; }
    return base[id];
  };
  // local lattice
  std::vector<int> li(N), lj(N), ll(N);
  {
    int n = 0;
    for (int l = 0; l < n1; ++l)
      for (int j = 0; j <= p; ++j)
        for (int i = 0; i <= p - j; ++i) { li[n] = i; lj[n] = j; ll[n] = l; ++n; }
  }
  // interior triangle index of (i,j) with i,j,k >= 1 (local order)
  std::vector<int> tri_int((p + 1) * (p + 1), -1);
  {
    int c = 0;
    for (int j = 0; j <= p; ++j)
      for (int i = 0; i <= p - j; ++i)
        if (i >= 1 && j >= 1 && p - i - j >= 1) tri_int[j * (p + 1) + i] = c++;
  }
  std::vector<uint8_t> seen;
  seen.reserve(1 << 20);
  int int_e = -1;
  int64_t int_base = -1;
  static const int he[3][2] = {{0, 1}, {1, 2}, {2, 0}};
  for (int e = 0; e < E; ++e) {
    const int32_t* v = &m.prism[(size_t)e * 6];
    for (int n = 0; n < N; ++n) {
      const int i = li[n], j = lj[n], l = ll[n], k = p - i - j;
      const int zeros = (i == 0) + (j == 0) + (k == 0);
      const int vert = (l == 0) ? 0 : (l == q ? 1 : 2);  // bottom, top, middle
      int64_t gid;
      if (zeros == 2) {  // triangle vertex t
        const int t = (k == p) ? 0 : (i == p ? 1 : 2);
        if (vert < 2) {
          gid = take(vbase, v[3 * vert + t], 1);
        } else {  // vertical edge, position l from the bottom vertex
          int32_t a = v[t], b = v[3 + t];
          int s = (a < b) ? l : q - l;
          gid = take(ebase, ent.edge[(size_t)e * 9 + 6 + t], nev) + (s - 1);
        }
      } else if (zeros == 1) {  // triangle edge
        int te, s;  // edge index (01, 12, 20) and position from its first vertex
        if (j == 0) { te = 0; s = i; }
        else if (k == 0) { te = 1; s = j; }
        else { te = 2; s = k; }
        const int ta = he[te][0], tb = he[te][1];
        if (vert < 2) {
          int32_t a = v[3 * vert + ta], b = v[3 * vert + tb];
          int ss = (a < b) ? s : p - s;
          gid = take(ebase, ent.edge[(size_t)e * 9 + 3 * vert + te], ne) + (ss - 1);
        } else {  // lateral quad face interior: canonical origin at the min corner
          int32_t c00 = v[ta], cp0 = v[tb], c0p = v[3 + ta], cpp = v[3 + tb];
          int32_t mn = std::min(std::min(c00, cp0), std::min(c0p, cpp));
          int ss = (mn == cp0 || mn == cpp) ? p - s : s;
          int lv = (mn == c0p || mn == cpp) ? q - l : l;
          gid = take(qbase, ent.qface[(size_t)e * 3 + te], nq) + (int64_t)(ss - 1) * (q - 1) + (lv - 1);
        }
      } else {  // triangle interior
        if (vert < 2) {
          std::array<std::pair<int32_t, int>, 3> vw = {std::make_pair(v[3 * vert + 0], k),
                                                        std::make_pair(v[3 * vert + 1], i),
                                                        std::make_pair(v[3 * vert + 2], j)};
          std::sort(vw.begin(), vw.end());
          const int wb = vw[1].second, wc = vw[2].second;
          int off = 0;
          for (int c = 1; c < wc; ++c) off += p - 1 - c;
          off += wb - 1;
          gid = take(tbase, ent.tface[(size_t)e * 2 + vert], nti) + off;
        } else {
          // element interior: one block per element, taken at the first interior node met
          if (int_e != e) { int_e = e; int_base = next; next += (int64_t)nti * (q - 1); }
          int64_t base = int_base;
          gid = base + (int64_t)tri_int[j * (p + 1) + i] * (q - 1) + (l - 1);
        }
      }
      if (gid >= (int64_t)INT32_MAX) throw std::runtime_error("node count exceeds int32");
      L.conn[(size_t)e * N + n] = (int32_t)gid;
      if ((size_t)gid >= seen.size()) seen.resize(std::max<size_t>(seen.size() * 2, gid + 1), 0);
      if (!seen[gid]) { seen[gid] = 1; L.owner[(size_t)e * N + n] = 1; }
    }
  }
  L.n = next;
  // Dirichlet: nodes of faces tagged 1 (bot l=0, top l=p, q01 j=0, q12 k=0, q20 i=0)
  L.dir.assign(L.n, 0);
  for (int e = 0; e < E; ++e) {
    const uint8_t* tg = &m.tag[(size_t)e * 5];
    for (int f = 0; f < 5; ++f) {
      if (tg[f] > 2) throw std::runtime_error("bad face tag");
      if (tg[f] != 1) continue;
      for (int n = 0; n < N; ++n) {
        const int i = li[n], j = lj[n], l = ll[n], k = p - i - j;
        bool on = (f == 0 && l == 0) || (f == 1 && l == q) || (f == 2 && j == 0) || (f == 3 && k == 0) ||
                  (f == 4 && i == 0);
        if (on) L.dir[L.conn[(size_t)e * N + n]] = 1;
      }
    }
  }
  int64_t nd = 0;
  for (auto d : L.dir) nd += d;
  L.nfree = L.n - nd;
  return L;
}

SchwarzTopo schwarz_topology(const LevelTopo& L, int E, int overlap, int nthreads) {
  SchwarzTopo S;
  const int p = L.p, q = L.q > 0 ? L.q : L.p, N = L.N;
  const int64_t n = L.n;
  // lattice pattern of reading O15: |dl| <= 1 and horizontal offset 0 or one
  // triangular-lattice step (barycentric offsets +-(1,-1,0) and permutations)
  std::vector<int> li(N), lj(N), ll(N);
  {
    int c = 0;
    for (int l = 0; l <= q; ++l)
      for (int j = 0; j <= p; ++j)
        for (int i = 0; i <= p - j; ++i) { li[c] = i; lj[c] = j; ll[c] = l; ++c; }
  }
  std::vector<std::vector<int>> pat(N);
  for (int a = 0; a < N; ++a)
    for (int b = 0; b < N; ++b) {
      if (a == b) continue;
      int di = li[a] - li[b], dj = lj[a] - lj[b];
      int dk = -(di + dj);
      int dl = ll[a] - ll[b];
      if (std::abs(dl) <= 1 && std::abs(di) + std::abs(dj) + std::abs(dk) <= 2) pat[a].push_back(b);
    }
  // node -> (element, local) incidence
  std::vector<int64_t> noff(n + 1, 0);
  for (size_t t = 0; t < L.conn.size(); ++t) noff[L.conn[t] + 1]++;
  for (int64_t i = 0; i < n; ++i) noff[i + 1] += noff[i];
  std::vector<int64_t> inc(L.conn.size());
  {
    std::vector<int64_t> fill(noff.begin(), noff.end() - 1);
    for (size_t t = 0; t < L.conn.size(); ++t) inc[fill[L.conn[t]]++] = (int64_t)t;  // t = e*N + local
  }
  std::vector<std::vector<int32_t>> sets(E), elists(E);
  int nth = std::max(1, nthreads);
#pragma omp parallel num_threads(nth)
  {
    std::vector<int32_t> stamp(n, -1), estamp(E, -1);
    std::vector<int32_t> cur, nxt, out, el;
#pragma omp for schedule(dynamic, 256)
    for (int k = 0; k < E; ++k) {
      cur.clear();
      out.clear();
      for (int a = 0; a < N; ++a) {
        int32_t g = L.conn[(size_t)k * N + a];
        if (stamp[g] != k) { stamp[g] = k; cur.push_back(g); out.push_back(g); }
      }
      for (int d = 0; d < overlap; ++d) {
        nxt.clear();
        for (int32_t g : cur) {
          for (int64_t t = noff[g]; t < noff[g + 1]; ++t) {
            int64_t en = inc[t];
            int64_t e2 = en / N;
            int a = (int)(en % N);
            for (int b : pat[a]) {
              int32_t h = L.conn[(size_t)e2 * N + b];
              if (stamp[h] != k) { stamp[h] = k; nxt.push_back(h); out.push_back(h); }
            }
          }
        }
        cur.swap(nxt);
      }
      std::vector<int32_t>& s = sets[k];
      s.clear();
      for (int32_t g : out)
        if (!L.dir[g]) s.push_back(g);
      std::sort(s.begin(), s.end());
      el.clear();
      for (int32_t g : s)
        for (int64_t t = noff[g]; t < noff[g + 1]; ++t) {
          int32_t e2 = (int32_t)(inc[t] / N);
          if (estamp[e2] != k) { estamp[e2] = k; el.push_back(e2); }
        }
      std::sort(el.begin(), el.end());
      elists[k] = el;
    }
  }
  S.off.assign(E + 1, 0);
  S.eoff.assign(E + 1, 0);
  for (int k = 0; k < E; ++k) {
    S.off[k + 1] = S.off[k] + (int64_t)sets[k].size();
    S.eoff[k + 1] = S.eoff[k] + (int64_t)elists[k].size();
    S.max_nk = std::max<int>(S.max_nk, (int)sets[k].size());
  }
  S.idx.resize(S.off[E]);
  S.elist.resize(S.eoff[E]);
  std::vector<double> cnt(n, 0.0);
  for (int k = 0; k < E; ++k) {
    std::copy(sets[k].begin(), sets[k].end(), S.idx.begin() + S.off[k]);
    std::copy(elists[k].begin(), elists[k].end(), S.elist.begin() + S.eoff[k]);
    for (int32_t g : sets[k]) cnt[g] += 1.0;
  }
  S.W.assign(n, 0.0);
  for (int64_t i = 0; i < n; ++i)
    if (!L.dir[i]) {
      if (cnt[i] == 0.0) throw std::runtime_error("free node outside every Schwarz subdomain");
      S.W[i] = 1.0 / cnt[i];
    }
  return S;
}

SchwarzTopo schwarz_subset(const SchwarzTopo& S, const std::vector<uint8_t>& keep_if_zero) {
  SchwarzTopo D;
  D.off.push_back(0);
  D.eoff.push_back(0);
  for (size_t k = 0; k + 1 < S.off.size(); ++k) {
    if (keep_if_zero[k]) continue;
    D.idx.insert(D.idx.end(), S.idx.begin() + S.off[k], S.idx.begin() + S.off[k + 1]);
    D.elist.insert(D.elist.end(), S.elist.begin() + S.eoff[k], S.elist.begin() + S.eoff[k + 1]);
    D.off.push_back((int64_t)D.idx.size());
    D.eoff.push_back((int64_t)D.elist.size());
    D.max_nk = std::max<int>(D.max_nk, (int)(S.off[k + 1] - S.off[k]));
  }
  D.W = S.W;
  return D;
}

}  // namespace sem
