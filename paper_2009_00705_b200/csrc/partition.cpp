#include "partition.h"

#include <algorithm>
#include <numeric>
#include <stdexcept>

namespace sem {

namespace {
void rcb(std::vector<int>& idx, size_t lo, size_t hi, int r0, int nr, const std::vector<double>& cx,
         const std::vector<double>& cy, std::vector<int>& part) {
  if (nr == 1) {
    for (size_t i = lo; i < hi; ++i) part[idx[i]] = r0;
    return;
  }
  double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
  for (size_t i = lo; i < hi; ++i) {
    xmin = std::min(xmin, cx[idx[i]]);
    xmax = std::max(xmax, cx[idx[i]]);
    ymin = std::min(ymin, cy[idx[i]]);
    ymax = std::max(ymax, cy[idx[i]]);
  }
  const bool byx = (xmax - xmin) >= (ymax - ymin);
  const std::vector<double>& a = byx ? cx : cy;
  const std::vector<double>& b = byx ? cy : cx;
  std::sort(idx.begin() + lo, idx.begin() + hi, [&](int i, int j) {
    if (a[i] != a[j]) return a[i] < a[j];
    if (b[i] != b[j]) return b[i] < b[j];
    return i < j;
  });
  const int nl = nr / 2;
  size_t cut = lo + (size_t)((double)(hi - lo) * nl / nr);
  // never split a column: move the cut past elements with the same (x, y)
  while (cut > lo && cut < hi && a[idx[cut]] == a[idx[cut - 1]] && b[idx[cut]] == b[idx[cut - 1]]) ++cut;
  rcb(idx, lo, cut, r0, nl, cx, cy, part);
  rcb(idx, cut, hi, r0 + nl, nr - nl, cx, cy, part);
}
}  // namespace

std::vector<int> partition_columns(const std::vector<double>& cx, const std::vector<double>& cy, int nranks) {
  const size_t E = cx.size();
  std::vector<int> part(E, 0), idx(E);
  std::iota(idx.begin(), idx.end(), 0);
  if (nranks > 1) rcb(idx, 0, E, 0, nranks, cx, cy, part);
  return part;
}

LocalPart extract_part(const std::vector<LevelTopo>& topo, const std::vector<SchwarzTopo>& sch,
                       const std::vector<int>& epart, int rank, int nranks) {
  if (nranks > 64) throw std::runtime_error("at most 64 ranks");
  const int nl = (int)topo.size();
  const int E = (int)epart.size();
  LocalPart P;
  P.rank = rank;
  P.nranks = nranks;
  // which ranks hold each element: its owner plus the owners of every subdomain (any level) touching it
  std::vector<uint64_t> held(E, 0);
  for (int e = 0; e < E; ++e) held[e] = 1ull << epart[e];
  for (int l = 0; l + 1 < nl; ++l) {
    const SchwarzTopo& S = sch[l];
    for (int k = 0; k < E; ++k)
      for (int64_t t = S.eoff[k]; t < S.eoff[k + 1]; ++t) held[S.elist[t]] |= 1ull << epart[k];
  }
  const uint64_t me = 1ull << rank;
  for (int e = 0; e < E; ++e)
    if (epart[e] == rank) P.elems.push_back(e);
  P.E_own = (int)P.elems.size();
  for (int e = 0; e < E; ++e)
    if (epart[e] != rank && (held[e] & me)) P.elems.push_back(e);
  std::vector<int32_t> eloc(E, -1);
  for (size_t i = 0; i < P.elems.size(); ++i) eloc[P.elems[i]] = (int32_t)i;
  P.L.resize(nl);
  for (int l = 0; l < nl; ++l) {
    const LevelTopo& T = topo[l];
    LocalLevel& L = P.L[l];
    const int N = T.N;
    // node holders and node owner rank (rank of the first element holding the node)
    std::vector<uint64_t> nh(T.n, 0);
    std::vector<int> orank(T.n, -1);
    for (int e = 0; e < E; ++e)
      for (int n = 0; n < N; ++n) {
        const int32_t g = T.conn[(size_t)e * N + n];
        nh[g] |= held[e];
        if (T.owner[(size_t)e * N + n]) orank[g] = epart[e];
      }
    std::vector<int32_t> loc(T.n, -1);
    for (int64_t g = 0; g < T.n; ++g)
      if (nh[g] & me) {
        loc[g] = (int32_t)L.gid.size();
        L.gid.push_back((int32_t)g);
      }
    L.n = (int64_t)L.gid.size();
    L.dir.resize(L.n);
    L.owned.resize(L.n);
    for (int64_t i = 0; i < L.n; ++i) {
      const int32_t g = L.gid[i];
      L.dir[i] = T.dir[g];
      L.owned[i] = orank[g] == rank;
      if (!L.dir[i]) L.nfree++;
    }
    const size_t El = P.elems.size();
    L.conn.resize(El * N);
    L.owner.assign(El * N, 0);
    for (size_t i = 0; i < El; ++i) {
      const int e = P.elems[i];
      for (int n = 0; n < N; ++n) {
        L.conn[i * N + n] = loc[T.conn[(size_t)e * N + n]];
        if ((int)i < P.E_own) L.owner[i * N + n] = T.owner[(size_t)e * N + n];
      }
    }
    // exchange lists: shared nodes with every other holder
    std::vector<std::vector<int32_t>> lists(nranks);
    for (int64_t i = 0; i < L.n; ++i) {
      uint64_t m = nh[L.gid[i]] & ~me;
      while (m) {
        const int q = __builtin_ctzll(m);
        m &= m - 1;
        lists[q].push_back((int32_t)i);
      }
    }
    for (int q = 0; q < nranks; ++q)
      if (!lists[q].empty()) {
        L.nbr.push_back(q);
        L.xidx.push_back(std::move(lists[q]));
      }
    if (l + 1 < nl) {
      const SchwarzTopo& S = sch[l];
      L.W.resize(L.n);
      for (int64_t i = 0; i < L.n; ++i) L.W[i] = S.W[L.gid[i]];
      L.S.off.assign(P.E_own + 1, 0);
      L.S.eoff.assign(P.E_own + 1, 0);
      for (int k = 0; k < P.E_own; ++k) {
        const int kg = P.elems[k];
        for (int64_t t = S.off[kg]; t < S.off[kg + 1]; ++t) L.S.idx.push_back(loc[S.idx[t]]);
        for (int64_t t = S.eoff[kg]; t < S.eoff[kg + 1]; ++t) L.S.elist.push_back(eloc[S.elist[t]]);
        // local ids of the subdomain stay ascending (global ids ascending, loc monotone)
        std::sort(L.S.elist.begin() + L.S.eoff[k], L.S.elist.end());
        L.S.off[k + 1] = (int64_t)L.S.idx.size();
        L.S.eoff[k + 1] = (int64_t)L.S.elist.size();
        L.S.max_nk = std::max<int>(L.S.max_nk, (int)(L.S.off[k + 1] - L.S.off[k]));
      }
      for (auto v : L.S.idx)
        if (v < 0) throw std::runtime_error("partition: subdomain node outside the local set");
      for (auto v : L.S.elist)
        if (v < 0) throw std::runtime_error("partition: subdomain element outside the local set");
      L.S.W = L.W;
    }
  }
  return P;
}

}  // namespace sem
