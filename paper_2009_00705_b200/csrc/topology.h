// Host topology of the prism mesh: global node numbering of V^p,
// Dirichlet nodes, prolongation owners (reading O17), Schwarz subdomains
// (eq 4.4-4.6, reading O15) and their element lists.
#pragma once
#include <cstdint>
#include <unordered_map>
#include <vector>

namespace sem {

struct HostMesh {
  int32_t nv = 0, E = 0;
  std::vector<double> xyz;        // [nv][3]
  std::vector<int32_t> prism;     // [E][6]
  std::vector<uint8_t> tag;       // [E][5]
};

// Edges / faces of the mesh, identified once and shared by all levels.
struct Entities {
  std::vector<int32_t> edge;      // [E][9]: bottom (01,12,20), top (01,12,20), vertical (0,1,2)
  std::vector<int32_t> tface;     // [E][2]: bottom, top triangle
  std::vector<int32_t> qface;     // [E][3]: lateral quads over edges 01, 12, 20
  int32_t n_edge = 0, n_tface = 0, n_qface = 0;
};
Entities build_entities(const HostMesh& m);

struct LevelTopo {
  int p = 0, q = 0, N = 0;          // horizontal / vertical order (q = p isotropic)
  int64_t n = 0, nfree = 0;
  std::vector<int32_t> conn;      // [E][N] global ids (unsigned)
  std::vector<uint8_t> dir;       // [n] 1 = Dirichlet
  std::vector<uint8_t> owner;     // [E][N] 1 = first occurrence of the node in element order
};
// throws std::runtime_error on bad input
LevelTopo number_level(const HostMesh& m, const Entities& ent, int p, int q = -1);

struct SchwarzTopo {
  std::vector<int64_t> off;       // [E+1] into idx (unpadded)
  std::vector<int32_t> idx;       // sorted free node ids of subdomain k
  std::vector<int64_t> eoff;      // [E+1] into elist
  std::vector<int32_t> elist;     // elements holding >= 1 node of subdomain k
  std::vector<double> W;          // [n] 1/count on free nodes, 0 on Dirichlet (eq 4.6)
  int max_nk = 0;
};
SchwarzTopo schwarz_topology(const LevelTopo& L, int E, int overlap, int nthreads);
// the subdomains k with keep[k] == 0 (W is left to the caller)
SchwarzTopo schwarz_subset(const SchwarzTopo& S, const std::vector<uint8_t>& keep_if_zero);

}  // namespace sem
