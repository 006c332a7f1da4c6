// Element partition for the multi-GPU solve (the paper has none,
// P:572 "ongoing work").  Whole vertical columns of prisms go to one rank
// (recursive coordinate bisection of column centroids); each rank holds its
// owned elements plus the halo elements its Schwarz subdomains touch.
#pragma once
#include <cstdint>
#include <vector>

#include "fdm.h"
#include "topology.h"

namespace sem {

// rank of every element: RCB on the (x, y) centroids of the elements' six
// vertices; elements with the same (x, y) centroid (one column) never split.
std::vector<int> partition_columns(const std::vector<double>& cx, const std::vector<double>& cy, int nranks);

struct LocalLevel {
  int64_t n = 0, nfree = 0;
  std::vector<int32_t> gid;      // local -> global node id (ascending)
  std::vector<int32_t> conn;     // [E_loc][N] local node ids (unsigned)
  std::vector<uint8_t> dir;      // [n]
  std::vector<uint8_t> owner;    // [E_loc][N] global owner-element flags (0 on halo elements)
  std::vector<uint8_t> owned;    // [n] 1 if this rank owns the node (dots, single-count init)
  std::vector<double> W;         // [n] Schwarz weights (global counts)
  SchwarzTopo S;                 // owned subdomains, local ids (levels < coarsest)
  std::vector<int> nbr;          // neighbour ranks sharing nodes
  std::vector<std::vector<int32_t>> xidx;  // per neighbour: local ids of shared nodes, ascending global id
};

struct LocalPart {
  int rank = 0, nranks = 1;
  std::vector<int32_t> elems;    // local -> global element id: owned (ascending) then halo (ascending)
  int E_own = 0;
  std::vector<LocalLevel> L;
  std::vector<FdmTopo> F;         // opts.local_solve = 1: per level < coarsest, the rank's FDM topology
};

// topo[l]: global numbering per level; sch[l]: global Schwarz topology for
// l < nl-1 (all subdomains); epart: rank of each element.
LocalPart extract_part(const std::vector<LevelTopo>& topo, const std::vector<SchwarzTopo>& sch,
                       const std::vector<int>& epart, int rank, int nranks);

}  // namespace sem
