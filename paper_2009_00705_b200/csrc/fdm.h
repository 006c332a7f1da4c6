// Fast-diagonalisation (FDM) local solves of the Schwarz smoother (reading
// O33): on layered prism meshes subdomain k is the product of a
// horizontal node patch H_k (2D lattice ball of radius `overlap` around the
// footprint triangle, O15) and a vertical node range V_k, and the local block
// of eq 4.4 is replaced by
//     B~_k = K_h[H,H] (x) M_v[V,V] + M_h[H,H] (x) K_v[V,V]
// (Lottes & Fischer, the paper's [FL05]), inverted as
//     (S_h (x) S_v) (L_h (x) I + I (x) L_v)^-1 (S_h (x) S_v)^T
// with K S = M S L, S^T M S = I per direction.  Exact on straight prisms with
// flat layers (config 1).
#pragma once
#include <cstdint>
#include <vector>

#include "topology.h"

namespace sem {

struct FdmTopo {
  int p = 0, q = 0, overlap = 0;        // horizontal / vertical order (q = p isotropic)
  int ncol = 0;
  int nh_max = 0, nv_max = 0;
  std::vector<int32_t> col, layer;      // [E] column and layer (0 = bottom) of every element
  // per column: horizontal patch (2D node ids, ascending) and its 2D operators
  std::vector<int64_t> hoff;            // [ncol+1] into hnode
  std::vector<int32_t> hnode;
  std::vector<int64_t> moff;            // [ncol+1] into Kh / Mh (nh^2 each, row-major)
  std::vector<double> Kh, Mh;
  // per element: vertical box [z0, z0+nv) and its 1D operators
  std::vector<int32_t> z0, nv;
  std::vector<int64_t> voff;            // [E+1] into Kv / Mv (nv^2 each)
  std::vector<double> Kv, Mv;
  // per element: global ids of the box nodes, box order (h outer, z inner), -1 = absent or Dirichlet
  std::vector<int64_t> ioff;            // [E+1]
  std::vector<int32_t> idx;
  std::vector<double> W;                // [n] eq 4.6 from the FDM subdomains (0 on Dirichlet)
  std::vector<uint8_t> regular;         // [E] reading O35: every column touching the patch as tall as the element's
  // column view for the column-batched kernel: elements of every column in layer order,
  // and the node ids of the whole column patch [nh][Z_c+1] (-1 = absent or Dirichlet)
  std::vector<int64_t> cfirst;          // [ncol+1] into colel
  std::vector<int32_t> colel;
  std::vector<int32_t> nzc;             // [ncol] Z_c + 1
  std::vector<int64_t> cioff;           // [ncol+1] into cidx
  std::vector<int32_t> cidx;
};

// The FDM topology of one rank's partition: the owned elements elems[0, E_own)
// (whole columns), node ids mapped to the rank's local numbering (gid: local ->
// global), W taken from the global hybrid weights Wg.  Throws if a box node is
// not held by the rank.
FdmTopo fdm_local(const FdmTopo& G, const std::vector<int32_t>& elems, int E_own, const std::vector<int32_t>& gid,
                  int64_t n_global, const std::vector<double>& Wg);

// X: [E][N(pg)][3] nodal map of order pg (the finest order; x, y are taken as
// affine per triangle from its corner nodes, z-thicknesses from the corners).
// Throws SemError(SEM_EUNSUPPORTED) if the mesh is not a stack of prism layers.
// pg, qg: horizontal / vertical order of the fine nodal map X (qg < 0: qg = pg)
FdmTopo fdm_topology(const HostMesh& m, const LevelTopo& L, const std::vector<double>& X, int pg, int overlap,
                     int qg = -1);

}  // namespace sem
