// Internal structures of the C-ABI library (not installed).
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sem_pmg.h"
#include "refelem.h"
#include "topology.h"

namespace sem {

struct SemError : std::runtime_error {
  int code;
  SemError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CUDA_CHECK(x)                                                                          \
  do {                                                                                         \
    cudaError_t _e = (x);                                                                      \
    if (_e != cudaSuccess)                                                                     \
      throw ::sem::SemError(_e == cudaErrorMemoryAllocation ? SEM_ENOMEM : SEM_ECUDA,          \
                            std::string(#x) + ": " + cudaGetErrorString(_e));                  \
  } while (0)

// per-device caches of kernel attributes (dynamic shared-memory opt-in, grid size):
// cudaFuncSetAttribute acts on the current device only
constexpr int kMaxDev = 64;

// Every C-ABI entry point that touches the device switches to the ctx's device and
// restores the caller's current device on return.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    int cur = -1;
    if (dev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// NVTX range for the timeline of nsys / ncu (--nvtx): header-only nvtx3, no-ops unless a tool
// injects itself (SURVEY §5 tracing).  Host-side only: kernels replayed from CUDA graphs carry
// the range of the call that launched the graph.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
inline const char* nvtx_level_name(int li) {
  static const char* names[] = {"V-cycle level 0", "V-cycle level 1", "V-cycle level 2", "V-cycle level 3",
                                "V-cycle level 4", "V-cycle level 5", "V-cycle level 6", "V-cycle level 7",
                                "V-cycle level 8"};
  return (li >= 0 && li < 9) ? names[li] : "V-cycle level";
}

inline int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < kMaxDev) ? d : 0;
}

// opt a kernel in to `smem` bytes of dynamic shared memory on the current device
template <class F>
inline void smem_opt_in(F* f, int smem, int (&cache)[kMaxDev]) {
  const int d = cur_device();
  if (smem > cache[d]) {
    CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cache[d] = smem;
  }
}

// apply-kernel flags
enum : int {
  AP_GATHER_ALL = 1,   // read u on Dirichlet nodes too (else treated as 0)
  AP_SCATTER_ALL = 2,  // write y on Dirichlet nodes too (else skipped)
  AP_NEGATE = 4,       // y -= A u instead of y += A u
};

struct DeviceLevel {
  int p = 0, q = 0, N = 0, Q = 0;   // horizontal / vertical order (q = p isotropic)
  int64_t n = 0, nfree = 0;
  LevelRef ref;                 // host copy
  int32_t* conn = nullptr;      // [E][N], Dirichlet nodes stored as ~gid
  uint8_t* owner = nullptr;     // [E][N]
  uint8_t* dmask = nullptr;     // [n]
  double* G = nullptr;          // [E][6][Q]
  double* mats = nullptr;       // B0 Br Bs [qt][nt|1], Bt Dt [qv][n1]
  double* frag = nullptr;       // DMMA fragment-ordered reference operands (apply_dmma.cu)
  double* wmats = nullptr;      // reference operands of the warp-per-element apply (apply_warp.cu), p <= 6
  double* Gw = nullptr;         // a-tile-major copy of G for k_apply_warp / k_apply_quad
  double* qmats = nullptr;      // reference operands of the four-elements-per-warp apply (apply_quad.cu), 3 <= p <= 5
  double* Ae1 = nullptr;        // P <= 2 levels: packed element matrices [N(N+1)/2][E] (k_apply_em)
  // Schwarz (not on the coarsest level)
  int32_t* sidx = nullptr;      // padded to 16 per subdomain, -1 = padding
  int64_t* sidx_off = nullptr;  // [E+1] (padded offsets)
  int64_t* tile_off = nullptr;  // [E+1] offsets in doubles into tiles
  double* tiles = nullptr;
  float* tiles32 = nullptr;     // opts.mixed_precision: FP32 copy of the packed inverses (tiles unused)
  double* W = nullptr;          // [n]
  // FDM local solves (opts.local_solve = 1; fdm.cu, reading O33)
  int fdm = 0, f_nh_max = 0, f_nv_max = 0;
  int32_t* f_col = nullptr;     // [E] column of every element
  int64_t* f_cfirst = nullptr;  // [ncol+1] first element slot of every column in f_colel
  double* f_kmref = nullptr;    // [2][n1][n1] 1D GLL stiffness / mass of the reference layer
  int64_t *f_hoff = nullptr, *f_moff = nullptr;   // [ncol+1] patch / S_h offsets
  int32_t* f_nv = nullptr;      // [E] vertical box size
  int64_t *f_voff = nullptr, *f_lvoff = nullptr, *f_ioff = nullptr;   // [E(+1)] S_v / l_v / index offsets
  int32_t* f_idx = nullptr;     // box node ids (h outer, z inner), -1 = absent / Dirichlet
  double *f_Sh = nullptr, *f_lh = nullptr, *f_Sv = nullptr, *f_lv = nullptr;
  // column-batched kernel: work units (column, first element slot, elements, box columns)
  int4* f_units = nullptr;
  int f_nunits = 0, f_mt = 0, f_nvt = 0, f_warp = 0, f_ldr = 0, f_nph = 2;
  int* f_udesc = nullptr;       // [units][34] descriptors of k_fdm_warp
  double *f_Svp = nullptr, *f_lvp = nullptr;   // [E][8 nvt][8 nvt] / [E][8 nvt] zero-padded S_v, l_v
  int32_t *f_colel = nullptr, *f_nzc = nullptr, *f_cidx = nullptr, *f_z0 = nullptr;
  int64_t* f_cioff = nullptr;
  int64_t schwarz_bytes = 0;
  int64_t f_bytes = 0;          // algorithmic bytes of one FDM sweep (fdm.cu)
  int nsub = 0;                 // dense subdomains (all owned elements, or the O35 subset of an FDM level)
  uint8_t* f_skip = nullptr;    // [E] 1 = subdomain solved densely (O35), skipped by the FDM kernels
  // deterministic mode (opts.deterministic): colours of node-disjoint subdomains, one launch each
  std::vector<int64_t> scol_off, fcol_off;   // [colours+1] into scol / fcol
  int32_t *scol = nullptr, *fcol = nullptr;  // dense subdomain ids / FDM element ids, grouped by colour
  int64_t nk_sum = 0, packed = 0;
  int max_tiles_1d = 0;
  // transfer from the next coarser level (level+1 -> this)
  double* Itri = nullptr;       // [ntf][ntc]
  double* I1 = nullptr;         // [n1f][n1c]
  // work vectors
  double *u = nullptr, *f = nullptr, *r = nullptr;
  std::vector<double> xyz;      // host [n][3]
  std::vector<int32_t> conn_host;    // single domain: host connectivity / owner flags (geometry updates)
  std::vector<uint8_t> owner_host;
  std::vector<uint8_t> dir_host;
  // partitioned solve (dist.cu)
  std::vector<int32_t> gid_host;     // local -> global node id
  std::vector<uint8_t> owned_host;   // node owned by this rank
  int32_t* gid = nullptr;            // device copy of gid_host
  uint8_t* ownfree = nullptr;        // owned and free (dots, single-count RHS)
  uint8_t* owned_dev = nullptr;      // owned (gather of global outputs)
  double* d = nullptr;               // partial-sum work vector
  // neighbour exchange of shared nodes
  std::vector<int> nbr;
  std::vector<int64_t> xoff;         // [nbr+1] offsets into xidx / send / recv
  int32_t* xidx = nullptr;           // concatenated local ids
  int32_t* xnbr = nullptr;           // neighbour slot of every entry (unused by NCCL path)
  double *sendbuf = nullptr, *recvbuf = nullptr;
  // owned elements touching an exchanged node (interface, applied first) and the rest (interior,
  // applied while the exchange of the interface sums is in flight; dist.cu)
  int32_t *e_if = nullptr, *e_in = nullptr;
  int n_if = 0, n_in = 0;
  int32_t *s_if = nullptr, *s_in = nullptr;   // the same split of the owned (dense) Schwarz subdomains
  int ns_if = 0, ns_in = 0;
  int32_t *fu_if = nullptr, *fu_in = nullptr;  // the same split of the FDM column units (column-unit kernels)
  int nfu_if = 0, nfu_in = 0;
};

// deterministic mode (opts.deterministic): colour-ordered gather-scatter and
// fixed-order reductions make repeated solves bit-identical
struct Det {
  int on = 0;
  std::vector<int64_t> ecol_off;  // [colours+1] element colours (no two elements of a colour share a node)
  int32_t* ecol = nullptr;        // element ids grouped by colour
  double* part = nullptr;         // per-block partial sums [2][blocks] of the reductions
};
// greedy colouring of node sets (set k = idx[off[k] .. off[k+1]), entries < 0 ignored, sets with
// skip[k] != 0 left out): returns colour offsets and the set ids grouped by colour
void colour_sets(int64_t nsets, const std::vector<int64_t>& off, const std::vector<int32_t>& idx, int64_t nnodes,
                 const std::vector<uint8_t>* skip, std::vector<int64_t>& coff, std::vector<int32_t>& clist);
void det_finalize(sem_ctx* c, int nb, double* out0, double* out1);

struct Dist;  // dist.cu
struct Fnpf;  // fnpf.cu
struct Condense;  // condense.cu

struct Coarse {
  int64_t nc = 0;               // free coarse nodes
  int32_t* fidx = nullptr;      // [nc] compact -> level gid
  double* Ainv = nullptr;       // [nc][nc] row-major, symmetric (dense path)
  double* Apack = nullptr;      // lower-triangular 64x64 tiles of Ainv (Ainv freed), k_coarse_symv
  double* Afull = nullptr;      // deterministic mode: the full symmetric inverse [nc][nc]
  float* Apack32 = nullptr;     // the same in FP32 storage (opts.mixed_precision, reading O36)
  double* x = nullptr;          // [nc] work
  // iterative path (reading O9): vertical-line block-Jacobi PCG on the P=1 operator (coarse.cu)
  int iterative = 0;
  double* dinv = nullptr;       // [n] diagonal during setup
  double *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr;
  int nlines = 0;               // vertical lines of free P=1 nodes (bottom to top)
  int64_t line_max = 0;
  int64_t* loff = nullptr;      // [nlines+1]
  int32_t* lnode = nullptr;     // [nfree] node of every line position
  double *ta = nullptr, *tinv = nullptr, *tc = nullptr;   // Thomas factors per line position
  double* cs = nullptr;         // device scalars of the solve (coarse.cu CS_*)
  unsigned int* done = nullptr; // block-completion counter of k_coarse_update
  // two-level correction of the line preconditioner (coarse.cu): z = T^-1 r + P_a A_a^-1 P_a^T r with
  // P_a piecewise constant on nagg aggregates of whole lines (RCB of the lines' (x, y)), A_a = P_a^T A P_a
  int nagg = 0;
  int32_t* aggn = nullptr;      // [n] aggregate of every free node (-1: Dirichlet)
  int32_t* aggl = nullptr;      // [nlines] aggregate of every line
  double* Aagg_inv = nullptr;   // [nagg][nagg] symmetric inverse of A_a
  double *rc = nullptr, *zc = nullptr;   // [nagg] restricted residual / aggregate correction
  cudaGraphExec_t exec = nullptr;                 // standalone graph of the solve (coarsest L.f -> L.u)
  cudaStream_t cap_stream = nullptr, body_stream = nullptr;
  int64_t exec_launches = 0, body_launches = 0;
};

// dist.cu (partitioned solve; c->dist != nullptr)
int dist_solve(sem_ctx* c, const double* rhs, const double* phiD, double tol, double* phi, sem_report* rep);
int dist_vcycle(sem_ctx* c, const double* r, double* z);
int dist_apply(sem_ctx* c, const double* u, double* y, int level, int masked);
void dist_info(const sem_ctx* c, sem_info* info);
const std::vector<double>& dist_xyz(const sem_ctx* c, int level);
const std::vector<uint8_t>& dist_dir(const sem_ctx* c, int level);
int dist_levels(const sem_ctx* c);
sem_ctx* dist_part0(const sem_ctx* c);
int64_t dist_launches(const sem_ctx* c, int reset);
void dist_destroy(sem_ctx* c);
void nccl_unique_id(void* out);
}  // namespace sem

struct sem_ctx {
  sem_opts opts;
  int device = 0;
  cudaStream_t stream = nullptr;
  int E_global = 0;             // elements of the whole mesh
  int E = 0;                    // elements held (owned + halo in a partition)
  int E_own = 0;                // elements owned (applied); the first E_own of the E
  int P = 0, PZ = 0;            // finest horizontal / vertical order
  std::vector<sem::DeviceLevel> L;
  sem::Coarse C;
  double* scal = nullptr;       // device scalars [32]
  double* hscal = nullptr;      // pinned host scalars [16]
  double *pw = nullptr, *qw = nullptr, *zw = nullptr, *bw = nullptr, *xw = nullptr, *rw_old = nullptr;  // solver work
  double *host_in = nullptr, *host_in2 = nullptr, *host_out = nullptr;               // device staging for *_host
  // ---- partitioned solve (dist.cu): nranks > 1
  sem::Dist* dist = nullptr;
  sem::Det det;                 // deterministic mode (opts.deterministic)
  // ---- FNPF time stages (fnpf.cu)
  sem::Fnpf* fnpf = nullptr;
  // ---- static condensation of element-interior nodes (condense.cu)
  sem::Condense* cond = nullptr;
  int64_t launches = 0;
  int64_t device_bytes = 0;
  double setup_ms = 0.0;
  double t_apply_ms = 0.0;      // one finest-level operator apply (timed at setup; work units)
  std::vector<void*> allocs;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // CUDA graphs of the V-cycle (PCG's z = V(r) with the ctx's own buffers; single domain, dense coarse)
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t vc_graph[2] = {nullptr, nullptr};   // output pw / zw, input bw
  int64_t vc_graph_launches[2] = {0, 0};
  int vc_eager = 0;                                    // eager V-cycles run before capturing
};

namespace sem {
// kernels.cu launchers (all enqueue on ctx->stream and count launches)
void launch_apply(sem_ctx* c, int level, const double* u, double* y, int flags);
void launch_apply_dmma(sem_ctx* c, int level, const double* u, double* y, int flags);
std::vector<double> dmma_fragments(const LevelRef& R);
std::vector<double> warp_apply_mats(const LevelRef& R);
bool launch_apply_warp(sem_ctx* c, int level, const double* u, double* y, int flags,
                       const int32_t* elist = nullptr, int ne = 0);   // elist: apply only these elements
std::vector<double> quad_apply_mats(const LevelRef& R);
bool launch_apply_quad(sem_ctx* c, int level, const double* u, double* y, int flags);
void build_g_tiles(sem_ctx* c, int level);
void launch_schwarz_dense(sem_ctx* c, int level, const double* r, double* u, int transpose);
bool launch_fdm_list(sem_ctx* c, int level, const double* r, double* u, int transpose, const int* ulist, int nu);
bool launch_apply_subset(sem_ctx* c, int level, const double* u, double* y, int flags, const int32_t* elist, int ne);
bool launch_apply_qs(sem_ctx* c, int level, const double* u, double* y, int flags, const int32_t* elist, int ne);
void build_p1_matrices(sem_ctx* c, int level, const double* d_D);
void launch_init_masked(sem_ctx* c, int level, const double* src, double* dst, int mode);
void launch_schwarz(sem_ctx* c, int level, const double* r, double* u, int transpose);
bool launch_schwarz_list(sem_ctx* c, int level, const double* r, double* u, int transpose, const int32_t* slist,
                         int nb);   // dense levels: sweep only subdomains slist[0..nb)
void launch_fdm(sem_ctx* c, int level, const double* r, double* u, int transpose);
int fdm_kernel_choice(const DeviceLevel& L);
void launch_restrict(sem_ctx* c, int level, const double* rf, double* rc);
void launch_prolong(sem_ctx* c, int level, const double* uc, double* uf);
void launch_coarse(sem_ctx* c, const double* r, double* z);
void launch_dot2(sem_ctx* c, int64_t n, const double* a, const double* b, const double* d, const double* e,
                 const uint8_t* mask, double* out2, bool clear = true);
void launch_axpy_pcg(sem_ctx* c, int64_t n, double* u, double* r, const double* p, const double* q,
                     const double* num, const double* den, double* rr, const uint8_t* mask = nullptr,
                     bool clear = true);
// coarse.cu: iterative P=1 solve (line-Jacobi PCG, device-side stop test in a CUDA-graph WHILE node)
void coarse_pcg(sem_ctx* c, const double* b, double* x);
void setup_coarse_lines(sem_ctx* c, const std::vector<int32_t>& conn, const std::vector<uint8_t>& dir,
                        const double* d_diag, const double* d_off);
int coarse_agg_count(const sem_ctx* c);   // aggregates the line preconditioner's correction will use
void setup_coarse_agg(sem_ctx* c, const double* d_D, void* cusolver_handle);
void launch_offdiag_accum(sem_ctx* c, const int32_t* conn, int ne, const double* Ae, double* off);
int64_t coarse_iters(sem_ctx* c, bool reset);
void coarse_reset_iters(sem_ctx* c);
void coarse_count_launches(sem_ctx* c, int64_t iters);
void coarse_destroy(sem_ctx* c);
// stage.cu: per-stage re-formation (strategies of P:350-356)
void fdm_refresh_vertical(sem_ctx* c, int li, const double* X);
void coarse_refresh_lines(sem_ctx* c);
void coarse_rebuild_dense(sem_ctx* c);   // capi.cu: the dense coarse inverse from the current G (setup-time)
void refresh_level_operator(sem_ctx* c, int li, const double* X, const double* d_gm, const double* d_w);
// fnpf.cu: FNPF time stage (eq 2.1)
void fnpf_init(sem_ctx* c, const double* node_xyz, int strategy);
void fnpf_stage(sem_ctx* c, const double* eta, const double* phis, double* deta, double* dphis, double* w,
                double tol, int linear, sem_report* rep);
void fnpf_erk4(sem_ctx* c, double* eta, double* phis, double dt, double tol, int linear, int* iters);
int64_t fnpf_surface(const sem_ctx* c, int32_t* ids);
void fnpf_destroy(sem_ctx* c);
// condense.cu: static condensation
void condense_setup(sem_ctx* c);
void condense_destroy(sem_ctx* c);
void cond_extend(sem_ctx* c, double* v);
void cond_interior(sem_ctx* c, const double* src, double* dst);
void cond_zero(sem_ctx* c, double* v);
void cond_sizes(const sem_ctx* c, int* ni, int* nb, int64_t* bytes);
void launch_xpby(sem_ctx* c, int64_t n, double* p, const double* z, const double* num, const double* den, int mode);
void launch_combine_phi(sem_ctx* c, int level, const double* uF, const double* phiD, double* phi);
void launch_axpy(sem_ctx* c, int64_t n, double a, const double* x, double* y);
void launch_to_float(sem_ctx* c, int64_t n, const double* a, float* b);
void launch_coarse_pack(sem_ctx* c, int64_t n, const double* A, double* P, float* P32);
// setup kernels
int launch_geometry(sem_ctx* c, int level, const double* d_xfine, const double* d_gmat, int Nf, const double* d_w);
void launch_elem_matrices(sem_ctx* c, int level, const double* d_D, double* Ae, int e0, int ne);
void launch_assemble_blocks(sem_ctx* c, int level, const int32_t* d_idx, const int64_t* d_off, const int32_t* d_elist,
                            const int64_t* d_eoff, const double* Ae, int ebase, int k0, int nb, int npad, double* B,
                            const int32_t* eslot = nullptr);
void launch_elem_matrices_list(sem_ctx* c, int level, const double* d_D, double* Ae, const int32_t* elist, int ne);
void launch_pack_tiles(sem_ctx* c, int level, const double* Binv, int k0, int nb, int npad, const int64_t* d_off);
void launch_assemble_coarse(sem_ctx* c, const double* Ae, const int32_t* d_cmap, double* A, int64_t nc);
void launch_symmetrize(sem_ctx* c, double* A, int64_t n);
void launch_set_identity(sem_ctx* c, double* X, int nb, int npad);
void launch_diag_accum_range(sem_ctx* c, const int32_t* conn, int N, int ne, const double* Ae, double* diag);
void launch_invert_masked(sem_ctx* c, int level, double* d);
void launch_jacobi_dot(sem_ctx* c, int64_t n, const double* dinv, const double* r, double* z, double* out2);
// dist.cu (partitioned solve; c->dist != nullptr)
int dist_solve(sem_ctx* c, const double* rhs, const double* phiD, double tol, double* phi, sem_report* rep);
int dist_vcycle(sem_ctx* c, const double* r, double* z);
int dist_apply(sem_ctx* c, const double* u, double* y, int level, int masked);
void dist_info(const sem_ctx* c, sem_info* info);
const std::vector<double>& dist_xyz(const sem_ctx* c, int level);
const std::vector<uint8_t>& dist_dir(const sem_ctx* c, int level);
int dist_levels(const sem_ctx* c);
sem_ctx* dist_part0(const sem_ctx* c);
int64_t dist_launches(const sem_ctx* c, int reset);
void dist_destroy(sem_ctx* c);
void nccl_unique_id(void* out);
}  // namespace sem
