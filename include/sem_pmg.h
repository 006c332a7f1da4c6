/*
 * sem_pmg.h — C ABI of the B200-native geometric p-multigrid Laplace solver
 * (arXiv 2009.00705, Engsig-Karup et al.).
 *
 * Citation keys: P:n = PAPER.md line n (the paper); S:n = SPEC.md line n;
 * On = reading n of DESIGN.md §"Readings" (= SURVEY.md §8(c) register).
 *
 * The problem (eq 2.2):   phi = phi~ on the free surface (Dirichlet),
 *   laplace(phi) = 0 in the fluid, n.grad(phi) = 0 on bottom / walls / hull,
 * discretised by continuous-Galerkin spectral elements on curvilinear prisms
 * (eq 3.8) and solved by PCG (Alg 4.3) preconditioned
 * with one geometric p-multigrid V-cycle (Alg 4.1): additive
 * Schwarz smoother (eq 4.4-4.6), R = P^T (eq 4.3),
 * exact P=1 coarse solve.
 *
 * General conventions
 *  - All floating point is IEEE FP64.  Indices are int32.
 *  - Vector arguments of the compute calls are DEVICE pointers (cudaMalloc or
 *    torch CUDA tensors) of length n_dof(level) in the library's node
 *    numbering, unless a name ends in _host.  They are caller-owned; the
 *    library never frees or retains them beyond the call.
 *  - Calls are asynchronous with respect to the host only where stated;
 *    every compute call is enqueued on opts.stream (NULL = legacy default
 *    stream) and the functions that return scalars synchronise that stream.
 *  - Return value: 0 on success, a negative SEM_E* code otherwise;
 *    sem_strerror() gives a message.  A failed call leaves the ctx usable
 *    unless the code is SEM_ECUDA (sticky device error).
 *  - A sem_ctx is not thread-safe: one ctx per device per thread.
 *  - Reference prism: {r,s >= -1, r+s <= 0} x [-1,1]; bottom vertices v0,v1,v2
 *    at (r,s) = (-1,-1),(1,-1),(-1,1), t = -1; top v3,v4,v5 above, t = +1.
 *    Local node n = m + Nt*l: m indexes the triangle nodes (for j in 0..p, for
 *    i in 0..p-j: barycentric (k=p-i-j, i, j) toward (v0, v1, v2)), l the
 *    vertical LGL level.  Triangle nodes: Blyth-Pozrikidis (reading O1).
 */
#ifndef SEM_PMG_H
#define SEM_PMG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes ---------------------- */
#define SEM_OK            0
#define SEM_EINVAL       -1   /* bad argument: p < 1 or > 8, bad tags, NULL    */
#define SEM_EBADELEM     -2   /* detJ <= 0 at a cubature point         */
#define SEM_ENOMEM       -3   /* device allocation failed (e.g. dense Schwarz) */
#define SEM_ESINGULAR    -4   /* Schwarz block / coarse Cholesky failed*/
#define SEM_ENOTCONV     -5   /* imax reached; phi holds the last iterate */
#define SEM_EBREAKDOWN   -6   /* PCG p^T q <= 0                        */
#define SEM_ECUDA        -7   /* CUDA runtime / cuSOLVER / cuBLAS error        */
#define SEM_ENCCL        -8   /* reserved: multi-GPU communication error       */
#define SEM_EUNSUPPORTED -9   /* option combination not built (see message)    */

/* ---- face tags ----------------------------------------------- */
#define SEM_FACE_INTERIOR  0
#define SEM_FACE_DIRICHLET 1  /* free surface Gamma^FS: phi = phi~            */
#define SEM_FACE_NEUMANN   2  /* bottom, walls, hull: n.grad phi = 0          */

typedef struct sem_ctx sem_ctx;   /* opaque; owns all of its device memory */

/* Prism mesh (host memory, caller-owned, copied during sem_setup). */
typedef struct {
  int32_t n_vert;
  const double *xyz;          /* [n_vert][3] vertex coordinates                      */
  int32_t n_prism;
  const int32_t *prism;       /* [n_prism][6] v0 v1 v2 bottom (CCW seen from +z), v3 v4 v5 above them */
  const uint8_t *face_tag;    /* [n_prism][5] faces (bot, top, q01, q12, q20), SEM_FACE_*            */
  const double *node_xyz;     /* [n_prism][N(p)][3] curvilinear nodes of the finest order in the local
                                 order above (the nodal element map), or NULL = straight-sided */
  const int32_t *part;        /* optional [n_prism] owning rank of every prism for partitioned solves
                                 (opts.nranks > 1), or NULL = the library's column partition (RCB of the
                                 column centroids).  FDM local solves need whole columns per rank
                                 (SEM_EUNSUPPORTED otherwise); ignored when nranks == 1. */
} sem_mesh;

typedef struct {
  int nu1, nu2;               /* pre/post smoothing steps; default 3,3 (O20)          */
  int overlap;                /* Schwarz overlap in nodes: 0 = block Jacobi, 1 (default),
                                 -1 = refined ceil((P+1)/2) per level                        */
  int literal_smoother;       /* 0 (default): post-smoothing with S^-T (reading O14, symmetric V-cycle);
                                 1: W left-applied pre and post exactly as eq 4.4 prints it         */
  int outer;                  /* 0 PCG (Alg 4.3, default), 1 PDC (Alg 4.2), 2 stand-alone MG        */
  const int *levels;          /* explicit level orders, finest first, last = 1, or NULL
                                 = P -> ceil((P+1)/2) with strict-decrease guard (O18)       */
  int n_levels;
  double atol;                /* absolute tolerance of the stop test, default 0              */
  int imax;                   /* max outer iterations, default 200                                  */
  void *stream;               /* cudaStream_t for every kernel; NULL = default stream               */
  int device;                 /* CUDA device ordinal used by sem_setup (default: current device)    */
  int verbose;                /* 1: setup timings to stderr                                         */
  int apply_kernel;           /* operator kernel (all the same arithmetic, eq 3.8): 0 (default) FP64
                                 tensor-core (DMMA) sum factorisation, one warp per element with
                                 TMA-staged geometric factors (p <= 6; p = 7, 8 use variant 2);
                                 1 CUDA-core FMA sum factorisation (reference variant);
                                 2 DMMA with CTA-wide element batches; 3 DMMA with four elements per
                                 warp (k_apply_quad, 3 <= p <= 5); 4 DMMA with four elements per
                                 group of warps, one warp per vertical row tile (k_apply_qs,
                                 3 <= p <= 6; the default (0) uses it at 3 <= p <= 5)              */
  int coarse_solver;          /* P=1 solve (reading O9): 0 auto (dense inverse if <= 46,000 free
                                 nodes, else iterative), 1 iterative (Jacobi-PCG, the outer PCG becomes
                                 flexible), 2 dense                                                  */
  double coarse_rtol;         /* relative tolerance of the iterative coarse solve, default 1e-10      */
  int coarse_maxit;           /* iteration cap of the iterative coarse solve, default 20000           */
  int nranks;                 /* partitioned solve over nranks column partitions (default 1)         */
  int rank;                   /* this process's rank when nccl_id != NULL                            */
  const void *nccl_id;        /* ncclUniqueId (128 bytes) shared by all ranks (sem_nccl_unique_id on
                                 rank 0, broadcast by the caller): one rank per process and GPU, NCCL
                                 exchanges.  NULL with nranks > 1: all nranks partitions emulated in
                                 this process on one device (validation of the partitioned path).
                                 In both modes every vector argument of the compute calls stays a
                                 GLOBAL vector (library numbering of the whole mesh), replicated on
                                 every rank; outputs are complete on every rank.                    */
  int local_solve;            /* Schwarz local solves: 0 (default) exact dense inverses of R_k A R_k^T
                                 (eq 4.4); 1 fast diagonalisation of the separable operator
                                 K_h (x) M_v + M_h (x) K_v on the product subdomain (reading O33,
                                 Lottes & Fischer [FL05]): exact on straight prisms with flat
                                 layers, needs a layered mesh (SEM_EUNSUPPORTED otherwise).
                                 Subdomains next to columns of a different height keep the exact
                                 inverse (reading O35).  Same subdomains (O15) and weights (eq 4.6);
                                 partitioned solves (nranks > 1) supported.                          */
  int mixed_precision;        /* 0 (default): everything stored and computed in FP64.  1: the exact
                                 dense Schwarz inverses and the dense coarse inverse are STORED in FP32
                                 (rounded once at setup) and applied with FP64 arithmetic -- the
                                 mixed-precision multigrid of P:35; the preconditioner stays a fixed
                                 symmetric linear operator, the outer PCG and the operator stay FP64. */
  int deterministic;          /* 0 (default): FP64 atomics in the gather-scatter and the reductions (results
                                 agree run to run to rounding).  1: bit-reproducible solves:
                                 every scatter is launched per colour of node-disjoint elements /
                                 subdomains, reductions sum per-block partials in a fixed order, the dense
                                 coarse solve is a row-wise GEMV of the full inverse, FDM levels use the
                                 generic k_fdm.  Slower; single-domain ctx only (SEM_EUNSUPPORTED otherwise). */
  int pz;                     /* vertical polynomial order of the finest level, 0 (default) = p: the element
                                 space P_p(triangle) x P_pz(t) -- the paper's (P_xy, P_z) pairs (
                                 SURVEY NEXT-2).  Anisotropic levels run the generic operator kernel
                                 (k_apply_pq) with dense local solves on a single domain
                                 (SEM_EUNSUPPORTED otherwise).  node_xyz then has N = (p+1)(p+2)/2 (pz+1)
                                 nodes per prism, local node m + Nt l with l = 0..pz (LGL of order pz). */
  const int *levels_z;        /* with levels: the vertical order of every level (Table 5.4:
                                 levels = {5, 3, 1}, levels_z = {3, 3, 1}); NULL = levels (isotropic), or,
                                 without levels, semi-coarsening of the larger order first until the
                                 orders agree, then P -> ceil((P+1)/2) (reading O19)                   */
  int coarse_agg;             /* iterative coarse solve (reading O9): aggregates of the two-level
                                 correction added to its vertical-line preconditioner,
                                 z = T^-1 r + P_a A_a^-1 P_a^T r (P_a piecewise constant on groups of
                                 whole lines, A_a = P_a^T A P_a, dense inverse formed at setup;
                                 reading O44).  -1 (default) auto: min(1024, lines / 32) when there are
                                 >= 4096 lines, else off; 0 off; > 0 that many (at most the line
                                 count).  Off in deterministic mode.  Under strategy III the lines are
                                 re-formed every stage and A_a^-1 stays that of setup.              */
} sem_opts;

typedef struct {
  int iters;                  /* outer iterations                                                   */
  int vcycles;                /* V-cycles applied: = iters for PCG (the V-cycle after the converged
                                 iteration is skipped) and for PDC / MG                 */
  int converged;              /* 1 if ||r|| <= rtol ||f|| + atol (O21)                        */
  double rel_res;             /* final ||r||_2 / ||f||_2 over free nodes                            */
  double q_mean;              /* geometric mean of q = ||r^m||/||r^m-1|| (eq 4.7; O22)        */
  double t_ms;                /* device time of the solve (CUDA events)                             */
  double norm_f;              /* ||b_F||_2                                                           */
  double wu;                  /* work units of this solve: t_ms / (device time of one finest-level
                                 operator apply, timed at setup) (reading O25)                 */
  int coarse_iters;           /* inner coarse-solve iterations in this solve (iterative coarse path)  */
  int n_hist;                 /* entries of res_hist used                                            */
  double res_hist[256];       /* ||r^m||_2, m = 0..iters                                            */
} sem_report;

typedef struct {
  int64_t n_dof;              /* nodes of the finest level (incl. Dirichlet)                        */
  int64_t n_free;             /* free (non-Dirichlet) nodes of the finest level                     */
  int64_t n_elem;             /* prisms                                                             */
  int n_levels;               /* multigrid levels, finest first                                     */
  int level_p[16];            /* polynomial order of each level                                     */
  int64_t level_n_dof[16];    /* nodes per level                                                    */
  int64_t level_n_free[16];
  int64_t schwarz_bytes[16];  /* bytes of stored Schwarz inverses per level (0 on the coarsest)     */
  int64_t schwarz_nk_sum[16]; /* sum over subdomains of n_k (free nodes per subdomain)              */
  int64_t schwarz_packed[16]; /* sum over subdomains of n_k (n_k+1)/2 (packed symmetric entries)    */
  int64_t coarse_n;           /* free nodes of the P=1 level (size of the dense coarse inverse)     */
  int64_t device_bytes;       /* total device memory held by the ctx                                */
  double setup_ms;            /* wall time of sem_setup                                             */
  int smoother_kernel[16];    /* sweep kernel of each level's smoother (SEM_SMOOTHER_*; 0 on the
                                 coarsest level)                                                     */
  int smoother_mt[16];        /* FDM levels: 8-row tiles of the largest horizontal patch, ceil(n_h/8) */
  int level_pz[16];           /* vertical polynomial order of each level (= level_p when isotropic)   */
  int coarse_agg;             /* aggregates of the iterative coarse solve's two-level correction (0: none) */
} sem_info;

/* sem_info.smoother_kernel */
#define SEM_SMOOTHER_NONE        0   /* coarsest level: exact coarse solve                             */
#define SEM_SMOOTHER_DENSE       1   /* k_schwarz: packed exact inverses (eq 4.4)                      */
#define SEM_SMOOTHER_FDM_WARP1   2   /* k_fdm_warp<MT,1>: FDM, one warp per element, n_v <= 8          */
#define SEM_SMOOTHER_FDM_WARP2   3   /* k_fdm_warp<MT,2>: FDM, one warp per element, n_v <= 16         */
#define SEM_SMOOTHER_FDM_CTA     4   /* k_fdm_cta<MT>: FDM, CTA-shared horizontal transforms (p >= 6)   */
#define SEM_SMOOTHER_FDM_COL     5   /* k_fdm_col<MT,NVT>: FDM, large patches (refined overlap)         */
#define SEM_SMOOTHER_FDM_GENERIC 6   /* k_fdm: FDM, any size (fallback)                                 */

/* Default options (values above). */
void sem_default_opts(sem_opts *opts);

/* Reference coordinates [N(p)][3] of the local prism nodes of order p in the
 * library's local order (see the conventions above).  rst: host, caller-owned,
 * 3*N(p) doubles, N(p) = (p+1)^2 (p+2)/2.  Returns SEM_EINVAL for p<1 or p>8. */
int sem_reference_nodes(int p, double *rst);
/* The same for P_p(triangle) x P_pz(t): [Nt(p) (pz+1)][3], local node m + Nt l,
 * l = 0..pz on the LGL points of order pz.  SEM_EINVAL outside 1..8. */
int sem_reference_nodes_pq(int p, int pz, double *rst);

/* Build the solver for order p (1..8) on `mesh` (all level
 * operators, smoothers and the coarse factor are formed once here and reused).
 * Allocates device memory on the current device; *out receives the ctx.
 * Errors: SEM_EINVAL, SEM_EBADELEM, SEM_ENOMEM, SEM_ESINGULAR, SEM_ECUDA. */
int sem_setup(const sem_mesh *mesh, int p, const sem_opts *opts, sem_ctx **out);

int sem_get_info(const sem_ctx *ctx, sem_info *info);

/* Copy the coordinates of the level's global nodes, [n_dof(level)][3], into
 * `xyz` (device pointer if on_device, else host).  Lets callers map the
 * library numbering to theirs (parity tests map by coordinates). */
int sem_node_xyz(const sem_ctx *ctx, int level, double *xyz, int on_device);

/* Dirichlet mask of a level, [n_dof(level)] uint8 (1 = Dirichlet), device or host. */
int sem_dirichlet_mask(const sem_ctx *ctx, int level, uint8_t *mask, int on_device);

/* y = A u on `level` (0 = finest), A = -L of eq 3.8 (reading O3),
 * matrix-free with gather-scatter of shared nodes.
 * masked = 0: the raw Neumann stiffness (every row and column).
 * masked = 1: the Dirichlet-eliminated operator: u is read on free nodes only
 *             (Dirichlet entries treated as 0), y_free = (A_FF u_F),
 *             y_Dirichlet = u_Dirichlet (identity rows).
 * u, y: device, distinct. */
int sem_apply_laplace(sem_ctx *ctx, const double *u, double *y, int level, int masked);

/* z = V(r): one V-cycle of Alg 4.1 from a zero initial guess on the finest
 * level (the preconditioner M^-1 of eq 4.1).  r is read on free nodes only;
 * z has zeros on Dirichlet nodes.  r, z: device, distinct. */
int pmg_vcycle(sem_ctx *ctx, const double *r, double *z);

/* Solve the discrete Laplace problem (eq 2.2 / 3.8):
 *   phi = dirichlet_phi on Dirichlet nodes; A_FF phi_F = b_F - A_FD phi_D,
 * b = rhs (Neumann load vector, NULL = 0), by the outer iteration opts.outer
 * until ||r||_2 <= tol*||b_F - A_FD phi_D||_2 + atol from phi_F = 0.
 * dirichlet_phi is read on Dirichlet nodes only; phi (output) holds the
 * solution including the Dirichlet values.  rep may be NULL.
 * Returns SEM_ENOTCONV (phi = last iterate, rep->converged = 0) if imax is
 * reached, SEM_EBREAKDOWN if p^T A p <= 0. */
int laplace_solve(sem_ctx *ctx, const double *rhs, const double *dirichlet_phi,
                  double tol, double *phi, sem_report *rep);

/* laplace_solve warm-started (the paper's per-stage solves,
 * P:350-356): phi is read on free nodes as the initial guess u_F and overwritten
 * with the solution; the stop test stays relative to ||b_F - A_FD phi_D||.
 * Single-domain ctx only (SEM_EUNSUPPORTED otherwise). */
int laplace_solve_guess(sem_ctx *ctx, const double *rhs, const double *dirichlet_phi,
                        double tol, double *phi, sem_report *rep);

/* laplace_solve on the statically condensed system (the
 * supplement's "Static Condensation", eq (laplacecondensed)
 * P:655-657; reading O43):
 *   S phi_b = b_b - A_bi A_ii^-1 b_i,  S = A_bb - A_bi A_ii^-1 A_ib,
 *   A_ii phi_i = b_i - A_ib phi_b,
 * with i = the element-interior nodes of the finest level (triangle lattice
 * i, j, k >= 1 and 0 < l < q: one element each, so A_ii is block diagonal) and
 * b = every other free node.  The outer iteration opts.outer runs on S with the
 * preconditioner phi_b <- (V(r))_b (the skeleton block of the full-system
 * V-cycle, which approximates (A^-1)_bb = S^-1); iterates keep their interior
 * values as the exact interior solve of their skeleton values, so phi (output,
 * including Dirichlet values) is the full solution and the residual tested
 * against tol*||b_F - A_FD phi_D|| + atol is the full system's.
 * guess != 0: phi is read on free skeleton nodes as the initial phi_b.
 * The per-element factors (A_ii^-1 A_ib and A_ii^-1, FP64, E*ni*(nb+ni)*8
 * bytes) are formed on the device on the first call and after every
 * sem_update_geometry (SEM_ENOMEM if they do not fit).  Element orders with
 * no interior nodes (p < 3 or q < 2) reduce to laplace_solve.  Single-domain
 * ctx only (SEM_EUNSUPPORTED otherwise).  rhs, dirichlet_phi, phi: device. */
int laplace_solve_condensed(sem_ctx *ctx, const double *rhs, const double *dirichlet_phi,
                            double tol, double *phi, int guess, sem_report *rep);

/* Sizes of the condensation (forms the factors if not yet formed): interior
 * and skeleton nodes per element and the device bytes of the factors. */
int sem_condensed_info(sem_ctx *ctx, int *n_interior, int *n_skeleton, int64_t *bytes);

/* New element geometry for the next time stage (Fig 5.1;
 * readings O41, O42): node_xyz is the nodal map in sem_mesh.node_xyz's layout (host,
 * copied), with the same mesh topology.
 *   strategy 1 (the paper's strategy I): only the finest operator follows the new
 *     geometry; the Schwarz inverses / FDM factors, the coarse-level operators and the
 *     coarse inverse stay those of sem_setup (t = 0);
 *   strategy 2 ("operators only", not one of the paper's strategies): the operators
 *     of every level follow it (G, the P <= 2 element matrices), the smoothers and the
 *     coarse inverse stay;
 *   strategy 4 (the paper's strategy III): every level's operator AND smoother (FDM
 *     vertical factors, re-formed on the device) and the iterative coarse solve's
 *     line-Jacobi preconditioner follow it; needs local_solve = 1 and coarse_solver
 *     = 1 (SEM_EUNSUPPORTED otherwise).  Strategy II (3) needs the still-water
 *     geometry: FNPF stages only (sem_fnpf_init).
 * Node coordinates (sem_node_xyz) are updated on the refreshed levels.  Single-domain
 * ctx only.  Errors: SEM_EINVAL, SEM_EBADELEM (detJ <= 0), SEM_EUNSUPPORTED. */
int sem_update_geometry(sem_ctx *ctx, const double *node_xyz, int strategy);

/* laplace_solve with HOST buffers (pinned recommended): copies rhs (if not
 * NULL) and dirichlet_phi host->device, solves, copies phi device->host, all
 * on opts.stream, and synchronises.  The end-to-end entry point. */
int laplace_solve_host(sem_ctx *ctx, const double *rhs_host, const double *dirichlet_phi_host,
                       double tol, double *phi_host, sem_report *rep);

/* ---- diagnostic entry points: each one step of the V-cycle, for parity ---- */
/* uf += P uc: prolongation from level+1 to level, uc read on free
 * nodes of level+1; only free fine nodes are updated. */
int sem_prolong(sem_ctx *ctx, int level, const double *uc, double *uf);
/* rc = P^T rf (eq 4.3): restriction from level to level+1; rf read on free
 * nodes; rc written on all nodes (0 on Dirichlet nodes). */
int sem_restrict(sem_ctx *ctx, int level, const double *rf, double *rc);
/* u += S^-1 r (transpose=0) or u += S^-T r (transpose=1): one additive Schwarz
 * correction of eq 4.2/4.4 on `level` (not the coarsest); r read on free nodes. */
int sem_schwarz(sem_ctx *ctx, int level, const double *r, double *u, int transpose);
/* z = A_1^-1 r on the coarsest level (exact coarse solve); z = 0 on Dirichlet. */
int sem_coarse_solve(sem_ctx *ctx, const double *r, double *z);

/* Time `reps` back-to-back launches of one hot kernel on the ctx's stream with
 * CUDA events (after 3 warm-ups), on this rank's partition in a partitioned
 * ctx: kernel 0 = one Schwarz sweep (k_schwarz) on `level` (not the coarsest),
 * 1 = one operator apply (k_apply) on `level`, 2 = one exact coarse solve
 * (k_coarse_symv or the FP32 GEMV; `level` ignored; SEM_EINVAL with the
 * iterative coarse solver).  mean_us: mean duration;
 * alg_bytes: algorithmic bytes per launch. */
int sem_bench_kernel(sem_ctx *ctx, int kernel, int level, int reps, double *mean_us, double *alg_bytes);

/* ---- FNPF time stages (eq 2.1a-b and 2.2; readings O37-O40) ----
 * The fully nonlinear potential-flow model that re-solves the Laplace problem at
 * every Runge-Kutta stage.  State: the free-surface elevation eta (z of the
 * free-surface node) and the surface potential phi~, DEVICE vectors of length
 * n_surface in the order of sem_fnpf_surface_nodes.  Needs a sigma-layered mesh
 * (every node on the vertical line of one free-surface node; SEM_EUNSUPPORTED
 * otherwise, e.g. under a body) and a single-domain ctx.
 *
 * sem_fnpf_init: node_xyz = the nodal map passed to sem_setup (host, [n_prism][N][3],
 * copied); strategy 1 = the paper's strategy I (only the finest operator follows the
 * free surface; smoothers and coarse operators from t = 0), 2 = every
 * level's operator follows it (smoothers and coarse inverse from t = 0), 3 = strategy
 * II (the finest operator and smoother follow the free surface every stage; the
 * coarse levels use the still-water (eta = 0) "LIN" operators and smoothers, formed
 * here once), 4 = strategy III (every level's operator and smoother, and the coarse
 * preconditioner, follow it every stage).  3 and 4 need local_solve = 1 (FDM smoother
 * re-formation on the device); 4 needs coarse_solver = 1. */
int sem_fnpf_init(sem_ctx *ctx, const double *node_xyz, int strategy, int64_t *n_surface);
/* library node id (finest level) of every free-surface node, host [n_surface] */
int sem_fnpf_surface_nodes(const sem_ctx *ctx, int32_t *node_ids);
/* One stage: move the fluid volume to eta (sigma map, O37), solve eq 2.2 with
 * phi = phi~ on the free surface to tol (warm-started from the previous stage),
 * recover w~ = dphi/dz (O38) and the surface gradients (O39), and return the rates
 * of eq 2.1a-b: deta = -grad eta.grad phi~ + w~ (1 + |grad eta|^2),
 * dphis = -g eta - (|grad phi~|^2 - w~^2 (1 + |grad eta|^2)) / 2, g = 9.81;
 * w (may be NULL) receives w~.  linear = 1: the small-amplitude version on the
 * t = 0 geometry (deta = w~, dphis = -g eta).  Returns SEM_ENOTCONV if the solve
 * did not converge (the rates are still written). */
int fnpf_rhs(sem_ctx *ctx, const double *eta, const double *phis, double *deta, double *dphis, double *w,
             double tol, int linear, sem_report *rep);
/* One classical RK4 step of length dt (ERK4; reading O40: four stages, one
 * Laplace solve each), eta and phis updated in place; iters (may be NULL) receives
 * the PCG iterations of the four stage solves. */
int fnpf_erk4_step(sem_ctx *ctx, double *eta, double *phis, double dt, double tol, int linear, int *iters);

/* Generate an NCCL unique id (128 bytes) for opts.nccl_id (call on rank 0). */
int sem_nccl_unique_id(void *id_out);

/* Number of kernel launches the library enqueued since the last reset. */
int64_t sem_launch_count(const sem_ctx *ctx, int reset);

void sem_destroy(sem_ctx *ctx);

/* ---- host-only diagnostics (no device needed; used by the CPU test tier) ---- */
/* Global numbering of V^p on `mesh` exactly as sem_setup builds it.  Two-call
 * pattern: pass NULL arrays to query sizes.  conn: [n_prism][N(p)] int32 node
 * ids; dirichlet: [n_dof] (1 = node on a face tagged SEM_FACE_DIRICHLET);
 * owner: [n_prism][N(p)] (1 = first element, in input order, holding the node). */
int sem_host_numbering(const sem_mesh *mesh, int p, int64_t *n_dof, int64_t *n_free,
                       int32_t *conn, uint8_t *dirichlet, uint8_t *owner);
/* Schwarz subdomains of level order p with `overlap` (reading O15): off
 * [n_prism+1], idx [total] sorted free node ids of each subdomain, W [n_dof]
 * weights of eq 4.6 (0 on Dirichlet nodes).  Two-call pattern as above. */
int sem_host_schwarz(const sem_mesh *mesh, int p, int overlap, int64_t *total, int64_t *off,
                     int32_t *idx, double *W);
/* Subdomains of the smoother with FDM local solves (opts.local_solve = 1,
 * reading O33) on level order p with `overlap`: off [n_prism+1], idx [total]
 * sorted free node ids of each subdomain -- the product box H_k x V_k where it
 * is regular, the reading-O15 set where the exact local inverse is kept
 * (reading O35) -- and W [n_dof] (eq 4.6).  Needs a layered mesh
 * (SEM_EUNSUPPORTED otherwise).  Two-call pattern as above. */
int sem_host_fdm(const sem_mesh *mesh, int p, int overlap, int64_t *total, int64_t *off, int32_t *idx,
                 double *W);
/* Column partition used by the partitioned solve (opts.nranks > 1), level
 * `level` of the default schedule of order p (>= 2), seen from `rank`:
 * sizes[5] = {elements held, elements owned, local nodes, neighbours, exchange
 * entries}; elems [held] global element ids (owned first), gid [local nodes]
 * global node ids, owned [local nodes] (each global node owned by exactly one
 * rank), nbr [neighbours] ranks, xoff [neighbours+1], xidx [entries] local ids
 * of the nodes shared with each neighbour in ascending global id.  Two-call
 * pattern (NULL arrays first). */
int sem_host_partition(const sem_mesh *mesh, int p, int nranks, int rank, int level, int64_t *sizes,
                       int32_t *elems, int32_t *gid, uint8_t *owned, int32_t *nbr, int64_t *xoff, int32_t *xidx);
/* Reference operator matrices of order p: B0, Br, Bs [(p+1)^2][Nt] (triangle
 * basis / d/dr / d/ds at the collapsed cubature), Bt, Dt [p+1][p+1] (1D basis /
 * derivative at vertical Gauss points), w [(p+1)^3] cubature weights. */
int sem_host_reference(int p, double *B0, double *Br, double *Bs, double *Bt, double *Dt, double *w);
const char *sem_strerror(int code);
/* Message of the last error raised in this thread (more detail than sem_strerror). */
const char *sem_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SEM_PMG_H */
