// Partitioned (multi-GPU) solve: SURVEY §8(e).  The paper has no parallel
// implementation ("ongoing work"); this is the build's domain
// decomposition of the same method.
//
// Every rank holds its owned elements (whole columns, partition.cpp) and the
// halo elements its Schwarz subdomains touch.  Each scatter kernel (operator,
// Schwarz, restriction, prolongation) leaves partial sums on the rank's nodes;
// one neighbour sum-exchange of the shared nodes completes them, so every
// vector is consistent on every rank's nodes after each step.  Dot products
// run over the nodes a rank owns (each global node exactly once) followed by an
// all-reduce.  The P=1 coarse problem is all-reduced into a global vector and
// solved redundantly on every rank (north_star: "may be gathered").
//
// Two transports behind one code path:
//   NCCL      one rank per process/GPU; grouped ncclSend/ncclRecv for the
//             exchange, ncclAllReduce for dots and the coarse gather (NCCL is
//             dlopen'ed, so torch's libnccl is reused in-process);
//   emulated  all R ranks in one process on one device, exchanges as device
//             copies between the ranks' buffers -- used to test the partitioned
//             algorithm against the single-domain one on a single GPU.
//
// Operator applies overlap their exchange with compute (apply_exchange): the owned
// elements touching an exchanged node (interface) are applied first, their partial
// sums packed and sent on a communication stream, and the interior elements -- which
// touch no exchanged node -- are applied on the compute stream while the transfer is
// in flight; the received sums are added after both.  Dense Schwarz sweeps and FDM
// sweeps split the same way over subdomains / column units.  On by default for the NCCL
// transport, off for emulated ranks (SEM_DIST_OVERLAP, see dist_setup).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <omp.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "setup_util.h"

namespace sem {

// ------------------------------------------------------------------ NCCL shim
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  if (!api.h) {
    api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!api.h) throw SemError(SEM_ENCCL, std::string("dlopen libnccl.so.2 failed: ") + dlerror());
    auto sym = [&](const char* n) {
      void* f = dlsym(api.h, n);
      if (!f) throw SemError(SEM_ENCCL, std::string("NCCL symbol missing: ") + n);
      return f;
    };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
  }
  return api;
}

#define NCCL_CHECK(x)                                                                             \
  do {                                                                                            \
    ncclResult_t _r = (x);                                                                        \
    if (_r != ncclSuccess) throw SemError(SEM_ENCCL, std::string(#x) + ": " + nccl().GetErrorString(_r)); \
  } while (0)

// ------------------------------------------------------------------ kernels
__global__ void k_pack(int64_t n, const int32_t* __restrict__ idx, const double* __restrict__ v,
                       double* __restrict__ buf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = v[idx[i]];
}
__global__ void k_unpack_add(int64_t n, const int32_t* __restrict__ idx, const double* __restrict__ buf,
                             double* __restrict__ v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(v + idx[i], buf[i]);
}
// local[i] = global[gid[i]]
__global__ void k_scatter_from_global(int64_t n, const int32_t* __restrict__ gid, const double* __restrict__ g,
                                      double* __restrict__ l) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    l[i] = g[gid[i]];
}
// global[gid[i]] = local[i] where own[i]
__global__ void k_gather_owned(int64_t n, const int32_t* __restrict__ gid, const uint8_t* __restrict__ own,
                               const double* __restrict__ l, double* __restrict__ g) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (own[i]) g[gid[i]] = l[i];
}

static int gsz(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

// ------------------------------------------------------------------ state
struct Dist {
  int rank = 0, nranks = 1;
  bool emulated = true;
  std::vector<sem_ctx*> parts;   // emulated: all ranks; NCCL: this rank only
  std::vector<int> part_rank;    // rank of each part
  sem_ctx* coarse = nullptr;     // whole-mesh P=1 solver (one per process)
  ncclComm_t comm = nullptr;
  // global sizes per level, host node data for the API
  std::vector<int64_t> gn, gnfree;
  std::vector<int> gp;
  std::vector<std::vector<double>> gxyz;
  std::vector<std::vector<uint8_t>> gdir;
  double* gbuf = nullptr;        // [gn[0]] global staging
  double* gbuf2 = nullptr;       // [gn[0]]
  double* gbuf3 = nullptr;       // [gn[0]]
  double *cx = nullptr, *cz = nullptr;  // global coarse rhs / solution [gn.back()]
  double* hsum = nullptr;        // pinned host [32] (emulated all-reduce)
  // overlap of operator applies with their exchange (apply_exchange)
  bool overlap = true;
  int fdm_ov_min = 0;            // least interface FDM units per part for the split sweep
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_pack = nullptr, ev_xfer = nullptr;
  // PCG's z = V(r) on fixed buffers (r = bw, z = pw / zw of every part) replayed from a CUDA
  // graph (vcycle_pcg below): kernels, exchanges (comm-stream fork/join, NCCL send/recv or the
  // emulated copies), the coarse all-reduce and solve
  cudaGraphExec_t vc_exec[2] = {nullptr, nullptr};
  std::vector<int64_t> vc_dl[2];   // kernel launches of one replay per part, coarse ctx last
  cudaStream_t cap_stream = nullptr;
  int vc_eager = 0;
};

template <class F>
static void each(Dist& D, F f) {
  for (size_t r = 0; r < D.parts.size(); ++r) f(D.parts[r], (int)r);
}

// exchange = pack (compute stream) -> transfer (stream st) -> unpack-add (compute stream)
static void pack_all(Dist& D, int li, const std::vector<double*>& v) {
  const int R = (int)D.parts.size();
  for (int r = 0; r < R; ++r) {
    sem_ctx* c = D.parts[r];
    DeviceLevel& L = c->L[li];
    const int64_t n = L.xoff.back();
    if (n) k_pack<<<gsz(n), 256, 0, c->stream>>>(n, L.xidx, v[r], L.sendbuf), c->launches++;
  }
}

static void unpack_all(Dist& D, int li, const std::vector<double*>& v) {
  const int R = (int)D.parts.size();
  for (int r = 0; r < R; ++r) {
    sem_ctx* c = D.parts[r];
    DeviceLevel& L = c->L[li];
    const int64_t n = L.xoff.back();
    if (n) k_unpack_add<<<gsz(n), 256, 0, c->stream>>>(n, L.xidx, L.recvbuf, v[r]), c->launches++;
  }
}

static void transfer(Dist& D, int li, cudaStream_t st) {
  const int R = (int)D.parts.size();
  if (D.emulated) {
    for (int r = 0; r < R; ++r) {
      DeviceLevel& L = D.parts[r]->L[li];
      for (size_t j = 0; j < L.nbr.size(); ++j) {
        const int q = L.nbr[j];
        DeviceLevel& Q = D.parts[q]->L[li];
        size_t jq = 0;
        while (jq < Q.nbr.size() && Q.nbr[jq] != D.part_rank[r]) ++jq;
        const int64_t cnt = L.xoff[j + 1] - L.xoff[j];
        if (jq == Q.nbr.size() || Q.xoff[jq + 1] - Q.xoff[jq] != cnt)
          throw SemError(SEM_ENCCL, "inconsistent exchange lists");
        CUDA_CHECK(cudaMemcpyAsync(L.recvbuf + L.xoff[j], Q.sendbuf + Q.xoff[jq], cnt * 8, cudaMemcpyDeviceToDevice,
                                   st));
      }
    }
  } else {
    sem_ctx* c = D.parts[0];
    DeviceLevel& L = c->L[li];
    NCCL_CHECK(nccl().GroupStart());
    for (size_t j = 0; j < L.nbr.size(); ++j) {
      const size_t cnt = (size_t)(L.xoff[j + 1] - L.xoff[j]);
      NCCL_CHECK(nccl().Send(L.sendbuf + L.xoff[j], cnt, ncclFloat64, L.nbr[j], D.comm, st));
      NCCL_CHECK(nccl().Recv(L.recvbuf + L.xoff[j], cnt, ncclFloat64, L.nbr[j], D.comm, st));
    }
    NCCL_CHECK(nccl().GroupEnd());
  }
}

// one exchange: complete the partial sums of v (one pointer per part) on level li
static void exchange(Dist& D, int li, const std::vector<double*>& v) {
  pack_all(D, li, v);
  transfer(D, li, D.parts[0]->stream);
  unpack_all(D, li, v);
}

// y (+)= A u on level li (each part's owned elements), then the exchange that completes y.
// Overlapped when every part can apply element subsets (k_apply_qs / k_apply_warp, p <= 6): interface
// elements -> pack -> [transfer on the comm stream || interior elements] -> unpack-add.
// Correct because interior elements write no exchanged node, so the packed partial sums
// are final once the interface elements are done.
static void apply_exchange(Dist& D, int li, const std::vector<double*>& u, const std::vector<double*>& y, int flags) {
  bool ov = D.overlap;
  for (auto* c : D.parts) ov = ov && c->L[li].e_if && c->L[li].wmats && c->L[li].Gw && !c->det.on &&
                               (c->opts.apply_kernel == 0 || c->opts.apply_kernel >= 3);
  if (!ov) {
    each(D, [&](sem_ctx* c, int i) { launch_apply(c, li, u[i], y[i], flags); });
    exchange(D, li, y);
    return;
  }
  sem_ctx* c0 = D.parts[0];
  each(D, [&](sem_ctx* c, int i) {
    DeviceLevel& L = c->L[li];
    if (L.n_if && !launch_apply_subset(c, li, u[i], y[i], flags, L.e_if, L.n_if))
      throw SemError(SEM_ECUDA, "interface apply");
  });
  pack_all(D, li, y);
  CUDA_CHECK(cudaEventRecord(D.ev_pack, c0->stream));
  CUDA_CHECK(cudaStreamWaitEvent(D.comm_stream, D.ev_pack, 0));
  transfer(D, li, D.comm_stream);
  CUDA_CHECK(cudaEventRecord(D.ev_xfer, D.comm_stream));
  each(D, [&](sem_ctx* c, int i) {
    DeviceLevel& L = c->L[li];
    if (L.n_in && !launch_apply_subset(c, li, u[i], y[i], flags, L.e_in, L.n_in))
      throw SemError(SEM_ECUDA, "interior apply");
  });
  CUDA_CHECK(cudaStreamWaitEvent(c0->stream, D.ev_xfer, 0));
  unpack_all(D, li, y);
}

// sum slots [s, s+k) of every part's scalar array over all ranks (in place)
static void allreduce_scal(Dist& D, int s, int k) {
  if (!D.emulated) {
    sem_ctx* c = D.parts[0];
    NCCL_CHECK(nccl().AllReduce(c->scal + s, c->scal + s, k, ncclFloat64, ncclSum, D.comm, c->stream));
    return;
  }
  const int R = (int)D.parts.size();
  std::vector<double> acc(k, 0.0);
  for (int r = 0; r < R; ++r) {
    sem_ctx* c = D.parts[r];
    CUDA_CHECK(cudaMemcpyAsync(D.hsum, c->scal + s, k * 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
    for (int i = 0; i < k; ++i) acc[i] += D.hsum[i];
  }
  for (int i = 0; i < k; ++i) D.hsum[i] = acc[i];
  for (int r = 0; r < R; ++r) {
    sem_ctx* c = D.parts[r];
    CUDA_CHECK(cudaMemcpyAsync(c->scal + s, D.hsum, k * 8, cudaMemcpyHostToDevice, c->stream));
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
  }
}

// all-reduce a global vector assembled from every rank's owned entries
static void allreduce_vec(Dist& D, double* g, int64_t n) {
  if (!D.emulated && D.nranks > 1) {
    sem_ctx* c = D.parts[0];
    NCCL_CHECK(nccl().AllReduce(g, g, n, ncclFloat64, ncclSum, D.comm, c->stream));
  }
  // emulated: every part wrote its owned entries into the same buffer
}

// ------------------------------------------------------------------ steps

using Vecs = std::vector<double*>;

static Vecs lvec(Dist& D, int li, double* DeviceLevel::*m) {
  Vecs v;
  for (auto* c : D.parts) v.push_back(c->L[li].*m);
  return v;
}

// r = f - A u on level li (complete on every rank's nodes)
static void residual(Dist& D, int li, const Vecs& f, const Vecs& u, const Vecs& r) {
  each(D, [&](sem_ctx* c, int i) { launch_init_masked(c, li, f[i], r[i], 2); });
  apply_exchange(D, li, u, r, AP_NEGATE);
}

// u += S^-1 r (transpose = 0) or u += S^-T r.  Dense levels overlap the exchange like
// apply_exchange: interface subdomains, pack, [transfer || interior subdomains], unpack-add.
static void schwarz_update(Dist& D, int li, const Vecs& r, const Vecs& u, int transpose) {
  Vecs d = lvec(D, li, &DeviceLevel::d);
  bool ov = D.overlap, fov = D.overlap;
  for (auto* c : D.parts) {
    ov = ov && c->L[li].s_if && !c->L[li].fdm && !c->det.on;
    fov = fov && c->L[li].fdm && c->L[li].fu_if && !c->det.on && c->L[li].nfu_if >= D.fdm_ov_min;
  }
  each(D, [&](sem_ctx* c, int i) { CUDA_CHECK(cudaMemsetAsync(d[i], 0, sizeof(double) * c->L[li].n, c->stream)); });
  if (fov) {  // FDM level: interface column units (+ the whole O35 dense subset), then the rest
    sem_ctx* c0 = D.parts[0];
    each(D, [&](sem_ctx* c, int i) {
      const DeviceLevel& L = c->L[li];
      if (!launch_fdm_list(c, li, r[i], d[i], transpose, L.fu_if, L.nfu_if)) throw SemError(SEM_ECUDA, "fdm");
      if (L.nsub) launch_schwarz_dense(c, li, r[i], d[i], transpose);
    });
    pack_all(D, li, d);
    CUDA_CHECK(cudaEventRecord(D.ev_pack, c0->stream));
    CUDA_CHECK(cudaStreamWaitEvent(D.comm_stream, D.ev_pack, 0));
    transfer(D, li, D.comm_stream);
    CUDA_CHECK(cudaEventRecord(D.ev_xfer, D.comm_stream));
    each(D, [&](sem_ctx* c, int i) {
      const DeviceLevel& L = c->L[li];
      if (!launch_fdm_list(c, li, r[i], d[i], transpose, L.fu_in, L.nfu_in)) throw SemError(SEM_ECUDA, "fdm");
    });
    CUDA_CHECK(cudaStreamWaitEvent(c0->stream, D.ev_xfer, 0));
    unpack_all(D, li, d);
  } else if (!ov) {
    each(D, [&](sem_ctx* c, int i) { launch_schwarz(c, li, r[i], d[i], transpose); });
    exchange(D, li, d);
  } else {
    sem_ctx* c0 = D.parts[0];
    each(D, [&](sem_ctx* c, int i) {
      const DeviceLevel& L = c->L[li];
      if (!launch_schwarz_list(c, li, r[i], d[i], transpose, L.s_if, L.ns_if)) throw SemError(SEM_ECUDA, "schwarz");
    });
    pack_all(D, li, d);
    CUDA_CHECK(cudaEventRecord(D.ev_pack, c0->stream));
    CUDA_CHECK(cudaStreamWaitEvent(D.comm_stream, D.ev_pack, 0));
    transfer(D, li, D.comm_stream);
    CUDA_CHECK(cudaEventRecord(D.ev_xfer, D.comm_stream));
    each(D, [&](sem_ctx* c, int i) {
      const DeviceLevel& L = c->L[li];
      if (!launch_schwarz_list(c, li, r[i], d[i], transpose, L.s_in, L.ns_in)) throw SemError(SEM_ECUDA, "schwarz");
    });
    CUDA_CHECK(cudaStreamWaitEvent(c0->stream, D.ev_xfer, 0));
    unpack_all(D, li, d);
  }
  each(D, [&](sem_ctx* c, int i) { launch_axpy(c, c->L[li].n, 1.0, d[i], u[i]); });
}

static void coarse_step(Dist& D, int li, const Vecs& f, const Vecs& u) {
  // gather the owned coarse residual into a global vector, all-reduce, solve
  // redundantly with the whole-mesh coarse solver, scatter back
  sem_ctx* c0 = D.parts[0];
  const int64_t gnc = D.gn[li];
  CUDA_CHECK(cudaMemsetAsync(D.cx, 0, sizeof(double) * gnc, c0->stream));
  each(D, [&](sem_ctx* c, int i) {
    DeviceLevel& L = c->L[li];
    k_gather_owned<<<gsz(L.n), 256, 0, c->stream>>>(L.n, L.gid, L.ownfree, f[i], D.cx);
    c->launches++;
  });
  allreduce_vec(D, D.cx, gnc);
  coarse_solve(D.coarse, D.cx, D.cz);
  each(D, [&](sem_ctx* c, int i) {
    DeviceLevel& L = c->L[li];
    k_scatter_from_global<<<gsz(L.n), 256, 0, c->stream>>>(L.n, L.gid, D.cz, u[i]);
    c->launches++;
  });
}

static void vcycle(Dist& D, int li, const Vecs& f, const Vecs& u) {
  const int nl = (int)D.parts[0]->L.size();
  if (li == nl - 1) {
    coarse_step(D, li, f, u);
    return;
  }
  const sem_opts& o = D.parts[0]->opts;
  const int post_t = o.literal_smoother ? 0 : 1;
  Vecs r = lvec(D, li, &DeviceLevel::r);
  each(D, [&](sem_ctx* c, int i) { CUDA_CHECK(cudaMemsetAsync(u[i], 0, sizeof(double) * c->L[li].n, c->stream)); });
  for (int m = 0; m < o.nu1; ++m) {
    if (m == 0) {
      schwarz_update(D, li, f, u, 0);
    } else {
      residual(D, li, f, u, r);
      schwarz_update(D, li, r, u, 0);
    }
  }
  if (o.nu1 > 0) residual(D, li, f, u, r);
  else each(D, [&](sem_ctx* c, int i) { launch_init_masked(c, li, f[i], r[i], 1); });
  Vecs cf = lvec(D, li + 1, &DeviceLevel::f), cu = lvec(D, li + 1, &DeviceLevel::u);
  each(D, [&](sem_ctx* c, int i) { launch_restrict(c, li, r[i], cf[i]); });
  exchange(D, li + 1, cf);
  vcycle(D, li + 1, cf, cu);
  Vecs d = lvec(D, li, &DeviceLevel::d);
  each(D, [&](sem_ctx* c, int i) {
    CUDA_CHECK(cudaMemsetAsync(d[i], 0, sizeof(double) * c->L[li].n, c->stream));
    launch_prolong(c, li, cu[i], d[i]);
  });
  exchange(D, li, d);
  each(D, [&](sem_ctx* c, int i) { launch_axpy(c, c->L[li].n, 1.0, d[i], u[i]); });
  for (int m = 0; m < o.nu2; ++m) {
    residual(D, li, f, u, r);
    schwarz_update(D, li, r, u, post_t);
  }
}

// z = V(r) for the PCG / MG loops, replayed from a CUDA graph after one eager V-cycle (function
// attributes and lazily sized buffers settled).  Every part and the coarse ctx must run on one
// stream (NCCL: one part per process; emulated: the parts share the caller's stream), else
// eager.  SEM_NO_GRAPHS=1 or SEM_DIST_GRAPHS=0 turn it off.
static void vcycle_pcg(Dist& D, const Vecs& r, const Vecs& z, int slot) {
  static const int off = [] {
    const char* e = getenv("SEM_NO_GRAPHS");
    const char* f = getenv("SEM_DIST_GRAPHS");
    return ((e && atoi(e)) || (f && !atoi(f))) ? 1 : 0;
  }();
  sem_ctx* c0 = D.parts[0];
  bool same = D.coarse->stream == c0->stream;
  for (auto* c : D.parts) same = same && c->stream == c0->stream;
  if (off || !same || D.vc_eager < 1) {
    vcycle(D, 0, r, z);
    D.vc_eager++;
    return;
  }
  const int R = (int)D.parts.size();
  if (!D.vc_exec[slot]) {
    if (!D.cap_stream) CUDA_CHECK(cudaStreamCreateWithFlags(&D.cap_stream, cudaStreamNonBlocking));
    CUDA_CHECK(cudaStreamSynchronize(c0->stream));
    CUDA_CHECK(cudaStreamSynchronize(D.comm_stream));
    const cudaStream_t keep = c0->stream;
    std::vector<int64_t> l0;
    for (auto* c : D.parts) l0.push_back(c->launches), c->stream = D.cap_stream;
    l0.push_back(D.coarse->launches);
    D.coarse->stream = D.cap_stream;
    auto restore = [&] {
      for (auto* c : D.parts) c->stream = keep;
      D.coarse->stream = keep;
    };
    cudaGraph_t g = nullptr;
    CUDA_CHECK(cudaStreamBeginCapture(D.cap_stream, cudaStreamCaptureModeThreadLocal));
    try {
      vcycle(D, 0, r, z);
    } catch (...) {
      cudaStreamEndCapture(D.cap_stream, &g);
      if (g) cudaGraphDestroy(g);
      restore();
      throw;
    }
    CUDA_CHECK(cudaStreamEndCapture(D.cap_stream, &g));
    restore();
    D.vc_dl[slot].assign(R + 1, 0);
    for (int i = 0; i < R; ++i) D.vc_dl[slot][i] = D.parts[i]->launches - l0[i], D.parts[i]->launches = l0[i];
    D.vc_dl[slot][R] = D.coarse->launches - l0[R];
    D.coarse->launches = l0[R];
    CUDA_CHECK(cudaGraphInstantiate(&D.vc_exec[slot], g, 0));
    CUDA_CHECK(cudaGraphDestroy(g));
  }
  CUDA_CHECK(cudaGraphLaunch(D.vc_exec[slot], c0->stream));
  for (int i = 0; i < R; ++i) D.parts[i]->launches += D.vc_dl[slot][i];
  D.coarse->launches += D.vc_dl[slot][R];
}

static void read_scal(Dist& D, int s, int k, double* out) {
  sem_ctx* c = D.parts[0];
  CUDA_CHECK(cudaMemcpyAsync(c->hscal, c->scal + s, k * 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < k; ++i) out[i] = c->hscal[i];
}

// masked dot over owned free nodes + all-reduce: out slots [s], ([s+1] if d)
static void dot(Dist& D, const Vecs& a, const Vecs& b, const Vecs* d, const Vecs* e, int s) {
  each(D, [&](sem_ctx* c, int i) {
    launch_dot2(c, c->L[0].n, a[i], b[i], d ? (*d)[i] : nullptr, e ? (*e)[i] : nullptr, c->L[0].ownfree,
                c->scal + s);
  });
  allreduce_scal(D, s, d ? 2 : 1);
}

static int solve(Dist& D, const Vecs& rhs, const Vecs& phiD, double tol, const Vecs& phi, sem_report* rep) {
  sem_ctx* c0 = D.parts[0];
  const sem_opts& o = c0->opts;
  sem_report R;
  memset(&R, 0, sizeof(R));
  coarse_reset_iters(D.coarse);
  CUDA_CHECK(cudaEventRecord(c0->ev0, c0->stream));
  Vecs u, r, p, q, z, ro;
  for (auto* c : D.parts) {
    u.push_back(c->xw);
    r.push_back(c->bw);
    p.push_back(c->pw);
    q.push_back(c->qw);
    z.push_back(c->zw);
    ro.push_back(c->rw_old);
  }
  // lift: b_F = rhs_F - A_FD phi_D
  each(D, [&](sem_ctx* c, int i) {
    launch_init_masked(c, 0, phiD[i], q[i], 0);
    launch_init_masked(c, 0, rhs.empty() ? nullptr : rhs[i], r[i], 2);
  });
  // PDC / MG keep this rank's partial b_F (summed by every later exchange)
  if (o.outer != 0) {
    each(D, [&](sem_ctx* c, int i) { launch_apply(c, 0, q[i], r[i], AP_GATHER_ALL | AP_NEGATE); });
    each(D, [&](sem_ctx* c, int i) {
      CUDA_CHECK(cudaMemcpyAsync(ro[i], r[i], sizeof(double) * c->L[0].n, cudaMemcpyDeviceToDevice, c->stream));
    });
    exchange(D, 0, r);
  } else {
    apply_exchange(D, 0, q, r, AP_GATHER_ALL | AP_NEGATE);
  }
  each(D, [&](sem_ctx* c, int i) { CUDA_CHECK(cudaMemsetAsync(u[i], 0, sizeof(double) * c->L[0].n, c->stream)); });
  double h[4];
  dot(D, r, r, nullptr, nullptr, 4);
  read_scal(D, 4, 1, h);
  const double nf = std::sqrt(h[0]);
  R.norm_f = nf;
  const double thresh = tol * nf + o.atol;
  double rn = nf;
  R.res_hist[R.n_hist++] = rn;
  int status = SEM_OK;
  const bool flex = D.coarse->C.iterative != 0;
  if (rn <= thresh) {
    R.converged = 1;
  } else if (o.outer == 0) {
    vcycle_pcg(D, r, p, 0);
    R.vcycles++;
    int dcur = 8, dnew = 10;
    dot(D, p, r, nullptr, nullptr, dcur);
    while (R.iters < o.imax) {
      each(D, [&](sem_ctx* c, int i) { CUDA_CHECK(cudaMemsetAsync(q[i], 0, sizeof(double) * c->L[0].n, c->stream)); });
      apply_exchange(D, 0, p, q, 0);
      dot(D, p, q, nullptr, nullptr, 1);
      each(D, [&](sem_ctx* c, int i) {
        if (flex) CUDA_CHECK(cudaMemcpyAsync(ro[i], r[i], sizeof(double) * c->L[0].n, cudaMemcpyDeviceToDevice, c->stream));
        launch_axpy_pcg(c, c->L[0].n, u[i], r[i], p[i], q[i], c->scal + dcur, c->scal + 1, c->scal + 3,
                        c->L[0].ownfree);
      });
      allreduce_scal(D, 3, 1);
      R.iters++;
      read_scal(D, 0, 4, h);
      if (!(h[1] > 0.0)) {
        status = SEM_EBREAKDOWN;
        break;
      }
      rn = std::sqrt(h[3]);
      if (R.n_hist < 256) R.res_hist[R.n_hist++] = rn;
      if (rn <= thresh) {
        R.converged = 1;
        break;
      }
      vcycle_pcg(D, r, z, 1);
      R.vcycles++;
      if (flex) {
        dot(D, z, r, &z, &ro, dnew);
        each(D, [&](sem_ctx* c, int i) { launch_xpby(c, c->L[0].n, p[i], z[i], c->scal + dnew, c->scal + dcur, 2); });
      } else {
        dot(D, z, r, nullptr, nullptr, dnew);
        each(D, [&](sem_ctx* c, int i) { launch_xpby(c, c->L[0].n, p[i], z[i], c->scal + dnew, c->scal + dcur, 0); });
      }
      std::swap(dcur, dnew);
    }
  } else {
    while (R.iters < o.imax) {
      vcycle_pcg(D, r, z, 1);
      R.vcycles++;
      each(D, [&](sem_ctx* c, int i) {
        launch_axpy(c, c->L[0].n, 1.0, z[i], u[i]);
        CUDA_CHECK(cudaMemcpyAsync(r[i], ro[i], sizeof(double) * c->L[0].n, cudaMemcpyDeviceToDevice, c->stream));
      });
      apply_exchange(D, 0, u, r, AP_NEGATE);
      R.iters++;
      dot(D, r, r, nullptr, nullptr, 3);
      read_scal(D, 3, 1, h);
      rn = std::sqrt(h[0]);
      if (R.n_hist < 256) R.res_hist[R.n_hist++] = rn;
      if (rn <= thresh) {
        R.converged = 1;
        break;
      }
    }
  }
  each(D, [&](sem_ctx* c, int i) { launch_combine_phi(c, 0, u[i], phiD[i], phi[i]); });
  for (auto* c : D.parts) CUDA_CHECK(cudaStreamSynchronize(c->stream));
  CUDA_CHECK(cudaEventRecord(c0->ev1, c0->stream));
  CUDA_CHECK(cudaEventSynchronize(c0->ev1));
  float ms = 0.f;
  CUDA_CHECK(cudaEventElapsedTime(&ms, c0->ev0, c0->ev1));
  R.t_ms = ms;
  R.coarse_iters = (int)coarse_iters(D.coarse, false);
  coarse_count_launches(D.coarse, R.coarse_iters);
  R.rel_res = nf > 0 ? rn / nf : 0.0;
  if (R.n_hist > 1) R.q_mean = std::pow(R.res_hist[R.n_hist - 1] / R.res_hist[0], 1.0 / (R.n_hist - 1));
  if (status == SEM_OK && !R.converged) status = SEM_ENOTCONV;
  if (rep) *rep = R;
  return status;
}

// ------------------------------------------------------------------ setup
static void setup_exchange(sem_ctx* c, const LocalPart& P) {
  for (size_t li = 0; li < c->L.size(); ++li) {
    DeviceLevel& L = c->L[li];
    const LocalLevel& LL = P.L[li];
    L.nbr = LL.nbr;
    L.xoff.assign(1, 0);
    std::vector<int32_t> all;
    for (auto& v : LL.xidx) {
      all.insert(all.end(), v.begin(), v.end());
      L.xoff.push_back((int64_t)all.size());
    }
    L.xidx = upload(c, all);
    L.sendbuf = dalloc<double>(c, all.size());
    L.recvbuf = dalloc<double>(c, all.size());
    // interface / interior owned elements (apply_exchange)
    std::vector<uint8_t> shared(L.n, 0);
    for (int32_t i : all) shared[i] = 1;
    std::vector<int32_t> eif, ein;
    const int N = L.N;
    for (int e = 0; e < P.E_own; ++e) {
      bool s = false;
      for (int k = 0; k < N && !s; ++k) s = shared[LL.conn[(size_t)e * N + k]] != 0;
      (s ? eif : ein).push_back(e);
    }
    L.n_if = (int)eif.size();
    L.n_in = (int)ein.size();
    L.e_if = upload(c, eif);
    L.e_in = upload(c, ein);
    if (li + 1 < c->L.size() && !L.fdm && L.nsub == (int)LL.S.off.size() - 1) {  // dense: subdomain k = owned element k
      std::vector<int32_t> sif, sin;
      for (int k = 0; k < L.nsub; ++k) {
        bool s = false;
        for (int64_t t = LL.S.off[k]; t < LL.S.off[k + 1] && !s; ++t) s = shared[LL.S.idx[t]] != 0;
        (s ? sif : sin).push_back(k);
      }
      L.ns_if = (int)sif.size();
      L.ns_in = (int)sin.size();
      L.s_if = upload(c, sif);
      L.s_in = upload(c, sin);
    }
    // FDM level on the column-unit kernels: a unit is on the interface if any node of its column
    // range (the nodes its scatter writes) is exchanged
    const int fk = li + 1 < c->L.size() ? fdm_kernel_choice(L) : SEM_SMOOTHER_DENSE;
    if (L.fdm && li < P.F.size() &&
        (fk == SEM_SMOOTHER_FDM_WARP1 || fk == SEM_SMOOTHER_FDM_WARP2 || fk == SEM_SMOOTHER_FDM_CTA)) {
      const FdmTopo& F = P.F[li];
      std::vector<int4> hu(L.f_nunits);
      CUDA_CHECK(cudaMemcpy(hu.data(), L.f_units, hu.size() * sizeof(int4), cudaMemcpyDeviceToHost));
      std::vector<int32_t> uif, uin;
      for (int i = 0; i < L.f_nunits; ++i) {
        const int q = hu[i].x, e0 = F.colel[hu[i].y], e1 = F.colel[hu[i].y + hu[i].z - 1];
        const int nh = (int)(F.hoff[q + 1] - F.hoff[q]), nz = F.nzc[q];
        const int zlo = F.z0[e0], zhi = F.z0[e1] + F.nv[e1];
        bool s = false;
        for (int h = 0; h < nh && !s; ++h)
          for (int z = zlo; z < zhi && !s; ++z) {
            const int32_t g = F.cidx[F.cioff[q] + (int64_t)h * nz + z];
            s = g >= 0 && shared[g] != 0;
          }
        (s ? uif : uin).push_back(i);
      }
      L.nfu_if = (int)uif.size();
      L.nfu_in = (int)uin.size();
      L.fu_if = upload(c, uif.empty() ? std::vector<int32_t>{0} : uif);
      L.fu_in = upload(c, uin.empty() ? std::vector<int32_t>{0} : uin);
    }
  }
}

// column partition of the elements (RCB on the x,y centroids of the prisms'
// vertices) and the global Schwarz topologies of the levels < coarsest
void compute_partition(const GlobalModel& gm, const sem_opts& o, std::vector<int>& epart,
                       std::vector<SchwarzTopo>& sch) {
  const int E = gm.hm.E;
  const int nl = (int)gm.sched.size();
  std::vector<double> cx(E), cy(E);
  if (!gm.hm.xyz.empty()) {
    for (int e = 0; e < E; ++e) {
      double sx = 0, sy = 0;
      for (int a = 0; a < 6; ++a) {
        const int v = gm.hm.prism[(size_t)e * 6 + a];
        sx += gm.hm.xyz[3 * (size_t)v];
        sy += gm.hm.xyz[3 * (size_t)v + 1];
      }
      cx[e] = sx / 6;
      cy[e] = sy / 6;
    }
  } else {  // centroid of the nodes of the nodal map
    const int Nf = n_prism(gm.P);
    for (int e = 0; e < E; ++e) {
      double sx = 0, sy = 0;
      for (int n = 0; n < Nf; ++n) {
        sx += gm.X[((size_t)e * Nf + n) * 3];
        sy += gm.X[((size_t)e * Nf + n) * 3 + 1];
      }
      cx[e] = sx / Nf;
      cy[e] = sy / Nf;
    }
  }
  epart = gm.user_part.empty() ? partition_columns(cx, cy, o.nranks) : gm.user_part;
  sch.assign(nl - 1, SchwarzTopo());
  const int nth = std::min(32, std::max(1, omp_get_max_threads()));
  for (int l = 0; l + 1 < nl; ++l) {
    const int ov = o.overlap >= 0 ? o.overlap : (gm.sched[l] + 2) / 2;
    sch[l] = schwarz_topology(gm.topo[l], E, ov, nth);
  }
}

void setup_distributed(sem_ctx* c, GlobalModel& gm) {
  const sem_opts& o = c->opts;
  Dist* D = new Dist();
  c->dist = D;
  D->nranks = o.nranks;
  D->rank = o.rank;
  D->emulated = (o.nccl_id == nullptr);
  const int E = gm.hm.E;
  const int nl = (int)gm.sched.size();
  if (nl < 2) throw SemError(SEM_EUNSUPPORTED, "a partitioned solve needs at least two levels (p >= 2)");
  double t0 = now_ms();
  std::vector<int> epart;
  std::vector<SchwarzTopo> sch;
  compute_partition(gm, o, epart, sch);
  if (o.verbose) fprintf(stderr, "[sem] partition + global Schwarz topology %.0f ms\n", now_ms() - t0);
  std::vector<int> lids(nl);
  for (int i = 0; i < nl; ++i) lids[i] = i;
  std::vector<int> ranks;
  if (D->emulated) {
    for (int r = 0; r < o.nranks; ++r) ranks.push_back(r);
  } else {
    ranks.push_back(o.rank);
  }
  // FDM local solves (reading O33/O35): global topologies and hybrid weights, restricted per rank
  std::vector<FdmTopo> Fg;
  std::vector<std::vector<double>> Wh;
  if (o.local_solve == 1) {
    for (int l = 0; l + 1 < nl; ++l) {
      const int ov = o.overlap >= 0 ? o.overlap : (gm.sched[l] + 2) / 2;
      Fg.push_back(fdm_topology(gm.hm, gm.topo[l], gm.X, gm.P, ov, gm.PZ));
      const FdmTopo& F = Fg.back();
      std::vector<double> cnt(gm.topo[l].n, 0.0);
      for (int e = 0; e < E; ++e)
        if (F.regular[e]) {
          for (int64_t t = F.ioff[e]; t < F.ioff[e + 1]; ++t)
            if (F.idx[t] >= 0) cnt[F.idx[t]] += 1.0;
        } else {
          for (int64_t t = sch[l].off[e]; t < sch[l].off[e + 1]; ++t) cnt[sch[l].idx[t]] += 1.0;
        }
      std::vector<double> W(gm.topo[l].n, 0.0);
      for (int64_t i = 0; i < gm.topo[l].n; ++i) W[i] = gm.topo[l].dir[i] ? 0.0 : 1.0 / cnt[i];
      Wh.push_back(std::move(W));
    }
  }
  for (int r : ranks) {
    LocalPart P = extract_part(gm.topo, sch, epart, r, o.nranks);
    if (o.local_solve == 1)
      for (int l = 0; l + 1 < nl; ++l)
        P.F.push_back(fdm_local(Fg[l], P.elems, P.E_own, P.L[l].gid, gm.topo[l].n, Wh[l]));
    sem_ctx* pc = new sem_ctx();
    D->parts.push_back(pc);
    D->part_rank.push_back(r);
    pc->opts = o;
    pc->device = c->device;
    pc->stream = c->stream;
    pc->E_global = E;
    build_levels(pc, gm, lids, &P, nullptr);
    setup_exchange(pc, P);
    if (o.verbose)
      fprintf(stderr, "[sem] rank %d: %d owned + %d halo elements, %lld nodes, %zu neighbours\n", r, P.E_own,
              (int)P.elems.size() - P.E_own, (long long)P.L[0].n, P.L[0].nbr.size());
  }
  // whole-mesh P=1 coarse solver (the coarse problem is gathered, north_star)
  D->coarse = new sem_ctx();
  D->coarse->opts = o;
  D->coarse->device = c->device;
  D->coarse->stream = c->stream;
  D->coarse->E_global = E;
  build_levels(D->coarse, gm, std::vector<int>{nl - 1}, nullptr, nullptr);
  // global bookkeeping for the API
  for (int l = 0; l < nl; ++l) {
    D->gn.push_back(gm.topo[l].n);
    D->gnfree.push_back(gm.topo[l].nfree);
    D->gp.push_back(gm.sched[l]);
    D->gdir.push_back(gm.topo[l].dir);
  }
  {  // global node coordinates per level from the whole-mesh map
    for (int l = 0; l < nl; ++l) {
      const LevelTopo& T = gm.topo[l];
      const int p = gm.P, pl = gm.sched[l];
      std::vector<double> It, I1;
      transfer_matrices(pl, p, It, I1);
      const int ntl = n_tri(pl), n1l = pl + 1, ntf = n_tri(p), n1f = p + 1, Nf = n_prism(p), Nl = T.N;
      std::vector<double> xyz((size_t)T.n * 3, 0.0);
#pragma omp parallel for
      for (int e = 0; e < E; ++e)
        for (int l2 = 0; l2 < n1l; ++l2)
          for (int m = 0; m < ntl; ++m) {
            const int n = m + ntl * l2;
            if (!T.owner[(size_t)e * Nl + n]) continue;
            double x[3] = {0, 0, 0};
            for (int lf = 0; lf < n1f; ++lf)
              for (int mf = 0; mf < ntf; ++mf) {
                const double w = It[(size_t)m * ntf + mf] * I1[(size_t)l2 * n1f + lf];
                if (w == 0.0) continue;
                const double* Xn = &gm.X[((size_t)e * Nf + mf + ntf * lf) * 3];
                for (int i = 0; i < 3; ++i) x[i] += w * Xn[i];
              }
            const int32_t g = T.conn[(size_t)e * Nl + n];
            for (int i = 0; i < 3; ++i) xyz[3 * (size_t)g + i] = x[i];
          }
      D->gxyz.push_back(std::move(xyz));
    }
  }
  D->gbuf = dalloc<double>(c, D->gn[0]);
  D->gbuf2 = dalloc<double>(c, D->gn[0]);
  D->gbuf3 = dalloc<double>(c, D->gn[0]);
  D->cx = dalloc<double>(c, D->gn.back());
  D->cz = dalloc<double>(c, D->gn.back());
  CUDA_CHECK(cudaMallocHost(&D->hsum, 32 * sizeof(double)));
  {
    // SEM_DIST_OVERLAP: unset = on for the NCCL transport, off for emulated ranks (one GPU runs
    // them one after another: there is no transfer to hide, only the split launches' tails);
    // 0 = off; 1 = on; 2 = on with every FDM sweep split (below)
    const char* ov = getenv("SEM_DIST_OVERLAP");
    D->overlap = ov ? atoi(ov) != 0 : !D->emulated;
    // FDM sweeps are split only when the interface units fill a few waves of the GPU by
    // themselves: a small interface launch under-fills the SMs and the split sweep loses more
    // to wave tails than the hidden transfer saves (emulated config 3, 4 ranks: 78.6 ms serial
    // vs 87.9 ms always split).  SEM_DIST_OVERLAP=2 splits every FDM sweep (tests).
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device >= 0 ? c->device : 0);
    D->fdm_ov_min = (ov && atoi(ov) == 2) ? 0 : 8 * sms;
    CUDA_CHECK(cudaStreamCreateWithFlags(&D->comm_stream, cudaStreamNonBlocking));
    CUDA_CHECK(cudaEventCreateWithFlags(&D->ev_pack, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&D->ev_xfer, cudaEventDisableTiming));
  }
  if (!D->emulated) {
    ncclUniqueId id;
    memcpy(&id, o.nccl_id, sizeof(id));
    NCCL_CHECK(nccl().CommInitRank(&D->comm, o.nranks, id, o.rank));
  }
  c->E = E;
  c->E_own = E;
  c->P = gm.P;
  CUDA_CHECK(cudaEventCreate(&c->ev0));
  CUDA_CHECK(cudaEventCreate(&c->ev1));
}

// ------------------------------------------------------------------ API glue (global vectors)
static Vecs scatter_global(Dist& D, int li, const double* g, double* sem_ctx::*buf) {
  Vecs out;
  each(D, [&](sem_ctx* c, int) {
    double* l = (buf == nullptr) ? c->L[li].f : c->*buf;
    if (g) {
      k_scatter_from_global<<<gsz(c->L[li].n), 256, 0, c->stream>>>(c->L[li].n, c->L[li].gid, g, l);
      c->launches++;
    }
    out.push_back(g ? l : nullptr);
  });
  return out;
}

static void gather_global(Dist& D, int li, const Vecs& l, double* g) {
  sem_ctx* c0 = D.parts[0];
  CUDA_CHECK(cudaMemsetAsync(g, 0, sizeof(double) * D.gn[li], c0->stream));
  each(D, [&](sem_ctx* c, int i) {
    DeviceLevel& L = c->L[li];
    k_gather_owned<<<gsz(L.n), 256, 0, c->stream>>>(L.n, L.gid, L.owned_dev, l[i], g);
    c->launches++;
  });
  allreduce_vec(D, g, D.gn[li]);
}

int dist_solve(sem_ctx* c, const double* rhs, const double* phiD, double tol, double* phi, sem_report* rep) {
  NvtxRange nv("laplace_solve (partitioned)");
  Dist& D = *c->dist;
  Vecs vr = scatter_global(D, 0, rhs, &sem_ctx::host_in2);
  Vecs vd = scatter_global(D, 0, phiD, &sem_ctx::host_in);
  Vecs vp;
  for (auto* pc : D.parts) vp.push_back(pc->host_out);
  if (!rhs) vr.clear();
  int st = solve(D, vr, vd, tol, vp, rep);
  gather_global(D, 0, vp, phi);
  for (auto* pc : D.parts) CUDA_CHECK(cudaStreamSynchronize(pc->stream));
  return st;
}

int dist_vcycle(sem_ctx* c, const double* r, double* z) {
  Dist& D = *c->dist;
  Vecs vr = scatter_global(D, 0, r, &sem_ctx::host_in);
  Vecs vz;
  for (auto* pc : D.parts) vz.push_back(pc->host_out);
  vcycle(D, 0, vr, vz);
  gather_global(D, 0, vz, z);
  return SEM_OK;
}

int dist_apply(sem_ctx* c, const double* u, double* y, int level, int masked) {
  Dist& D = *c->dist;
  if (level < 0 || level >= (int)D.gn.size()) return SEM_EINVAL;
  Vecs vu, vy;
  each(D, [&](sem_ctx* pc, int) {
    DeviceLevel& L = pc->L[level];
    k_scatter_from_global<<<gsz(L.n), 256, 0, pc->stream>>>(L.n, L.gid, u, L.f);
    pc->launches++;
    vu.push_back(L.f);
    vy.push_back(L.r);
    if (masked) {
      // y_F = A_FF u_F (partial), y_D = u_D on the owning rank only (single count)
      CUDA_CHECK(cudaMemsetAsync(L.r, 0, sizeof(double) * L.n, pc->stream));
      launch_apply(pc, level, L.f, L.r, 0);
    } else {
      CUDA_CHECK(cudaMemsetAsync(L.r, 0, sizeof(double) * L.n, pc->stream));
      launch_apply(pc, level, L.f, L.r, AP_GATHER_ALL | AP_SCATTER_ALL);
    }
  });
  exchange(D, level, vy);
  if (masked)
    each(D, [&](sem_ctx* pc, int i) {
      // Dirichlet rows: identity (y_D = u_D)
      launch_init_masked(pc, level, vu[i], vy[i], 3);
    });
  gather_global(D, level, vy, y);
  return SEM_OK;
}

void dist_info(const sem_ctx* c, sem_info* info) {
  const Dist& D = *c->dist;
  info->n_dof = D.gn[0];
  info->n_free = D.gnfree[0];
  info->n_elem = c->E_global;
  info->n_levels = (int)D.gn.size();
  for (size_t i = 0; i < D.gn.size(); ++i) {
    info->level_p[i] = D.gp[i];
    info->level_n_dof[i] = D.gn[i];
    info->level_n_free[i] = D.gnfree[i];
    for (auto* pc : D.parts) {
      info->schwarz_bytes[i] += pc->L[i].schwarz_bytes;
      info->schwarz_nk_sum[i] += pc->L[i].nk_sum;
      info->schwarz_packed[i] += pc->L[i].packed;
    }
    const sem_ctx* p0 = D.parts[0];
    if (i + 1 < D.gn.size() && i < p0->L.size()) {
      info->smoother_kernel[i] = fdm_kernel_choice(p0->L[i]);
      info->smoother_mt[i] = p0->L[i].fdm ? p0->L[i].f_mt : 0;
    }
  }
  info->coarse_n = D.coarse->C.nc;
  info->coarse_agg = D.coarse->C.nagg;
  info->device_bytes = c->device_bytes + D.coarse->device_bytes;
  for (auto* pc : D.parts) info->device_bytes += pc->device_bytes;
}

const std::vector<double>& dist_xyz(const sem_ctx* c, int level) { return c->dist->gxyz[level]; }
const std::vector<uint8_t>& dist_dir(const sem_ctx* c, int level) { return c->dist->gdir[level]; }
int dist_levels(const sem_ctx* c) { return (int)c->dist->gn.size(); }
sem_ctx* dist_part0(const sem_ctx* c) { return c->dist->parts[0]; }

int64_t dist_launches(const sem_ctx* c, int reset) {
  Dist& D = *c->dist;
  int64_t v = 0;
  for (auto* pc : D.parts) {
    v += pc->launches;
    if (reset) pc->launches = 0;
  }
  v += D.coarse->launches;
  if (reset) D.coarse->launches = 0;
  return v;
}

void dist_destroy(sem_ctx* c) {
  Dist* D = c->dist;
  if (!D) return;
  cudaDeviceSynchronize();
  for (auto* pc : D->parts) sem_destroy(pc);
  if (D->coarse) sem_destroy(D->coarse);
  if (D->comm) nccl().CommDestroy(D->comm);
  if (D->hsum) cudaFreeHost(D->hsum);
  if (D->ev_pack) cudaEventDestroy(D->ev_pack);
  if (D->ev_xfer) cudaEventDestroy(D->ev_xfer);
  if (D->comm_stream) cudaStreamDestroy(D->comm_stream);
  for (auto& e : D->vc_exec)
    if (e) cudaGraphExecDestroy(e);
  if (D->cap_stream) cudaStreamDestroy(D->cap_stream);
  delete D;
  c->dist = nullptr;
}

void nccl_unique_id(void* out) {
  ncclUniqueId id;
  NCCL_CHECK(nccl().GetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
}

}  // namespace sem
