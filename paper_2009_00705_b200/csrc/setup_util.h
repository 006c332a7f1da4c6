// Setup helpers shared by capi.cu (single domain) and dist.cu (partitioned).
#pragma once
#include <algorithm>
#include <string>
#include <vector>

#include "internal.h"
#include "partition.h"

namespace sem {

template <class T>
inline T* dalloc(sem_ctx* c, size_t count) {
  if (count == 0) count = 1;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw SemError(SEM_ENOMEM, "cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed");
  }
  c->allocs.push_back(p);
  c->device_bytes += (int64_t)(count * sizeof(T));
  return (T*)p;
}

template <class T>
inline T* upload(sem_ctx* c, const std::vector<T>& v) {
  T* d = dalloc<T>(c, v.size());
  if (!v.empty()) CUDA_CHECK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

// scratch allocation freed at the end of setup
struct Scratch {
  std::vector<void*> ptrs;
  template <class T>
  T* get(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw SemError(SEM_ENOMEM, "setup scratch cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed");
    }
    ptrs.push_back(p);
    return (T*)p;
  }
  template <class T>
  T* put(const std::vector<T>& v) {
    T* d = get<T>(v.size());
    if (!v.empty()) CUDA_CHECK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
  }
  void release(void* p) {
    auto it = std::find(ptrs.begin(), ptrs.end(), p);
    if (it != ptrs.end()) { cudaFree(p); ptrs.erase(it); }
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFree(p);
  }
};

struct GlobalModel {
  HostMesh hm;
  int P = 0, PZ = 0;              // finest horizontal / vertical order (PZ = P isotropic)
  std::vector<int> sched;         // horizontal order of every level, finest first
  std::vector<int> schedz;        // vertical order of every level
  std::vector<double> X;          // [E][N(P)][3] finest nodal map
  std::vector<LevelTopo> topo;    // global numbering per level
  std::vector<int> user_part;     // sem_mesh.part (empty = the library's column partition)
};

void build_levels(sem_ctx* c, const GlobalModel& gm, const std::vector<int>& lids, const LocalPart* part,
                  const std::vector<SchwarzTopo>* gsch);
void setup_distributed(sem_ctx* c, GlobalModel& gm);
void compute_partition(const GlobalModel& gm, const sem_opts& o, std::vector<int>& epart,
                       std::vector<SchwarzTopo>& sch);
void prepare_global(const sem_mesh* mesh, int p, const sem_opts& o, GlobalModel& gm);
double now_ms();
void read_scalars(sem_ctx* c, int n);
void coarse_solve(sem_ctx* c, const double* f, double* u);

}  // namespace sem
