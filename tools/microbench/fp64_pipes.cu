// FP64 pipe microbenchmark (sm_100a): DMMA m8n8k4 / m16n8k8 / m16n8k16 alone, DFMA alone,
// and DMMA + DFMA issued together (same warp interleaved; split across warps) to see
// whether the tensor FP64 path and the FP64 FMA pipe add up.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_pipes fp64_pipes.cu
#include <cstdio>

#define DMMA4(c0, c1, a, b) \
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b))

__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16] = {0};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) DMMA4(c[2 * j], c[2 * j + 1], a, b);
  }
  double s = 0;
  for (int j = 0; j < 16; ++j) s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_m16n8k8(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 1.0 + threadIdx.x * 1e-4, b1 = b0 + 1;
  double c[16] = {0};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+d"(c[4 * j]), "+d"(c[4 * j + 1]), "+d"(c[4 * j + 2]), "+d"(c[4 * j + 3])
          : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
  for (int j = 0; j < 16; ++j) s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_m16n8k16(double* out, int iters) {
  double a[8], b[4];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int j = 0; j < 4; ++j) b[j] = 1.0 + threadIdx.x * 1e-4 + j;
  double c[16] = {0};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
          "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
          : "+d"(c[4 * j]), "+d"(c[4 * j + 1]), "+d"(c[4 * j + 2]), "+d"(c[4 * j + 3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
            "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  for (int j = 0; j < 16; ++j) s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16];
  for (int j = 0; j < 16; ++j) c[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = fma(a, c[j], b);
  }
  double s = 0;
  for (int j = 0; j < 16; ++j) s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mode 0: every warp issues 8 DMMA + NF DFMA per iteration; mode 1: even warps DMMA, odd warps DFMA
template <int NF>
__global__ void k_mix(double* out, int iters, int mode) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16] = {0};
  double f[16];
  for (int j = 0; j < 16; ++j) f[j] = j;
  const int w = threadIdx.x >> 5;
  const bool do_d = mode == 0 || (w & 1) == 0, do_f = mode == 0 || (w & 1) == 1;
  for (int i = 0; i < iters; ++i) {
    if (do_d) {
#pragma unroll
      for (int j = 0; j < 8; ++j) DMMA4(c[2 * j], c[2 * j + 1], a, b);
    }
    if (do_f) {
#pragma unroll
      for (int j = 0; j < NF; ++j) f[j & 15] = fma(a, f[j & 15], b);
    }
  }
  double s = 0;
  for (int j = 0; j < 16; ++j) s += c[j] + f[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* o;
  cudaMalloc(&o, 148 * 32 * 1024 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int it = 20000, G = 148 * 4, T = 256;
  float ms;
  auto timeit = [&](auto launch) {
    launch();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    return (double)ms;
  };
  const double thr = (double)G * T, warps = thr / 32;
  double t;
  t = timeit([&] { k_dmma<<<G, T>>>(o, it); });
  printf("DMMA m8n8k4 alone: %.2f TFLOP/s\n", warps * it * 8 * 512.0 / t / 1e9);
  t = timeit([&] { k_m16n8k8<<<G, T>>>(o, it); });
  printf("DMMA m16n8k8 alone: %.2f TFLOP/s\n", warps * it * 4 * 2048.0 / t / 1e9);
  t = timeit([&] { k_m16n8k16<<<G, T>>>(o, it); });
  printf("DMMA m16n8k16 alone: %.2f TFLOP/s\n", warps * it * 4 * 4096.0 / t / 1e9);
  t = timeit([&] { k_dfma<<<G, T>>>(o, it); });
  printf("DFMA alone: %.2f TFLOP/s\n", thr * it * 16 * 2.0 / t / 1e9);
  for (int mode = 0; mode < 2; ++mode) {
    const double wd = mode == 0 ? warps : warps / 2, wf = mode == 0 ? warps : warps / 2;
    t = timeit([&] { k_mix<8><<<G, T>>>(o, it, mode); });
    printf("mix mode %d NF=8 : DMMA %.2f + DFMA %.2f = %.2f TFLOP/s (%.3f ms)\n", mode, wd * it * 8 * 512.0 / t / 1e9,
           wf * 32 * it * 8 * 2.0 / t / 1e9, (wd * it * 8 * 512.0 + wf * 32 * it * 8 * 2.0) / t / 1e9, t);
    t = timeit([&] { k_mix<16><<<G, T>>>(o, it, mode); });
    printf("mix mode %d NF=16: DMMA %.2f + DFMA %.2f = %.2f TFLOP/s (%.3f ms)\n", mode, wd * it * 8 * 512.0 / t / 1e9,
           wf * 32 * it * 16 * 2.0 / t / 1e9, (wd * it * 8 * 512.0 + wf * 32 * it * 16 * 2.0) / t / 1e9, t);
    t = timeit([&] { k_mix<64><<<G, T>>>(o, it, mode); });
    printf("mix mode %d NF=64: DMMA %.2f + DFMA %.2f = %.2f TFLOP/s (%.3f ms)\n", mode, wd * it * 8 * 512.0 / t / 1e9,
           wf * 32 * it * 64 * 2.0 / t / 1e9, (wd * it * 8 * 512.0 + wf * 32 * it * 64 * 2.0) / t / 1e9, t);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
