#include <cstdio>
__global__ void k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8] = {0,0,0,0,0,0,0,0};
  double d0=0,d1=0,d2=0,d3=0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[2*j]), "+d"(c[2*j+1]) : "d"(a), "d"(b));
    }
  }
  double s=0; for (int j=0;j<8;++j) s+=c[j];
  out[blockIdx.x*blockDim.x+threadIdx.x] = s;
}
__global__ void k16(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0+1, a2=a0+2, a3=a0+3, b0 = 1.0 + threadIdx.x * 1e-4, b1=b0+1;
  double c[16] = {0};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[4*j]), "+d"(c[4*j+1]), "+d"(c[4*j+2]), "+d"(c[4*j+3]) : "d"(a0),"d"(a1),"d"(a2),"d"(a3), "d"(b0),"d"(b1));
    }
  }
  double s=0; for (int j=0;j<16;++j) s+=c[j];
  out[blockIdx.x*blockDim.x+threadIdx.x] = s;
}
__global__ void kf(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16]; for(int j=0;j<16;++j) c[j]=j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = fma(a, c[j], b);
  }
  double s=0; for (int j=0;j<16;++j) s+=c[j];
  out[blockIdx.x*blockDim.x+threadIdx.x] = s;
}
int main() {
  double* o; cudaMalloc(&o, 148*32*256*8);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int it = 20000; float ms;
  for (int rep=0; rep<2; ++rep) {
  k<<<148*4, 256>>>(o, it); cudaEventRecord(e0); k<<<148*4, 256>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 148.0*4*8 * it * 4 * 512.0; printf("m8n8k4 DMMA: %.2f TFLOP/s\n", fl/ms/1e9);
  k16<<<148*4, 256>>>(o, it); cudaEventRecord(e0); k16<<<148*4, 256>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  fl = 148.0*4*8 * it * 4 * 2048.0; printf("m16n8k8 DMMA: %.2f TFLOP/s\n", fl/ms/1e9);
  kf<<<148*4, 256>>>(o, it); cudaEventRecord(e0); kf<<<148*4, 256>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  fl = 148.0*4*256 * it * 16 * 2.0; printf("DFMA: %.2f TFLOP/s\n", fl/ms/1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
