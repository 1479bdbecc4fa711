// FP64 dependent-chain latency and LDS latency on one warp (clock64 timed).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dadd(double* out, double a, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x = __dadd_rn(x, a);
    x = __dadd_rn(x, a);
    x = __dadd_rn(x, a);
    x = __dadd_rn(x, a);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_dmul(double* out, double a, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x = __dmul_rn(x, a);
    x = __dmul_rn(x, a);
    x = __dmul_rn(x, a);
    x = __dmul_rn(x, a);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_lds(double* out, int n, long long* cyc) {
  __shared__ long long idx[256];
  idx[threadIdx.x] = (threadIdx.x + 1) % 32;
  __syncthreads();
  long long j = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    j = idx[j];
    j = idx[j];
    j = idx[j];
    j = idx[j];
  }
  long long t1 = clock64();
  out[threadIdx.x] = (double)j;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 1024 * 8);
  cudaMalloc(&c, 8);
  long long h;
  const int n = 4096;
  k_dadd<<<1, 32>>>(o, 1.0000001, n, c);
  k_dadd<<<1, 32>>>(o, 1.0000001, n, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  k_dmul<<<1, 32>>>(o, 1.0000001, n, c);
  k_dmul<<<1, 32>>>(o, 1.0000001, n, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DMUL dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  k_lds<<<1, 32>>>(o, n, c);
  k_lds<<<1, 32>>>(o, n, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("LDS.64 dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  return 0;
}
