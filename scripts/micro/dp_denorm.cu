// FP64 throughput vs operand class (normal / subnormal / zero): 8 independent
// DMUL+DADD chains per thread, 148*8 blocks x 256 threads, CUDA-event timed.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, double a, double b, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = a * (1.0 + threadIdx.x * 1e-9 + i * 1e-10);
  for (int n = 0; n < iters; ++n) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __dadd_rn(__dmul_rn(x[i], b), a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* o;
  cudaMalloc(&o, 148 * 8 * 256 * 8);
  struct { const char* nm; double a, b; } cases[] = {
      {"normal", 1.0e-3, 0.5}, {"zero", 0.0, 0.0}, {"subnormal", 1e-310, 0.5}, {"sub*normal->sub", 3e-310, 0.999},
      {"normal*tiny->sub", 1e-300, 1e-10}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (auto& c : cases) {
    k<<<148 * 8, 256>>>(o, c.a, c.b, 100);
    cudaEventRecord(e0);
    const int it = 4000;
    k<<<148 * 8, 256>>>(o, c.a, c.b, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 148.0 * 8 * 256 * it * 8 * 2;
    printf("%-18s %8.3f ms  %7.2f G DP-ops/s\n", c.nm, ms, ops / ms / 1e6);
  }
  return 0;
}
