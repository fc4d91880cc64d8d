// FP64 pipe microbenchmark: DFMA throughput vs (warps/SM, independent chains/thread).
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void k(double* out, int iters, double x, double y) {
  double a[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = fma(a[i], x, y);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}
template <int ILP>
void run(int sms, int warps_per_sm) {
  double* d; cudaMalloc(&d, 8);
  int threads = 32 * (warps_per_sm < 32 ? warps_per_sm : 32);
  int blocks = sms * warps_per_sm * 32 / threads;
  int iters = 4096;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<ILP><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(a);
  k<ILP><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = double(blocks) * threads * iters * ILP;
  printf("ILP %2d warps/SM %2d: %.1f TFMA-lane/s  (%.1f lane-FMA/clk/SM @1.965GHz)\n", ILP, warps_per_sm,
         ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
  cudaFree(d);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 12, 16, 24, 32}) { run<1>(sms, w); run<2>(sms, w); run<4>(sms, w); run<8>(sms, w); }
  // dependent-chain latency: 1 warp per SM, ILP 1
  run<1>(sms, 1);
  return 0;
}
