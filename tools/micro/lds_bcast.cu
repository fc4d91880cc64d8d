// L1 / shared-memory -> register delivery microbenchmark: how many bytes per
// clock per SM reach registers when the lanes of a warp read the SAME
// address (broadcast), a few distinct addresses, or all-distinct addresses,
// for 128-bit shared loads (LDS.128) and 256-bit / 128-bit global .nc loads
// that hit L1.  Decides whether a shared-memory cell cache can replace the
// register cell cache of the FAST mover.
#include <cstdio>
#include <cuda_runtime.h>

// MODE: 0 broadcast, 1 two groups, 2 four groups, 3 all lanes distinct
template <int MODE>
__device__ __forceinline__ int lane_off(int lane) {
  if (MODE == 0) return 0;
  if (MODE == 1) return (lane >> 4) * 24;   // 384 B apart (another cell), in double2 units
  if (MODE == 2) return (lane >> 3) * 24;
  return lane;                               // consecutive 16 B
}

template <int MODE>
__global__ void lds_k(int iters, unsigned* out) {
  __shared__ double2 s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_double2(i, -i);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int base = lane_off<MODE>(lane);
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const double2 v = s[(base + u * 2 + (it & 7) * 32) & 2047];
      acc ^= __double2loint(v.x) ^ __double2hiint(v.y);
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int MODE, bool WIDE>
__global__ void ldg_k(const double2* __restrict__ g, int iters, unsigned* out) {
  const int lane = threadIdx.x & 31;
  const int base = (WIDE && MODE == 3) ? 2 * lane : lane_off<MODE>(lane);
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const double2* p = g + ((base + u * 2 + (it & 7) * 32) & 2047);
      if (WIDE) {
        double a, b, c, d;
        asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
        acc ^= __double2loint(a) ^ __double2hiint(b) ^ __double2loint(c) ^ __double2hiint(d);
      } else {
        const double2 v = __ldg(p);
        acc ^= __double2loint(v.x) ^ __double2hiint(v.y);
      }
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <typename K, typename... A>
void timeit(const char* name, K kern, int sms, int warps, int bytes_per_load, A... args) {
  const int threads = 32 * warps;
  const int iters = 2048;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<sms, threads>>>(args..., iters, nullptr);
  cudaEventRecord(a);
  kern<<<sms, threads>>>(args..., iters, nullptr);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = double(sms) * threads * iters * 16 * bytes_per_load;
  const double clk = ms * 1e-3 * 1.965e9;
  printf("%-34s warps %2d: %7.1f B/clk/SM delivered to registers (%6.2f warp-loads/clk/SM)\n", name,
         warps, bytes / clk / sms, double(sms) * warps * iters * 16 / clk / sms);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double2* g;
  cudaMalloc(&g, 2048 * sizeof(double2) + 64);
  cudaMemset(g, 0, 2048 * sizeof(double2) + 64);
  for (int w : {8, 16}) {
    timeit("LDS.128 broadcast", lds_k<0>, sms, w, 16);
    timeit("LDS.128 2 addresses", lds_k<1>, sms, w, 16);
    timeit("LDS.128 4 addresses", lds_k<2>, sms, w, 16);
    timeit("LDS.128 all distinct", lds_k<3>, sms, w, 16);
    timeit("LDG.128 broadcast (L1 hit)", ldg_k<0, false>, sms, w, 16, (const double2*)g);
    timeit("LDG.128 all distinct (L1 hit)", ldg_k<3, false>, sms, w, 16, (const double2*)g);
    timeit("LDG.256 broadcast (L1 hit)", ldg_k<0, true>, sms, w, 32, (const double2*)g);
    timeit("LDG.256 2 addresses (L1 hit)", ldg_k<1, true>, sms, w, 32, (const double2*)g);
    timeit("LDG.256 all distinct (L1 hit)", ldg_k<3, true>, sms, w, 32, (const double2*)g);
  }
  return 0;
}
