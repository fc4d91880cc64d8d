// div_check.cu -- the STRICT locate's division RN(x/d) as q = x*rd,
// r = fma(-q, d, x), fma(r, rd, q) with rd = RN(1/d) from the host (b2m::div_axis in b2m_mover.cuh), against
// the IEEE division __ddiv_rn, for x in [0, l): random mantissas over the
// top 40 binades below l, and every x within +-32 ulps of each cell face k*d
// (the truncation boundary).  Divisors: the C1-C5 grid spacings, the test
// grids, and random d.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -Iinclude -Ipaper_1904_03684_b200/csrc tools/micro/div_check.cu -o /tmp/div_check
//   && /tmp/div_check [rounds]
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// the product's function itself (B2M_STRICT_DIV=1 path)
#define B2M_STRICT_DIV 1
#include "b2m_mover.cuh"

__device__ __forceinline__ double fast_div(double x, double d, double rd) {
  return b2m::div_axis(x, d, rd);
}

__global__ void random_x(const double* ds, const double* rds, const double* ls, int nd,
                         uint64_t per_d, uint64_t seed, unsigned long long* bad,
                         double* example) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (int di = 0; di < nd; ++di) {
    const double d = ds[di], rd = rds[di], l = ls[di];
    int el;
    frexp(l, &el);
    for (uint64_t s = t; s < per_d; s += stride) {
      const uint64_t h = mix(seed ^ (s * 0x632BE59BD9B4E019ull) ^ ((uint64_t)di << 56));
      const int e = el - 1 - (int)((h >> 52) % 40);
      const double m = 1.0 + (double)(h & ((1ull << 52) - 1)) * 0x1p-52;
      const double x = ldexp(m, e);
      if (!(x < l)) continue;
      if (fast_div(x, d, rd) != __ddiv_rn(x, d)) {
        if (atomicAdd(bad, 1ull) == 0) { example[0] = x; example[1] = d; }
      }
    }
  }
}

__global__ void faces(const double* ds, const double* rds, const int* ns, int nd,
                      unsigned long long* bad, double* example) {
  const int di = blockIdx.y;
  const double d = ds[di], rd = rds[di];
  const int n = ns[di];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k <= n; k += gridDim.x * blockDim.x) {
    const double c = __dmul_rn((double)k, d);
    long long cb = __double_as_longlong(c);
    for (int u = -32; u <= 32; ++u) {
      const long long b = cb + u;
      if (b < 0) continue;
      const double x = __longlong_as_double(b);
      if (fast_div(x, d, rd) != __ddiv_rn(x, d)) {
        if (atomicAdd(bad, 1ull) == 0) { example[0] = x; example[1] = d; }
      }
    }
  }
}

int main(int argc, char** argv) {
  const int rounds = argc > 1 ? atoi(argv[1]) : 4;
  // (l, n) of C1..C5 and the test grids
  std::vector<double> L = {6.4, 25.6, 12.8, 6.4, 51.2, 25.6, 12.8, 4.0, 3.0, 2.5, 3.5, 6.4, 12.8,
                           1.0, 10.0, 7.0};
  std::vector<int> N = {8, 64, 64, 32, 128, 128, 64, 4, 6, 5, 7, 16, 32, 3, 7, 9};
  srand(12345);
  for (int i = 0; i < 4000; ++i) {  // random (l, n): l in [0.01, 1000), n in [2, 1024]
    const double l = std::exp(std::log(0.01) + (std::log(1000.0) - std::log(0.01)) * (rand() / (RAND_MAX + 1.0)));
    L.push_back(l);
    N.push_back(2 + rand() % 1023);
  }
  const int nd = (int)L.size();
  std::vector<double> D(nd), RD(nd);
  for (int i = 0; i < nd; ++i) { D[i] = L[i] / N[i]; RD[i] = 1.0 / D[i]; }
  double *dd, *drd, *dl, *ex;
  int* dn;
  unsigned long long* bad;
  cudaMalloc(&dd, nd * 8); cudaMalloc(&drd, nd * 8); cudaMalloc(&dl, nd * 8); cudaMalloc(&dn, nd * 4);
  cudaMalloc(&ex, 16); cudaMalloc(&bad, 8);
  cudaMemcpy(dd, D.data(), nd * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(drd, RD.data(), nd * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dl, L.data(), nd * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dn, N.data(), nd * 4, cudaMemcpyHostToDevice);
  cudaMemset(bad, 0, 8);
  faces<<<dim3(8, nd), 128>>>(dd, drd, dn, nd, bad, ex);
  unsigned long long hb = 0;
  double hex[2] = {0, 0};
  cudaDeviceSynchronize();
  cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hex, ex, 16, cudaMemcpyDeviceToHost);
  uint64_t faces_n = 0;
  for (int i = 0; i < nd; ++i) faces_n += (uint64_t)(N[i] + 1) * 65;
  printf("faces: %llu values, %llu mismatches%s\n", (unsigned long long)faces_n, hb,
         hb ? "" : "");
  if (hb) printf("  e.g. x=%a d=%a\n", hex[0], hex[1]);
  // random x: 16 named spacings x 2^30 each, random spacings x 2^22 each, per round
  unsigned long long total = 0, tb = 0;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < rounds; ++r) {
    cudaMemset(bad, 0, 8);
    random_x<<<148 * 16, 256>>>(dd, drd, dl, 16, 1ull << 30, 1000 + r, bad, ex);
    random_x<<<148 * 16, 256>>>(dd + 16, drd + 16, dl + 16, nd - 16, 1ull << 22, 2000 + r, bad, ex);
    cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
    total += 16ull * (1ull << 30) + (uint64_t)(nd - 16) * (1ull << 22);
    tb += hb;
    if (hb) {
      cudaMemcpy(hex, ex, 16, cudaMemcpyDeviceToHost);
      printf("  round %d mismatch e.g. x=%a d=%a\n", r, hex[0], hex[1]);
    }
  }
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("random: %llu values over %d divisors, %llu mismatches (%.1f s)\n", total, nd, tb,
         ms / 1e3);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 2; }
  return (tb || hb) ? 1 : 0;
}
