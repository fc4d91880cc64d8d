// b2m_field.cu — the field phase stand-in on the GPU.
//
// Reference: pic::field_phase_stub (kernels.cpp:185-215): `passes` rounds of
//   E'(n) = e + (1/12) * ((((d_im + d_ip) + d_jm) + d_jp) + d_km) + d_kp),
//   d_x = E(x) - e, e = E(n),
// over the unique periodic nodes (i < nx, j < ny, k < nz), ping-ponging
// between two meshes, then mirror_seams (field_mesh.hpp:46-59) copies the
// 0-planes of E and B onto the n-planes; B passes through.  Every operation
// is rounded on its own in the reference's order (no FMA), so the result is
// bit-identical.  One thread per (node, component): an HBM-bound stencil
// whose neighbours come from L1/L2.
#include "b2m_internal.hpp"

namespace b2m {

namespace {

constexpr int kStubThreads = 256;

unsigned grid_for(long long n, int threads) {
  return static_cast<unsigned>((n + threads - 1) / threads);
}

// grid (ceil(3*nx / threads), ny, nz): a thread per (i, component) of one
// (j, k) row -- no 64-bit index divisions
__global__ void __launch_bounds__(kStubThreads)
    field_stub_kernel(int nx, int ny, int nz, const double* __restrict__ cur,
                      double* __restrict__ nxt) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 3 * nx) return;
  const int a = t % 3, i = t / 3;
  const int j = blockIdx.y, k = blockIdx.z;
  const int im = i == 0 ? nx - 1 : i - 1, ip = i + 1 == nx ? 0 : i + 1;
  const int jm = j == 0 ? ny - 1 : j - 1, jp = j + 1 == ny ? 0 : j + 1;
  const int km = k == 0 ? nz - 1 : k - 1, kp = k + 1 == nz ? 0 : k + 1;
  const long long sx = nx + 1, sy = ny + 1;
  auto at = [&](int ii, int jj, int kk) { return __ldg(cur + 3 * (ii + sx * (jj + sy * kk)) + a); };
  const double e = at(i, j, k);
  double sum = __dsub_rn(at(im, j, k), e);
  sum = __dadd_rn(sum, __dsub_rn(at(ip, j, k), e));
  sum = __dadd_rn(sum, __dsub_rn(at(i, jm, k), e));
  sum = __dadd_rn(sum, __dsub_rn(at(i, jp, k), e));
  sum = __dadd_rn(sum, __dsub_rn(at(i, j, km), e));
  sum = __dadd_rn(sum, __dsub_rn(at(i, j, kp), e));
  nxt[3 * (i + sx * (j + sy * k)) + a] = __dadd_rn(e, __dmul_rn(1.0 / 12.0, sum));
}

// field_mesh.hpp:46-59: every node with i == nx, j == ny or k == nz takes the
// value of its periodic image on the 0-planes, for E and B.
__global__ void __launch_bounds__(kStubThreads)
    mirror_seams_kernel(int nx, int ny, int nz, double* __restrict__ E, double* __restrict__ B) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long sx = nx + 1, sy = ny + 1;
  const long long nodes = sx * sy * (nz + 1);
  if (t >= nodes) return;
  const int i = static_cast<int>(t % sx);
  const int j = static_cast<int>((t / sx) % sy);
  const int k = static_cast<int>(t / (sx * sy));
  const int is = i == nx ? 0 : i, js = j == ny ? 0 : j, ks = k == nz ? 0 : k;
  if (is == i && js == j && ks == k) return;
  const long long src = is + sx * (js + sy * ks);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    E[3 * t + a] = E[3 * src + a];
    B[3 * t + a] = B[3 * src + a];
  }
}

}  // namespace

double* launch_field_stub(int nx, int ny, int nz, double* E, double* B, double* scratch,
                          int passes, cudaStream_t st) {
  if (passes <= 0) return E;  // the reference returns the input unchanged
  const long long nodes = static_cast<long long>(nx + 1) * (ny + 1) * (nz + 1);
  double* cur = E;
  double* nxt = scratch;
  for (int p = 0; p < passes; ++p) {
    const dim3 grid(grid_for(3 * nx, kStubThreads), ny, nz);
    field_stub_kernel<<<grid, kStubThreads, 0, st>>>(nx, ny, nz, cur, nxt);
    note_launch();
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
  mirror_seams_kernel<<<grid_for(nodes, kStubThreads), kStubThreads, 0, st>>>(nx, ny, nz, cur, B);
  note_launch();
  return cur;
}

}  // namespace b2m
