// b2m_moments.cu — moment deposition on the GPU: the next stage after the
// mover on the reference's cycle.
//
// Reference: pic::deposit_moments (kernels.cpp:147-183).  Every particle
// scatters wq = ((q/V * wx) * wy) * wz onto the 8 corners of its cell
// (grid_cell_of, grid.hpp:64-82; corner c = di + 2dj + 4dk; the upper corners
// wrap onto node 0, nodes == cells, index i + nx*(j + ny*k), kernels.hpp:63-65):
//   rho += wq, j_a += wq*u_a, and with pressure p_ab += (wq*u_a)*u_b.
//
// The cell and the weights are computed exactly as the reference does (IEEE
// divisions, truncation, the same products), so every per-particle term is
// bit-identical; only the order of the sums differs (the reference adds in
// particle order; here each lane first sums its run of particles in one cell
// in registers, then adds the run to the mesh with FP64 atomics).  The
// result matches the reference to rounding of the sums (tests: 1e-12 of the
// mesh scale), like the reference's own multi-worker sums (runtime.cpp:256-
// 262 adds per-worker meshes).
//
// Layout: every lane owns a contiguous range of the species (32 ranges per
// warp, side by side) and streams it 4 particles at a time with 256-bit
// loads (each a full 32-byte sector).  With cell-sorted particles a lane
// stays in one cell for a whole run (~216 particles per species in GEM), so
// it adds 8 corners x NM moments to the mesh once per run, and the 32 lanes
// of a warp work in 32 different cells -- no colliding atomics.
#include "b2m_internal.hpp"

namespace b2m {

namespace {

constexpr int kDepositThreads = 128;
constexpr int kDepositGroup = 4;  // particles per 256-bit load

struct MomentPtrs {
  double* m[10];  // rho, jx, jy, jz, pxx, pxy, pxz, pyy, pyz, pzz
};

__device__ __forceinline__ void load4(const double* p, double (&v)[4]) {
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
      : "l"(p));
}

// SET 0: rho, jx, jy, jz.  SET 1: the six pressure components.
// EXACT (STRICT contexts): the cell and weights with the reference's IEEE
// divisions, every per-particle term bit-identical.  Otherwise (FAST) the
// position is scaled by 1/d and the products may contract into FMAs: the
// terms change by an ulp and a particle exactly on a cell face may pick the
// neighbouring cell -- the deposit is continuous across faces, so the mesh
// still agrees to rounding.
template <int SET, bool EXACT>
__global__ void __launch_bounds__(kDepositThreads, 2)
    deposit_kernel(const __grid_constant__ DevGrid g, const __grid_constant__ SpeciesLaunch sp,
                   double qv, const __grid_constant__ MomentPtrs M, unsigned long long span,
                   FaultWord* fault) {
  constexpr int NM = SET == 0 ? 4 : 6;
  const double rdx = 1.0 / g.dx, rdy = 1.0 / g.dy, rdz = 1.0 / g.dz;
  const unsigned long long t =
      static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const unsigned long long lb = t * span;  // this lane's range [lb, le)
  if (lb >= sp.n) return;
  const unsigned long long le = lb + span < sp.n ? lb + span : sp.n;

  double acc[NM][8];
  int ai = -1, aj = 0, ak = 0;  // cell of the run being summed (ai < 0: none)
  auto flush = [&]() {  // add the run to the mesh
    const int i1 = ai + 1 == g.nx ? 0 : ai + 1;
    const int j1 = aj + 1 == g.ny ? 0 : aj + 1;
    const int k1 = ak + 1 == g.nz ? 0 : ak + 1;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int ii = (c & 1) ? i1 : ai, jj = (c & 2) ? j1 : aj, kk = (c & 4) ? k1 : ak;
      const long long idx =
          ii + static_cast<long long>(g.nx) * (jj + static_cast<long long>(g.ny) * kk);
#pragma unroll
      for (int m = 0; m < NM; ++m) atomicAdd(M.m[SET * 4 + m] + idx, acc[m][c]);
    }
  };

  // EXACT: every product/sum rounded on its own, as the reference (no FMA)
  auto mul_ = [](double a, double b) { return EXACT ? __dmul_rn(a, b) : a * b; };
  auto add_ = [](double a, double b) { return EXACT ? __dadd_rn(a, b) : a + b; };
  auto sub_ = [](double a, double b) { return EXACT ? __dsub_rn(a, b) : a - b; };
  auto particle = [&](double px, double py, double pz, double ux, double uy, double uz,
                      unsigned long long p) {
    // grid.hpp:65-67: the reference throws DomainError
    if (!(px >= 0.0 && px < g.lx && py >= 0.0 && py < g.ly && pz >= 0.0 && pz < g.lz)) {
      atomicMin(&fault->domain, fault_key(sp.species, sp.base + p));
      return;
    }
    // grid.hpp:69-80, bit for bit
    const double sx = EXACT ? __ddiv_rn(px, g.dx) : px * rdx;
    const double sy = EXACT ? __ddiv_rn(py, g.dy) : py * rdy;
    const double sz = EXACT ? __ddiv_rn(pz, g.dz) : pz * rdz;
    int i = __double2int_rz(sx), j = __double2int_rz(sy), k = __double2int_rz(sz);
    if (i >= g.nx) i = g.nx - 1;
    if (j >= g.ny) j = g.ny - 1;
    if (k >= g.nz) k = g.nz - 1;
    const double fx = fmin(sub_(sx, static_cast<double>(i)), 1.0);
    const double fy = fmin(sub_(sy, static_cast<double>(j)), 1.0);
    const double fz = fmin(sub_(sz, static_cast<double>(k)), 1.0);
    if (i != ai || j != aj || k != ak) {
      if (ai >= 0) flush();
      ai = i; aj = j; ak = k;
#pragma unroll
      for (int m = 0; m < NM; ++m)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[m][c] = 0.0;
    }
    const double wx[2] = {sub_(1.0, fx), fx};
    const double wy[2] = {sub_(1.0, fy), fy};
    const double wz[2] = {sub_(1.0, fz), fz};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      // kernels.cpp:168: qv * wx * wy * wz, left to right
      const double wq = mul_(mul_(mul_(qv, wx[c & 1]), wy[(c >> 1) & 1]),
                                  wz[(c >> 2) & 1]);
      if (SET == 0) {
        acc[0][c] = add_(acc[0][c], wq);
        acc[1][c] = add_(acc[1][c], mul_(wq, ux));
        acc[2][c] = add_(acc[2][c], mul_(wq, uy));
        acc[3][c] = add_(acc[3][c], mul_(wq, uz));
      } else {
        const double wu = mul_(wq, ux), wv = mul_(wq, uy), ww = mul_(wq, uz);
        acc[0][c] = add_(acc[0][c], mul_(wu, ux));
        acc[1][c] = add_(acc[1][c], mul_(wu, uy));
        acc[2][c] = add_(acc[2][c], mul_(wu, uz));
        acc[3][c] = add_(acc[3][c], mul_(wv, uy));
        acc[4][c] = add_(acc[4][c], mul_(wv, uz));
        acc[5][c] = add_(acc[5][c], mul_(ww, uz));
      }
    }
  };

  unsigned long long p = lb;
  // 256-bit groups (the species arrays are 256-byte aligned and span is a
  // multiple of the group)
  for (; p + kDepositGroup <= le; p += kDepositGroup) {
    double X[4], Y[4], Z[4], U[4], V[4], W[4];
    load4(sp.x + p, X); load4(sp.y + p, Y); load4(sp.z + p, Z);
    load4(sp.u + p, U); load4(sp.v + p, V); load4(sp.w + p, W);
#pragma unroll
    for (int q = 0; q < kDepositGroup; ++q) particle(X[q], Y[q], Z[q], U[q], V[q], W[q], p + q);
  }
  for (; p < le; ++p) particle(sp.x[p], sp.y[p], sp.z[p], sp.u[p], sp.v[p], sp.w[p], p);
  if (ai >= 0) flush();
}

}  // namespace

void launch_deposit(const DevGrid& g, const SpeciesLaunch& sp, double qv, double* const* mesh,
                    bool pressure, bool exact, FaultWord* fault, cudaStream_t st) {
  if (sp.n == 0) return;
  const int sms = device_sms();
  // enough lanes to fill the GPU, each a contiguous range of whole groups
  const unsigned long long lanes = static_cast<unsigned long long>(sms) * 12 * 32;
  unsigned long long span = (sp.n + lanes - 1) / lanes;
  span = (span + kDepositGroup - 1) / kDepositGroup * kDepositGroup;
  if (span < 64) span = 64;
  const unsigned long long used = (sp.n + span - 1) / span;
  const int blocks = static_cast<int>((used + kDepositThreads - 1) / kDepositThreads);
  MomentPtrs M{};
  for (int m = 0; m < (pressure ? 10 : 4); ++m) M.m[m] = mesh[m];
  if (exact)
    deposit_kernel<0, true><<<blocks, kDepositThreads, 0, st>>>(g, sp, qv, M, span, fault);
  else
    deposit_kernel<0, false><<<blocks, kDepositThreads, 0, st>>>(g, sp, qv, M, span, fault);
  note_launch();
  if (pressure) {
    if (exact)
      deposit_kernel<1, true><<<blocks, kDepositThreads, 0, st>>>(g, sp, qv, M, span, fault);
    else
      deposit_kernel<1, false><<<blocks, kDepositThreads, 0, st>>>(g, sp, qv, M, span, fault);
    note_launch();
  }
}

}  // namespace b2m
