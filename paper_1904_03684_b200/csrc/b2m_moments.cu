// b2m_moments.cu — moment deposition on the GPU: the next stage after the
// mover on the reference's cycle.
//
// Reference: pic::deposit_moments (kernels.cpp:147-183).  Every particle
// scatters wq = ((q/V * wx) * wy) * wz onto the 8 corners of its cell
// (grid_cell_of, grid.hpp:64-82; corner c = di + 2dj + 4dk; the upper corners
// wrap onto node 0, nodes == cells, index i + nx*(j + ny*k), kernels.hpp:63-65):
//   rho += wq, j_a += wq*u_a, and with pressure p_ab += (wq*u_a)*u_b.
//
// The cell and the weights are computed exactly as the reference does
// (correctly rounded divisions, truncation, the same products), so every
// per-particle term is bit-identical; only the order of the sums differs (the
// reference adds in particle order; here terms are summed per cell in
// registers and shared memory before FP64 atomics add them to the mesh).  The
// result matches the reference to rounding of the sums (tests: 1e-12 of the
// mesh scale), like the reference's own multi-worker sums (runtime.cpp:256-
// 262 adds per-worker meshes).  A first kernel that gave every lane its own
// contiguous range and flushed a run at every change of cell degraded 4.5x
// with drift since the last sort; profiles/README.md has both.
#include "b2m_fused.cuh"
#include "b2m_internal.hpp"

namespace b2m {

namespace {

struct MomentPtrs {
  double* m[10];  // rho, jx, jy, jz, pxx, pxy, pxz, pyy, pyz, pzz
};

// A warp streams a contiguous chunk of the species 32 particles at a time
// (coalesced loads, one particle per lane, the next 32 prefetched into
// registers).
//  * The warp carries one cell: each lane sums, in registers, the terms of
//    its own particles in that cell.  Cell-sorted particles stay in one cell
//    for ~216 particles per species, so the common iteration is FP64
//    arithmetic only -- no shared memory, no atomics.
//  * When another cell's group among the 32 outnumbers the carried cell's
//    (the sorted order moved on, or drift), the carry is reduced across the
//    warp with a shuffle transpose (lane j ends with column j), added to the
//    mesh with one atomic per lane, and that group becomes the carry.
//  * Other particles (drifted out of the sorted order) are grouped by cell
//    (__match_any_sync): one alone in its cell adds its terms to the mesh
//    directly; a group writes its terms to shared-memory rows and lane j sums
//    column j over them before one atomic per column.
constexpr int kGroupThreads = 128;
#ifndef B2M_DMMA_MINB
#define B2M_DMMA_MINB 6  // blocks per SM of the DMMA deposit (<= 85 registers)
#endif
#ifndef B2M_DEP_WSORT
#define B2M_DEP_WSORT 0  // 1: sort windows of 128 particles by cell in the warp (measured slower)
#endif
#ifndef B2M_DEP_DMMA
#define B2M_DEP_DMMA 1  // FAST rho + J: the DMMA kernel (0: the register-carry kernel)
#endif
#ifndef B2M_DEP_DIRECT_MAX
#define B2M_DEP_DIRECT_MAX 1  // groups up to this size add their terms with direct atomics
#endif

template <int SET>
constexpr int group_row() { return (SET == 0 ? 32 : 48) + 1; }  // +1: conflict-free rows

template <int SET>
constexpr size_t group_smem() {
  return sizeof(double) * (kGroupThreads / 32) * 32 * group_row<SET>();
}

// v[0..H2-1] over the 32 lanes -> lane j holds sum over lanes of v[j mod H2]
// (H2 = 32: lane j gets column j; H2 = 16: lanes j and j+16 get column j%16)
template <int H2, bool EXACT, int N>
__device__ __forceinline__ double xreduce(double (&v)[N], int o, int lane) {
#pragma unroll
  for (int h = H2 / 2; h >= 1; h >>= 1) {
    const bool up = lane & h;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = up ? v[o + i] : v[o + i + h];
      const double keep = up ? v[o + i + h] : v[o + i];
      const double r = __shfl_xor_sync(0xffffffffu, send, h);
      v[o + i] = EXACT ? __dadd_rn(keep, r) : keep + r;
    }
  }
  double x = v[o];
  if (H2 == 16) {
    const double r = __shfl_xor_sync(0xffffffffu, x, 16);
    x = EXACT ? __dadd_rn(x, r) : x + r;
  }
  return x;
}

template <int SET, bool EXACT>
__global__ void __launch_bounds__(kGroupThreads, 3)
    deposit_group_kernel(const __grid_constant__ DevGrid g, const __grid_constant__ SpeciesLaunch sp,
                         double qv, const __grid_constant__ MomentPtrs M, unsigned long long span,
                         FaultWord* fault) {
  constexpr int NM = SET == 0 ? 4 : 6;
  constexpr int NV = NM * 8;
  constexpr int CPL = (NV + 31) / 32;  // columns per lane in a reduction
  constexpr int LD = group_row<SET>();
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(128) double sbuf[];
  const int lane = threadIdx.x & 31;
  double* const wbuf = sbuf + (threadIdx.x >> 5) * 32 * LD;
  double* const row = wbuf + lane * LD;
  const unsigned long long wid =
      (static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const unsigned long long lb = wid * span;
  if (lb >= sp.n) return;
  const unsigned long long le = lb + span < sp.n ? lb + span : sp.n;

  auto mul_ = [](double a, double b) { return EXACT ? __dmul_rn(a, b) : a * b; };
  auto add_ = [](double a, double b) { return EXACT ? __dadd_rn(a, b) : a + b; };
  auto sub_ = [](double a, double b) { return EXACT ? __dsub_rn(a, b) : a - b; };

  // add t to the mesh at column col (moment col/8, corner col%8) of cell (ci, cj, ck)
  auto red = [&](int col, int ci, int cj, int ck, double t) {
    const int mom = col >> 3, c = col & 7;
    const int ii = (c & 1) ? (ci + 1 == g.nx ? 0 : ci + 1) : ci;
    const int jj = (c & 2) ? (cj + 1 == g.ny ? 0 : cj + 1) : cj;
    const int kk = (c & 4) ? (ck + 1 == g.nz ? 0 : ck + 1) : ck;
    atomicAdd(M.m[SET * 4 + mom] + ii +
                  static_cast<long long>(g.nx) * (jj + static_cast<long long>(g.ny) * kk),
              t);
  };

  double acc[NV];  // this lane's sums for the carried cell
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = 0.0;
  long long ckey = -1;  // carried cell (warp-uniform); -1: none
  int cci = 0, ccj = 0, cck = 0;
  // reduce the carry across the warp into the mesh and clear it
  auto flush_carry = [&]() {
    const double c0 = xreduce<32, EXACT>(acc, 0, lane);
    red(lane, cci, ccj, cck, c0);
    if (NV > 32) {
      const double c1 = xreduce<16, EXACT>(acc, 32, lane);
      if (lane < 16) red(32 + lane, cci, ccj, cck, c1);
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = 0.0;
  };

  auto load = [&](unsigned long long p, double (&q)[6]) {
    if (p < le) {
      q[0] = sp.x[p]; q[1] = sp.y[p]; q[2] = sp.z[p];
      q[3] = sp.u[p]; q[4] = sp.v[p]; q[5] = sp.w[p];
    }
  };
  double nxt[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  load(lb + lane, nxt);

  for (unsigned long long base = lb; base < le; base += 32) {
    const unsigned long long p = base + lane;
    bool ok = p < le;
    const double px = nxt[0], py = nxt[1], pz = nxt[2], ux = nxt[3], uy = nxt[4], uz = nxt[5];
    load(p + 32, nxt);
    // grid.hpp:65-67: the reference throws DomainError
    if (ok && !(px >= 0.0 && px < g.lx && py >= 0.0 && py < g.ly && pz >= 0.0 && pz < g.lz)) {
      atomicMin(&fault->domain, fault_key(sp.species, sp.base + p));
      ok = false;
    }
    // grid.hpp:69-80, bit for bit
    const double sx = EXACT ? div_axis(px, g.dx, g.rdx) : px * g.rdx;
    const double sy = EXACT ? div_axis(py, g.dy, g.rdy) : py * g.rdy;
    const double sz = EXACT ? div_axis(pz, g.dz, g.rdz) : pz * g.rdz;
    int i = __double2int_rz(sx), j = __double2int_rz(sy), k = __double2int_rz(sz);
    if (i >= g.nx) i = g.nx - 1;
    if (j >= g.ny) j = g.ny - 1;
    if (k >= g.nz) k = g.nz - 1;
    const double fx = fmin(sub_(sx, static_cast<double>(i)), 1.0);
    const double fy = fmin(sub_(sy, static_cast<double>(j)), 1.0);
    const double fz = fmin(sub_(sz, static_cast<double>(k)), 1.0);
    const double wx[2] = {sub_(1.0, fx), fx};
    const double wy[2] = {sub_(1.0, fy), fy};
    const double wz[2] = {sub_(1.0, fz), fz};
    // the NV terms of this particle, column by column (kernels.cpp:168-181)
    auto terms = [&](auto&& f) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        // kernels.cpp:168: qv * wx * wy * wz, left to right
        const double wq = mul_(mul_(mul_(qv, wx[c & 1]), wy[(c >> 1) & 1]), wz[(c >> 2) & 1]);
        if (SET == 0) {
          f(c, wq);
          f(8 + c, mul_(wq, ux));
          f(16 + c, mul_(wq, uy));
          f(24 + c, mul_(wq, uz));
        } else {
          const double wu = mul_(wq, ux), wv = mul_(wq, uy), ww = mul_(wq, uz);
          f(c, mul_(wu, ux));
          f(8 + c, mul_(wu, uy));
          f(16 + c, mul_(wu, uz));
          f(24 + c, mul_(wv, uy));
          f(32 + c, mul_(wv, uz));
          f(40 + c, mul_(ww, uz));
        }
      }
    };
    const long long key =
        ok ? i + static_cast<long long>(g.nx) * (j + static_cast<long long>(g.ny) * k) : -1;
    const bool in_carry = ok && key == ckey;
    if (in_carry) terms([&](int v, double t) { acc[v] = add_(acc[v], t); });
    unsigned rest = __ballot_sync(FULL, ok && !in_carry);
    if (rest == 0) continue;  // the common case after a sort

    const unsigned grp = __match_any_sync(FULL, key);
    // the sorted order moved on (or drift): the largest other group takes
    // over the carry when it outnumbers the carried cell here; ties go to the
    // group of the last lane (the sorted order continues there)
    const unsigned score = (ok && !in_carry)
                               ? (static_cast<unsigned>(__popc(grp)) << 6) |
                                     (((grp >> 31) & 1u) << 5) | static_cast<unsigned>(lane)
                               : 0u;
    const unsigned best = __reduce_max_sync(FULL, score);
    const int ncarried = __popc(__ballot_sync(FULL, in_carry));
    if (static_cast<int>(best >> 6) >= (ncarried > 1 ? ncarried : 2) ||
        (ncarried == 0 && (best >> 6) >= 1 && ckey < 0)) {
      const int bl = best & 31;
      if (ckey >= 0) flush_carry();
      ckey = __shfl_sync(FULL, key, bl);
      cci = __shfl_sync(FULL, i, bl);
      ccj = __shfl_sync(FULL, j, bl);
      cck = __shfl_sync(FULL, k, bl);
      const unsigned took = __shfl_sync(FULL, grp, bl);
      if ((took >> lane) & 1) terms([&](int v, double t) { acc[v] = t; });
      rest &= ~took;
      if (rest == 0) continue;
    }
    const bool mine = (rest >> lane) & 1;
    // alone in its cell: straight to the mesh
    const bool single = mine && __popc(grp) <= B2M_DEP_DIRECT_MAX;
    if (single) terms([&](int v, double t) { red(v, i, j, k, t); });
    unsigned multi = rest & ~__ballot_sync(FULL, single);
    if (multi == 0) continue;
    if ((multi >> lane) & 1) terms([&](int v, double t) { row[v] = t; });
    __syncwarp();
    while (multi) {
      const int leader = __ffs(multi) - 1;
      const unsigned mem = __shfl_sync(FULL, grp, leader);
      multi &= ~mem;
      const int gi = __shfl_sync(FULL, i, leader), gj = __shfl_sync(FULL, j, leader),
                gk = __shfl_sync(FULL, k, leader);
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int col = lane + 32 * q;
        if (col < NV) {
          double a0 = 0.0, a1 = 0.0;  // two chains over the member rows
          unsigned b = mem;
          while (b) {
            a0 = add_(a0, wbuf[(__ffs(b) - 1) * LD + col]);
            b &= b - 1;
            if (b) {
              a1 = add_(a1, wbuf[(__ffs(b) - 1) * LD + col]);
              b &= b - 1;
            }
          }
          red(col, gi, gj, gk, add_(a0, a1));
        }
      }
    }
    __syncwarp();
  }
  if (ckey >= 0) flush_carry();
}

// FAST rho + J (set 0) with the fused mover's deposit machinery
// (b2m_fused.cuh): a warp streams its contiguous span 32 particles at a time
// (the next row prefetched into registers), stages the 8 corner weights and
// u, v, w per lane (3.2 KB per warp), and runs one FP64 DMMA pass per row --
// the carried cell's sums live in the 8x8 accumulator (2 registers per lane),
// the row's largest other cell rides in the other half and is flushed, strays
// add their terms with direct atomics.  ~70 registers instead of 166, so 8
// blocks (32 warps) per SM hide the loads that bound the register-carry
// kernel.
constexpr int kDmmaThreads = 128;
template <int SET>
__global__ void __launch_bounds__(kDmmaThreads, SET == 2 ? B2M_DMMA_MINB - 1 : B2M_DMMA_MINB)
    deposit_dmma_kernel(const __grid_constant__ DevGrid g, const __grid_constant__ SpeciesLaunch sp,
                        double qv, const __grid_constant__ MomentPtrs M,
                        unsigned long long span, FaultWord* fault) {
  __shared__ __align__(16) double sbuf[kDmmaThreads / 32][11 * kDepRow];
  __shared__ __align__(16) double wbuf[kDmmaThreads / 32][B2M_DEP_WSORT ? 6 : 1][4 * 32];
  const int lane = threadIdx.x & 31;
  double* const sw = sbuf[threadIdx.x >> 5];
  const unsigned long long wid =
      (static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const unsigned long long lb = wid * span;
  if (lb >= sp.n) return;
  const unsigned long long le = lb + span < sp.n ? lb + span : sp.n;
  DepCarry C, Pc;  // Pc: the pressure accumulator of the carried cell (SET 2)
  dep_reset(C);
  dep_reset(Pc);
  if (B2M_DEP_WSORT && SET == 0) {
    // Windows of 4 rows (128 particles): loaded together, sorted by cell in
    // the warp (bitonic network over (key << 8 | slot), 4 per lane), then
    // deposited row by row in cell order -- so particles that drifted out of
    // the sorted order meet their cell-mates of the window in one DMMA group
    // instead of taking a stray's 32 atomics.  An already sorted window (a
    // freshly sorted species) skips the network.
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int WR = 4;
    constexpr unsigned long long kInvalid = 0xffffffffull;
    double (*const win)[WR * 32] = wbuf[threadIdx.x >> 5];
    for (unsigned long long base = lb; base < le; base += WR * 32) {
      unsigned long long pk[WR];
#pragma unroll
      for (int r = 0; r < WR; ++r) {
        const unsigned long long p = base + 32 * r + lane;
        const int slot = 32 * r + lane;
        unsigned long long key = kInvalid;
        if (p < le) {
          const double px = sp.x[p], py = sp.y[p], pz = sp.z[p];
          win[0][slot] = px; win[1][slot] = py; win[2][slot] = pz;
          win[3][slot] = sp.u[p]; win[4][slot] = sp.v[p]; win[5][slot] = sp.w[p];
          if (px >= 0.0 && px < g.lx && py >= 0.0 && py < g.ly && pz >= 0.0 && pz < g.lz) {
            const int i = min(__double2int_rz(px * g.rdx), g.nx - 1);
            const int j = min(__double2int_rz(py * g.rdy), g.ny - 1);
            const int k = min(__double2int_rz(pz * g.rdz), g.nz - 1);
            // the cell sort's order (z fastest, b2m_kernels.cu cell_key), so a
            // freshly sorted window passes the check below
            key = static_cast<unsigned long long>(k) +
                  static_cast<unsigned long long>(g.nz) *
                      (static_cast<unsigned long long>(i) +
                       static_cast<unsigned long long>(g.nx) * static_cast<unsigned long long>(j));
          } else {
            atomicMin(&fault->domain, fault_key(sp.species, sp.base + p));
          }
        }
        pk[r] = (key << 8) | static_cast<unsigned long long>(slot);
      }
      // sorted already?  (position 32r + lane <= its successor)
      bool sorted = true;
#pragma unroll
      for (int r = 0; r < WR; ++r) {
        unsigned long long nx = __shfl_down_sync(FULL, pk[r], 1);
        const unsigned long long wrap = __shfl_sync(FULL, pk[r + 1 < WR ? r + 1 : r], 0);
        if (lane == 31) nx = r + 1 < WR ? wrap : ~0ull;
        sorted = sorted && (pk[r] >> 8) <= (nx >> 8);
      }
      if (!__all_sync(FULL, sorted)) {
#pragma unroll
        for (int k = 2; k <= WR * 32; k <<= 1) {
#pragma unroll
          for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
              const int rj = j >> 5;
#pragma unroll
              for (int r = 0; r < WR; ++r) {
                if (r & rj) continue;
                const bool asc = ((32 * r + lane) & k) == 0;
                const unsigned long long a = pk[r], b = pk[r | rj];
                if ((a > b) == asc) {
                  pk[r] = b;
                  pk[r | rj] = a;
                }
              }
            } else {
#pragma unroll
              for (int r = 0; r < WR; ++r) {
                const unsigned long long o = __shfl_xor_sync(FULL, pk[r], j);
                const bool asc = ((32 * r + lane) & k) == 0;
                const bool lower = (lane & j) == 0;
                pk[r] = (lower == asc) ? (pk[r] < o ? pk[r] : o) : (pk[r] < o ? o : pk[r]);
              }
            }
          }
        }
      }
#pragma unroll 1
      for (int r = 0; r < WR; ++r) {
        if (base + 32 * r >= le) break;
        const int slot = static_cast<int>(pk[r] & 0xff);
        const bool ok = (pk[r] >> 8) != kInvalid;
        sw[8 * kDepRow + lane] = win[3][slot];
        sw[9 * kDepRow + lane] = win[4][slot];
        sw[10 * kDepRow + lane] = win[5][slot];
        dep_row<kDepRow, true>(C, g, qv, M.m, sw, sw + 8 * kDepRow, win[0][slot], win[1][slot],
                               win[2][slot], ok, lane);
      }
      __syncwarp();  // the window is rewritten by the next one
    }
    dep_finish(C, g, M.m, lane);
    return;
  }
  auto load = [&](unsigned long long p, double (&q)[6]) {
    if (p < le) {
      q[0] = sp.x[p]; q[1] = sp.y[p]; q[2] = sp.z[p];
      q[3] = sp.u[p]; q[4] = sp.v[p]; q[5] = sp.w[p];
    }
  };
  double nxt[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  load(lb + lane, nxt);
  for (unsigned long long base = lb; base < le; base += 32) {
    const unsigned long long p = base + lane;
    bool ok = p < le;
    const double px = nxt[0], py = nxt[1], pz = nxt[2];
    sw[8 * kDepRow + lane] = nxt[3];
    sw[9 * kDepRow + lane] = nxt[4];
    sw[10 * kDepRow + lane] = nxt[5];
    load(p + 32, nxt);
    // grid.hpp:65-67: the reference throws DomainError
    if (ok && !(px >= 0.0 && px < g.lx && py >= 0.0 && py < g.ly && pz >= 0.0 && pz < g.lz)) {
      atomicMin(&fault->domain, fault_key(sp.species, sp.base + p));
      ok = false;
    }
    if (SET == 0)
      dep_row<kDepRow, true>(C, g, qv, M.m, sw, sw + 8 * kDepRow, px, py, pz, ok, lane);
    else if (SET == 1)
      dep_row_p(C, g, qv, M.m, sw, sw + 8 * kDepRow, kDepRow, px, py, pz, ok, lane);
    else
      dep_row_all(C, Pc, g, qv, M.m, sw, sw + 8 * kDepRow, px, py, pz, ok, lane);
  }
  if (SET == 0) {
    dep_finish(C, g, M.m, lane);
  } else if (C.key >= 0) {
    if (SET == 2) dep_flush_half(C.d0, C.d1, 0, C.ci, C.cj, C.ck, g, M.m, lane);
    dep_flush_p(SET == 2 ? Pc.d0 : C.d0, SET == 2 ? Pc.d1 : C.d1, C.ci, C.cj, C.ck, g, M.m, lane);
  }
}

template <int SET>
void launch_dmma(const DevGrid& g, const SpeciesLaunch& sp, double qv, const MomentPtrs& M,
                 FaultWord* fault, cudaStream_t st) {
  static const int per_sm = [] {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, deposit_dmma_kernel<SET>, kDmmaThreads, 0);
    cudaGetLastError();
    return b > 0 ? b : 1;
  }();
  const unsigned long long warps =
      static_cast<unsigned long long>(device_sms()) * per_sm * (kDmmaThreads / 32);
  unsigned long long span = (sp.n + warps - 1) / warps;
  span = (span + 31) / 32 * 32;
  const unsigned long long used = (sp.n + span - 1) / span;
  const int blocks = static_cast<int>((used + kDmmaThreads / 32 - 1) / (kDmmaThreads / 32));
  deposit_dmma_kernel<SET><<<blocks, kDmmaThreads, 0, st>>>(g, sp, qv, M, span, fault);
  note_launch();
}

template <int SET, bool EXACT>
void launch_group(const DevGrid& g, const SpeciesLaunch& sp, double qv, const MomentPtrs& M,
                  FaultWord* fault, cudaStream_t st) {
  constexpr size_t smem = group_smem<SET>();
  static const int per_sm = [] {
    cudaFuncSetAttribute(deposit_group_kernel<SET, EXACT>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, deposit_group_kernel<SET, EXACT>,
                                                  kGroupThreads, smem);
    cudaGetLastError();
    return b > 0 ? b : 1;
  }();
  const unsigned long long warps =
      static_cast<unsigned long long>(device_sms()) * per_sm * (kGroupThreads / 32);
  unsigned long long span = (sp.n + warps - 1) / warps;
  span = (span + 31) / 32 * 32;
  const unsigned long long used = (sp.n + span - 1) / span;
  const int blocks = static_cast<int>((used + kGroupThreads / 32 - 1) / (kGroupThreads / 32));
  deposit_group_kernel<SET, EXACT><<<blocks, kGroupThreads, smem, st>>>(g, sp, qv, M, span, fault);
  note_launch();
}

}  // namespace

void launch_deposit(const DevGrid& g, const SpeciesLaunch& sp, double qv, double* const* mesh,
                    bool pressure, bool exact, FaultWord* fault, cudaStream_t st) {
  if (sp.n == 0) return;
  MomentPtrs M{};
  for (int m = 0; m < (pressure ? 10 : 4); ++m) M.m[m] = mesh[m];
  if (!exact && B2M_DEP_DMMA) {
    // FAST: one pass for rho + J, or rho + J + pressure (SET 2: the particles
    // read once, locate / weights / groups shared)
    if (pressure) launch_dmma<2>(g, sp, qv, M, fault, st);
    else launch_dmma<0>(g, sp, qv, M, fault, st);
    return;
  }
  if (exact) launch_group<0, true>(g, sp, qv, M, fault, st);
  else launch_group<0, false>(g, sp, qv, M, fault, st);
  if (pressure) {
    if (exact) launch_group<1, true>(g, sp, qv, M, fault, st);
    else launch_group<1, false>(g, sp, qv, M, fault, st);
  }
}

}  // namespace b2m
