// b2m_tile.cuh — device code of the production movers (FAST and STRICT).
//
// Both modes run the same warp-tile pipeline (b2m_kernels.cu,
// warp_tile_kernel): each warp streams tiles of 32*PPT particles -- all six
// SoA arrays in ONE 2-D tensor-map TMA box -- through its own shared-memory
// ring, and every lane moves PPT particles one after the other with the
// field of its current cell held in registers.
//
// Why this shape (profiles/README.md has the measured log): delivering a
// cell's 48 field values to a lane costs L1->register bandwidth (128 B/clk
// per SM) whether or not lanes share addresses, so the values must be reused
// from registers.  Keeping them across the 3 predictor rounds of a particle
// and across the lane's next particles (mostly in the same cell) does that
// without depending on neighbouring particles sharing a cell, so performance
// does not decay as particles drift out of cell order.
#pragma once

#include <cuda.h>

#include "b2m_mover.cuh"

namespace b2m {

// ---- tunables (tools/build_variants.sh sweeps them) ------------------------
#ifndef B2M_TPB
#define B2M_TPB 128            // threads per block of the warp-tile kernel
#endif
#ifndef B2M_WARP_STAGES
#define B2M_WARP_STAGES 2      // TMA ring depth per warp (2: larger L1, profiles/README.md)
#endif
#ifndef B2M_FAST_PPT
#define B2M_FAST_PPT 4         // particles per lane per tile (sequential)
#endif
#ifndef B2M_FAST_MINBLOCKS
#define B2M_FAST_MINBLOCKS 3   // __launch_bounds__ residency (-> 168 registers)
#endif
constexpr int kWarpThreads = B2M_TPB;
constexpr int kWarpStages = B2M_WARP_STAGES;
constexpr int kMaxTileSpans = 8;

// ---------------------------------------------------------------------------
// TMA / mbarrier primitives (PTX ISA 8.x, sm_90+; SASS UTMALDG / UTMASTG / SYNCS)
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Non-blocking probe of an mbarrier phase (true: the phase completed).
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// L2 eviction priorities: the particle stream (2.9 GB per cycle at C2) is
// evict-first so it does not sweep the 50 MB coefficient table, which is
// evict-last (createpolicy, PTX ISA 7.4+).
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1,
                                             const void* smem_src, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(smem_u32(smem_src)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void tma_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void tma_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// ---------------------------------------------------------------------------
// launch parameters
// ---------------------------------------------------------------------------

// FAST: the per-launch scalars every span of the launch shares (the launcher
// splits a batch whose spans differ), so the hot loop reads them as
// constant-bank operands instead of per-species registers.
struct FastUniform {
  double dt;          // MoverParams::dt
  double dc[3];       // 0.5*dt/d per axis: cell-unit predictor step
  int rounds;         // pc_iterations
};

struct TileField {
  FastGrid fg;
  DevGrid dg;
  const double* nodes;   // STRICT: per-cell corner node values (strict_nodes_kernel)
  FastUniform U;
  const int* zvar;       // FAST: device flag, 0 = field z-invariant (null: general kernel only)
  double* mom[4];        // fused deposit (b2m_fused.cuh): rho, jx, jy, jz mesh arrays
};

// FAST launch: per span a 2-D tensor map over the species' [6][stride]
// block (dims {col0 + n, 6}), so one TMA box moves all six arrays of a tile
// and the hardware clips partial tiles.
struct alignas(64) TensorSpans {
  CUtensorMap tmap[kMaxTileSpans];
  SpeciesLaunch sp[kMaxTileSpans];
  unsigned long long tile_start[kMaxTileSpans + 1];
  uint8_t* flags[kMaxTileSpans];  // migration: per-particle destination flag (or null)
  unsigned long long* tcnt[kMaxTileSpans];  // migration: per-tile (next << 32 | prev) counts
  int n;
};
// ---------------------------------------------------------------------------
// FAST: FMA arithmetic, per-cell polynomial gather, integer-only control flow
// ---------------------------------------------------------------------------
//
// Every range check is an unsigned compare of the IEEE bit pattern (for
// x >= +0 the bit patterns order like the values; negatives, -0, NaN and Inf
// all land above any positive bound), cell indices are clamped so a NaN can
// never address memory, and a sticky per-particle flag records every event
// the reference would have thrown on (x0 outside [0,l), a non-finite
// predictor position, a non-finite result), so faults name the same
// particles.

__device__ __forceinline__ unsigned long long dbits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}

constexpr unsigned long long kSign = 0x8000000000000000ull;
constexpr unsigned long long kAbs = 0x7fffffffffffffffull;
constexpr unsigned long long kExp = 0x7ff0000000000000ull;

// x in [0, l) exactly as `x >= 0.0 && x < l` (accepts -0.0, rejects NaN)
__device__ __forceinline__ bool in_range(double x, unsigned long long lbits) {
  const unsigned long long b = dbits(x);
  return b < lbits || b == kSign;
}

__device__ __forceinline__ bool finite_bits(double x) { return (dbits(x) & kExp) != kExp; }

// Cell-unit periodic fold of the predictor into [0, n).  The in-range test is
// one unsigned compare; everything else (c < 0 incl. -0, c >= n, NaN, Inf) is
// the rare slow path, which also flags non-finite values.
__device__ __forceinline__ double fold_fast(double c, double n, unsigned long long nbits,
                                            double rn, unsigned& bad) {
  if (dbits(c) >= nbits) {
    if (!finite_bits(c)) bad = 1u;
    c = fma(-n, floor(c * rn), c);
    if (c >= n) c -= n;
    if (c < 0.0) c += n;
    if (!(c < n)) c = 0.0;
  }
  return c;
}

// Bit-exact wrap_len(v, l) (grid.hpp:45-50) with integer compares: the
// thresholds of WrapAxis give floor(RN(v/l)) without a division.
__device__ __forceinline__ double wrap_exact_bits(double v, const WrapAxis& a,
                                                  unsigned long long hi0b,
                                                  unsigned long long hi1b,
                                                  unsigned long long lomb) {
  const unsigned long long b = dbits(v);
  double w;
  if (b <= hi0b) {
    w = v;                                  // q = 0 (v in [+0, hi0])
  } else if (b <= hi1b) {
    w = __dsub_rn(v, a.l);                  // q = 1
  } else if (b > kSign && (b & kAbs) <= lomb) {
    w = __dadd_rn(v, a.l);                  // q = -1 (v in [lom1, 0))
  } else {
    const double q = floor(__ddiv_rn(v, a.l));  // -0, far out of range, NaN
    w = __dsub_rn(v, __dmul_rn(a.l, q));
  }
  // fix-ups: if (w >= l) w -= l;  if (w < 0.0) w = 0.0;
  const unsigned long long wb = dbits(w);
  if (wb < kSign && wb >= dbits(a.l)) w = __dsub_rn(w, a.l);
  if (dbits(w) > kSign) w = 0.0;
  return w;
}

// One component's 8 coefficients = two 256-bit loads (LDG.E.256 on sm_100a).
struct Coef8 {
  double p0, q0, p1, q1, p2, q2, p3, q3;
};

// One component's 8 coefficients: two 256-bit loads (LDG.E.256 on sm_100a),
// L2 evict-last so the particle stream does not sweep the table.
__device__ __forceinline__ Coef8 load_coef8(const double2* c) {
  Coef8 k;
  const uint64_t pol = policy_evict_last();
  asm("ld.global.nc.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
      : "=d"(k.p0), "=d"(k.q0), "=d"(k.p1), "=d"(k.q1)
      : "l"(c), "l"(pol));
  asm("ld.global.nc.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
      : "=d"(k.p2), "=d"(k.q2), "=d"(k.p3), "=d"(k.q3)
      : "l"(c + 2), "l"(pol));
  return k;
}

__device__ __forceinline__ double poly8(const Coef8& k, double fx, double fy, double fz) {
  return fma(fx, fma(fy, fma(fz, k.q3, k.p3), fma(fz, k.q2, k.p2)),
             fma(fy, fma(fz, k.q1, k.p1), fma(fz, k.q0, k.p0)));
}

// Everything the hot loop needs, hoisted into registers once per tile.
struct FastConst {
  double rdx, rdy, rdz;
  double nxd, nyd, nzd;
  double rnx, rny, rnz;
  unsigned long long nxb, nyb, nzb;       // bits of nxd, nyd, nzd
  unsigned long long lxb, lyb, lzb;       // bits of lx, ly, lz
  int nx1, ny1, nz1;                      // n - 1
  int nx, nxny;
  double dt, dcx, dcy, dcz;               // dcx = 0.5*dt/dx
  int rounds;
};

__device__ __forceinline__ FastConst make_const(const FastGrid& g, const SpeciesLaunch& sp) {
  FastConst k;
  k.rdx = g.rdx; k.rdy = g.rdy; k.rdz = g.rdz;
  k.nxd = g.nxd; k.nyd = g.nyd; k.nzd = g.nzd;
  k.rnx = g.rnx; k.rny = g.rny; k.rnz = g.rnz;
  k.nxb = dbits(g.nxd); k.nyb = dbits(g.nyd); k.nzb = dbits(g.nzd);
  k.lxb = dbits(g.lx); k.lyb = dbits(g.ly); k.lzb = dbits(g.lz);
  k.nx1 = g.nx - 1; k.ny1 = g.ny - 1; k.nz1 = g.nz - 1;
  k.nx = g.nx; k.nxny = g.nx * g.ny;
  k.dt = sp.dt;
  k.dcx = sp.dto2_cell[0]; k.dcy = sp.dto2_cell[1]; k.dcz = sp.dto2_cell[2];
  k.rounds = sp.rounds;
  return k;
}

// Cell of a folded cell-unit position and the fractions within it.  Indices
// are clamped into the grid (a NaN position -- already flagged -- reads a
// valid cell and the particle is discarded at the end).
__device__ __forceinline__ int locate_fast(const FastConst& k, double tx, double ty, double tz,
                                           double& fx, double& fy, double& fz) {
  const int i = max(min(__double2int_rz(tx), k.nx1), 0);
  const int j = max(min(__double2int_rz(ty), k.ny1), 0);
  const int m = max(min(__double2int_rz(tz), k.nz1), 0);
  fx = tx - static_cast<double>(i);
  fy = ty - static_cast<double>(j);
  fz = tz - static_cast<double>(m);
  return i + k.nx * j + k.nxny * m;
}

// Implicit velocity (kernels.cpp:83-90), FMA form, from the gathered
// F = (beta*E, beta*B) (the cell table is pre-scaled): vt = v0 + beta*E,
// W = beta*B, vbar = (vt + vt x W + (vt.W) W) / (1 + |W|^2).  The reciprocal
// is the MUFU.RCP64H seed (~2^-23) refined by one third-order step (~2^-66).
__device__ __forceinline__ void implicit_v(double u0, double v0, double w0, const double* F,
                                           double& bx, double& by, double& bz) {
  const double ox = F[3], oy = F[4], oz = F[5];
  const double vtx = u0 + F[0];
  const double vty = v0 + F[1];
  const double vtz = w0 + F[2];
  const double den = 1.0 + fma(oz, oz, fma(oy, oy, ox * ox));
  double rc;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(den));
  const double e = fma(-den, rc, 1.0);
  rc = fma(rc, fma(e, e, e), rc);  // rc * (1 + e + e^2)
  const double vdot = fma(vtz, oz, fma(vty, oy, vtx * ox));
  bx = fma(vdot, ox, fma(vty, oz, fma(-vtz, oy, vtx))) * rc;
  by = fma(vdot, oy, fma(vtz, ox, fma(-vtx, oz, vty))) * rc;
  bz = fma(vdot, oz, fma(vtx, oy, fma(-vty, ox, vtz))) * rc;
}

// Fold of all three predictor coordinates at once: one combined (integer)
// range test, the slow path only for the rare lane that crossed a boundary.
__device__ __forceinline__ void fold3(double& tx, double& ty, double& tz, const FastConst& k,
                                      unsigned& bad) {
  if ((dbits(tx) >= k.nxb) | (dbits(ty) >= k.nyb) | (dbits(tz) >= k.nzb)) {
    tx = fold_fast(tx, k.nxd, k.nxb, k.rnx, bad);
    ty = fold_fast(ty, k.nyd, k.nyb, k.rny, bad);
    tz = fold_fast(tz, k.nzd, k.nzb, k.rnz, bad);
  }
}

// One FAST particle of a staged tile (kernels.cpp:52-104 in FMA form).
// buf[a][p] holds input a (x,y,z,u,v,w) of particle p and receives its result
// when it finishes clean; returns 1 for a particle to report as faulted.
// (K, kcell) is the lane's register cell cache, carried across particles;
// ROUNDS > 0 unrolls that many predictor rounds.  The cache is reloaded only
// when the predictor moves to another cell (~2 % of rounds in GEM), in a
// branch that contains loads only, so the evaluation code stays warp-uniform.
template <int TILE, int ROUNDS = 0>
__device__ __forceinline__ unsigned fast_tile_thread_p1(const FastGrid& g,
                                                        const double2* __restrict__ cells,
                                                        const FastConst& k, double (*buf)[TILE],
                                                        int p, int cnt, Coef8 (&K)[6],
                                                        int& kcell) {
  const double x0 = buf[0][p], y0 = buf[1][p], z0 = buf[2][p];
  const double u0 = buf[3][p], v0 = buf[4][p], w0 = buf[5][p];
  const bool inside = (p < cnt) && in_range(x0, k.lxb) && in_range(y0, k.lyb) && in_range(z0, k.lzb);
  unsigned bad = inside ? 0u : 1u;
  const double cx0 = inside ? x0 * k.rdx : 0.0;
  const double cy0 = inside ? y0 * k.rdy : 0.0;
  const double cz0 = inside ? z0 * k.rdz : 0.0;
  double fx, fy, fz;
  int cell = locate_fast(k, cx0, cy0, cz0, fx, fy, fz);
  double bx = u0, by = v0, bz = w0;
  const int rounds = ROUNDS > 0 ? ROUNDS : k.rounds;
#pragma unroll
  for (int r = 0; r < rounds; ++r) {
    if (cell != kcell) {  // rare: the predictor left the cached cell
      const double2* c = cells + static_cast<long long>(cell) * 24;
#pragma unroll
      for (int q = 0; q < 6; ++q) K[q] = load_coef8(c + 4 * q);
      kcell = cell;
    }
    double F[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) F[q] = poly8(K[q], fx, fy, fz);
    implicit_v(u0, v0, w0, F, bx, by, bz);
    if (r + 1 < rounds) {
      double tx = fma(bx, k.dcx, cx0);
      double ty = fma(by, k.dcy, cy0);
      double tz = fma(bz, k.dcz, cz0);
      fold3(tx, ty, tz, k, bad);
      cell = locate_fast(k, tx, ty, tz, fx, fy, fz);
    }
  }
  // kernels.cpp:95-99
  double x1 = fma(bx, k.dt, x0);
  double y1 = fma(by, k.dt, y0);
  double z1 = fma(bz, k.dt, z0);
  if ((dbits(x1) > dbits(g.ax.hi0)) | (dbits(y1) > dbits(g.ay.hi0)) |
      (dbits(z1) > dbits(g.az.hi0))) {
    x1 = wrap_exact_bits(x1, g.ax, dbits(g.ax.hi0), dbits(g.ax.hi1), dbits(g.ax.lom1) & kAbs);
    y1 = wrap_exact_bits(y1, g.ay, dbits(g.ay.hi0), dbits(g.ay.hi1), dbits(g.ay.lom1) & kAbs);
    z1 = wrap_exact_bits(z1, g.az, dbits(g.az.hi0), dbits(g.az.hi1), dbits(g.az.lom1) & kAbs);
  }
  const double u1 = fma(2.0, bx, -u0);
  const double v1 = fma(2.0, by, -v0);
  const double w1 = fma(2.0, bz, -w0);
  const bool fin = finite_bits(x1) && finite_bits(y1) && finite_bits(z1) && finite_bits(u1) &&
                   finite_bits(v1) && finite_bits(w1);
  if (bad == 0u && fin) {
    buf[0][p] = x1; buf[1][p] = y1; buf[2][p] = z1;
    buf[3][p] = u1; buf[4][p] = v1; buf[5][p] = w1;
    return 0u;
  }
  return p < cnt ? 1u : 0u;
}
// ---------------------------------------------------------------------------
// FAST v2: fractions relative to the cached cell
// ---------------------------------------------------------------------------
//
// The lane's cache also holds its cell's integer corner (ci, cj, ck) as
// doubles.  A particle's fractions are taken relative to that corner --
// f0 = x0/d - c at the start, f = f0 + vbar*dt/(2d) for a predictor -- and
// when all three lie in [+0, 1) (one integer compare of the high word each)
// the position is inside the cached cell: no truncation, no conversions, no
// periodic fold, no reload.  Only a lane that left the cell (a few % of
// rounds) takes the slow path: fold, locate, reload.  The trilinear field is
// continuous across faces and seams, so which of two touching cells a
// boundary position is evaluated in only changes rounding.

#ifndef B2M_V2_R1_LOCATE
#define B2M_V2_R1_LOCATE 1  // every particle's start is located (no frame test): 2.15 -> 2.12 ms
#endif

// f in [+0, 1): the high word of +0..1-ulp is below that of 1.0; negatives
// (sign bit), -0, NaN and everything >= 1 are not
__device__ __forceinline__ bool in_unit(double f) {
  return static_cast<unsigned>(__double2hiint(f)) < 0x3ff00000u;
}

// x in [+0, l): the fast-path form of in_range (-0 takes the slow path)
__device__ __forceinline__ bool below_bits(double x, unsigned long long lbits) {
  return dbits(x) < lbits;
}

// a shared-memory load the compiler cannot merge with an earlier one (so the
// value need not stay live in a register in between)
__device__ __forceinline__ double lds_f64(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(p)));
  return v;
}

// High word of a double through an opaque move, so that exponent tests stay
// integer ALU work (the compiler turns a visible bit test into DSETP, FP64 pipe)
__device__ __forceinline__ unsigned hi_word(double x) {
  unsigned lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(x));
  return hi;
}

// all three finite: no exponent field all ones
__device__ __forceinline__ bool finite3(double a, double b, double c) {
  constexpr unsigned kE = 0x7ff00000u;
  const unsigned m = max(max(hi_word(a) & kE, hi_word(b) & kE), hi_word(c) & kE);
  return m != kE;
}

#ifndef B2M_3D_PRED_RELOAD
#define B2M_3D_PRED_RELOAD 1    // the general kernel's cell reload as predicated loads (2.515 -> 2.46 ms; not in the fused kernel: spills)
#endif

struct FastCell {
  Coef8 K[6];
  double ci, cj, ck;  // the cached cell's corner in cell units
  int cell;
};

__device__ __forceinline__ void fast_cell_reset(FastCell& C) {
  C.cell = -1;
  C.ci = C.cj = C.ck = -4.0;  // no fraction relative to it is in [0, 1)
}

// Locate a folded cell-unit position (indices clamped: a flagged NaN reads a
// valid cell), load its coefficients when it is not the cached cell, and
// return the fractions relative to it.
template <bool PRED = false>
__device__ __forceinline__ void fast_enter(const FastGrid& g, const double2* __restrict__ cells,
                                           FastCell& C, double tx, double ty, double tz,
                                           double& fx, double& fy, double& fz) {
  const int i = max(min(__double2int_rz(tx), g.nx - 1), 0);
  const int j = max(min(__double2int_rz(ty), g.ny - 1), 0);
  const int m = max(min(__double2int_rz(tz), g.nz - 1), 0);
  const double di = static_cast<double>(i), dj = static_cast<double>(j),
               dk = static_cast<double>(m);
  fx = tx - di;
  fy = ty - dj;
  fz = tz - dk;
  const int cell = i + g.nx * (j + g.ny * m);
  if (PRED) {
    const double2* c = cells + static_cast<long long>(cell) * 24;
    const uint64_t pol = policy_evict_last();
    const int diff = cell != C.cell;
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %5, 0;\n\t"
          "@p ld.global.nc.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %6;\n\t}"
          : "+d"(C.K[q].p0), "+d"(C.K[q].q0), "+d"(C.K[q].p1), "+d"(C.K[q].q1)
          : "l"(c + 4 * q), "r"(diff), "l"(pol));
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %5, 0;\n\t"
          "@p ld.global.nc.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %6;\n\t}"
          : "+d"(C.K[q].p2), "+d"(C.K[q].q2), "+d"(C.K[q].p3), "+d"(C.K[q].q3)
          : "l"(c + 4 * q + 2), "r"(diff), "l"(pol));
    }
    C.cell = cell;
  } else if (cell != C.cell) {
    const double2* c = cells + static_cast<long long>(cell) * 24;
#pragma unroll
    for (int q = 0; q < 6; ++q) C.K[q] = load_coef8(c + 4 * q);
    C.cell = cell;
  }
  C.ci = di;
  C.cj = dj;
  C.ck = dk;
}

// Implicit velocity (kernels.cpp:83-90) up to its last product: returns the
// numerator (vt + vt x W + (vt.W) W) and rc = 1/(1 + |W|^2), vbar = num*rc.
__device__ __forceinline__ void implicit_num(double u0, double v0, double w0, const double* F,
                                             double& nx, double& ny, double& nz, double& rc) {
  const double ox = F[3], oy = F[4], oz = F[5];
  const double vtx = u0 + F[0];
  const double vty = v0 + F[1];
  const double vtz = w0 + F[2];
  const double den = fma(oz, oz, fma(oy, oy, fma(ox, ox, 1.0)));
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
  const double e = fma(-den, r, 1.0);
  rc = fma(r, fma(e, e, e), r);  // r * (1 + e + e^2)
  const double vdot = fma(vtz, oz, fma(vty, oy, vtx * ox));
  nx = fma(vdot, ox, fma(vty, oz, fma(-vtz, oy, vtx)));
  ny = fma(vdot, oy, fma(vtz, ox, fma(-vtx, oz, vty)));
  nz = fma(vdot, oz, fma(vtx, oy, fma(-vty, ox, vtz)));
}

// One FAST particle (kernels.cpp:52-104 in FMA form).  buf[a][p] holds input
// a of particle p and receives its result when it finishes clean; returns 1
// for a particle to report as faulted.
template <int TILE, int ROUNDS, bool PRED = false>
__device__ __forceinline__ unsigned fast_particle_v2(const FastGrid& g, const FastUniform& U,
                                                     const double2* __restrict__ cells,
                                                     double (*buf)[TILE], int p, int cnt,
                                                     FastCell& C) {
  const double x0 = buf[0][p], y0 = buf[1][p], z0 = buf[2][p];
  const double u0 = buf[3][p], v0 = buf[4][p], w0 = buf[5][p];
  double fx0, fy0, fz0;
  unsigned bad = 0u;
  {
    const double cx = x0 * g.rdx, cy = y0 * g.rdy, cz = z0 * g.rdz;
    fx0 = cx - C.ci; fy0 = cy - C.cj; fz0 = cz - C.ck;
  if (B2M_V2_R1_LOCATE || !((p < cnt) & below_bits(x0, dbits(g.lx)) & below_bits(y0, dbits(g.ly)) &
        below_bits(z0, dbits(g.lz)) & in_unit(fx0) & in_unit(fy0) & in_unit(fz0))) {
    // another cell, or a position the reference rejects (outside [0, l))
    const bool inside = (p < cnt) && in_range(x0, dbits(g.lx)) && in_range(y0, dbits(g.ly)) &&
                        in_range(z0, dbits(g.lz));
    bad = inside ? 0u : 1u;
    fast_enter<PRED>(g, cells, C, inside ? cx : 0.0, inside ? cy : 0.0, inside ? cz : 0.0, fx0, fy0,
               fz0);
  }
  }
  double fx = fx0, fy = fy0, fz = fz0;
  double nx, ny, nz, rc;
  const int rounds = ROUNDS > 0 ? ROUNDS : U.rounds;
#pragma unroll
  for (int r = 0; r < rounds; ++r) {
    double F[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) F[q] = poly8(C.K[q], fx, fy, fz);
    implicit_num(u0, v0, w0, F, nx, ny, nz, rc);
    if (r + 1 < rounds) {
      // predictor x0 + vbar*dt/2 in the cached cell's frame (kernels.cpp:92)
      fx = fma(nx * U.dc[0], rc, fx0);
      fy = fma(ny * U.dc[1], rc, fy0);
      fz = fma(nz * U.dc[2], rc, fz0);
      if (!(in_unit(fx) & in_unit(fy) & in_unit(fz))) {
        // left the cell: fold the absolute cell-unit position, locate, reload
        const double bx = nx * rc, by = ny * rc, bz = nz * rc;
        // (x0 re-read from the tile rather than kept live across the rounds)
        const double cx = lds_f64(&buf[0][p]) * g.rdx, cy = lds_f64(&buf[1][p]) * g.rdy,
                     cz = lds_f64(&buf[2][p]) * g.rdz;
        double tx = fma(bx, U.dc[0], cx), ty = fma(by, U.dc[1], cy), tz = fma(bz, U.dc[2], cz);
        if ((dbits(tx) >= dbits(g.nxd)) | (dbits(ty) >= dbits(g.nyd)) |
            (dbits(tz) >= dbits(g.nzd))) {
          tx = fold_fast(tx, g.nxd, dbits(g.nxd), g.rnx, bad);
          ty = fold_fast(ty, g.nyd, dbits(g.nyd), g.rny, bad);
          tz = fold_fast(tz, g.nzd, dbits(g.nzd), g.rnz, bad);
        }
        fast_enter<PRED>(g, cells, C, tx, ty, tz, fx, fy, fz);
        // the start position in the new cell's (folded) frame
        fx0 = fma(-bx, U.dc[0], fx);
        fy0 = fma(-by, U.dc[1], fy);
        fz0 = fma(-bz, U.dc[2], fz);
      }
    }
  }
  // kernels.cpp:95-99
  const double bx = nx * rc, by = ny * rc, bz = nz * rc;
  double x1 = fma(bx, U.dt, lds_f64(&buf[0][p]));
  double y1 = fma(by, U.dt, lds_f64(&buf[1][p]));
  double z1 = fma(bz, U.dt, lds_f64(&buf[2][p]));
  const double u1 = fma(2.0, bx, -u0);
  const double v1 = fma(2.0, by, -v0);
  const double w1 = fma(2.0, bz, -w0);
  const bool fin_v = finite3(u1, v1, w1);
  if (!((dbits(x1) <= dbits(g.ax.hi0)) & (dbits(y1) <= dbits(g.ay.hi0)) &
        (dbits(z1) <= dbits(g.az.hi0)))) {
    x1 = wrap_exact_bits(x1, g.ax, dbits(g.ax.hi0), dbits(g.ax.hi1), dbits(g.ax.lom1) & kAbs);
    y1 = wrap_exact_bits(y1, g.ay, dbits(g.ay.hi0), dbits(g.ay.hi1), dbits(g.ay.lom1) & kAbs);
    z1 = wrap_exact_bits(z1, g.az, dbits(g.az.hi0), dbits(g.az.hi1), dbits(g.az.lom1) & kAbs);
    if (!finite3(x1, y1, z1)) bad = 1u;
  }
  if ((bad == 0u) & fin_v) {
    buf[0][p] = x1; buf[1][p] = y1; buf[2][p] = z1;
    buf[3][p] = u1; buf[4][p] = v1; buf[5][p] = w1;
    return 0u;
  }
  return p < cnt ? 1u : 0u;
}

// ---------------------------------------------------------------------------
// FAST, z-invariant field ("2-D in 3-D", the GEM configurations)
// ---------------------------------------------------------------------------
//
// When every node plane k of E and B equals plane 0 bit for bit (checked on
// the device whenever the field changes, zinv_check_kernel), the z
// coefficients Q of every cell polynomial are exactly zero: P + fz*Q == P, so
// the gather is the bilinear (p0 + fy*p1) + fx*(p2 + fy*p3) of the same P
// values -- the 3-D FAST result up to the sign of an exact zero -- from a
// table of nx*ny columns (24 doubles each).  z crossings need no reload and
// the z predictor feeds nothing but the gather, so it is not formed (a
// non-finite vbar_z is still flagged, and z1 is checked at the end).

#ifndef B2M_2D_PRED_RELOAD
#define B2M_2D_PRED_RELOAD 1    // column reload as predicated loads, not a branch (1.158 -> 1.134 ms; not in the fused kernel)
#endif
#ifndef B2M_2D_LOCATE_ALWAYS
#define B2M_2D_LOCATE_ALWAYS 1  // locate every particle's start (no frame test): 1.16 -> 1.13 ms
#endif

struct Coef4 {
  double p0, p1, p2, p3;
};

__device__ __forceinline__ Coef4 load_coef4(const double* c) {
  Coef4 k;
  const uint64_t pol = policy_evict_last();
  asm("ld.global.nc.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
      : "=d"(k.p0), "=d"(k.p1), "=d"(k.p2), "=d"(k.p3)
      : "l"(c), "l"(pol));
  return k;
}

__device__ __forceinline__ double poly4(const Coef4& k, double fx, double fy) {
  return fma(fx, fma(fy, k.p3, k.p2), fma(fy, k.p1, k.p0));
}

struct FastCol {
  Coef4 K[6];
  double ci, cj;
  int col;
};

__device__ __forceinline__ void fast_col_reset(FastCol& C) {
  C.col = -1;
  C.ci = C.cj = -4.0;
}

// Column reload as six predicated 256-bit loads (no divergent branch, so no
// reconvergence barrier: the scheduler can interleave the unrolled particles
// around it); en = false leaves the cache untouched.
__device__ __forceinline__ void reload_col_pred(FastCol& C, const double* __restrict__ cols,
                                                int col, bool en) {
  const double* c = cols + static_cast<long long>(col) * 24;
  const uint64_t pol = policy_evict_last();
  const int diff = en && col != C.col;
#pragma unroll
  for (int q = 0; q < 6; ++q)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %5, 0;\n\t"
        "@p ld.global.nc.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %6;\n\t}"
        : "+d"(C.K[q].p0), "+d"(C.K[q].p1), "+d"(C.K[q].p2), "+d"(C.K[q].p3)
        : "l"(c + 4 * q), "r"(diff), "l"(pol));
}

template <bool PRED = false>
__device__ __forceinline__ void fast_enter2(const FastGrid& g, const double* __restrict__ cols,
                                            FastCol& C, double tx, double ty, double& fx,
                                            double& fy) {
  const int i = max(min(__double2int_rz(tx), g.nx - 1), 0);
  const int j = max(min(__double2int_rz(ty), g.ny - 1), 0);
  const double di = static_cast<double>(i), dj = static_cast<double>(j);
  fx = tx - di;
  fy = ty - dj;
  const int col = i + g.nx * j;
  if (PRED) {
    reload_col_pred(C, cols, col, true);
    C.col = col;
  } else if (col != C.col) {
    const double* c = cols + static_cast<long long>(col) * 24;
#pragma unroll
    for (int q = 0; q < 6; ++q) C.K[q] = load_coef4(c + 4 * q);
    C.col = col;
  }
  C.ci = di;
  C.cj = dj;
}

// Prefetch into L1 the column table of the particle at (x, y) when it is not
// the lane's cached column: a lane whose next particle sits in another column
// then reloads from L1 instead of waiting an L2 round trip with its whole warp.
__device__ __forceinline__ void col_prefetch(const FastGrid& g, const double* __restrict__ cols,
                                             const FastCol& C, double x, double y) {
  const int i = max(min(__double2int_rz(x * g.rdx), g.nx - 1), 0);
  const int j = max(min(__double2int_rz(y * g.rdy), g.ny - 1), 0);
  const int col = i + g.nx * j;
  if (col != C.col) {
    const double* c = cols + static_cast<long long>(col) * 24;
    prefetch_l1(c);
    prefetch_l1(c + 23);
  }
}

// y_out: the new y of a particle that moved clean (the migration scan reads
// it from a register instead of the tile)
template <int TILE, int ROUNDS, bool PRED = false>
__device__ __forceinline__ unsigned fast_particle_2d(const FastGrid& g, const FastUniform& U,
                                                     const double* __restrict__ cols,
                                                     double (*buf)[TILE], int p, int cnt,
                                                     FastCol& C, double* y_out = nullptr) {
  const double x0 = buf[0][p], y0 = buf[1][p], z0 = buf[2][p];
  const double u0 = buf[3][p], v0 = buf[4][p], w0 = buf[5][p];
  double fx0, fy0;
  unsigned bad = 0u;
  if (B2M_2D_LOCATE_ALWAYS) {
    // every start located (no frame test, no divergent slow path): only the
    // column reload is a branch, and it holds loads only
    const bool inside = (p < cnt) & in_range(x0, dbits(g.lx)) & in_range(y0, dbits(g.ly)) &
                        in_range(z0, dbits(g.lz));
    bad = inside ? 0u : 1u;
    fast_enter2<PRED>(g, cols, C, inside ? x0 * g.rdx : 0.0, inside ? y0 * g.rdy : 0.0, fx0,
                      fy0);
  } else {
    const double cx = x0 * g.rdx, cy = y0 * g.rdy;
    fx0 = cx - C.ci;
    fy0 = cy - C.cj;
    if (!((p < cnt) & below_bits(x0, dbits(g.lx)) & below_bits(y0, dbits(g.ly)) &
          below_bits(z0, dbits(g.lz)) & in_unit(fx0) & in_unit(fy0))) {
      const bool inside = (p < cnt) && in_range(x0, dbits(g.lx)) && in_range(y0, dbits(g.ly)) &&
                          in_range(z0, dbits(g.lz));
      bad = inside ? 0u : 1u;
      fast_enter2(g, cols, C, inside ? cx : 0.0, inside ? cy : 0.0, fx0, fy0);
    }
  }
  double fx = fx0, fy = fy0;
  double nx, ny, nz, rc;
  const int rounds = ROUNDS > 0 ? ROUNDS : U.rounds;
#pragma unroll
  for (int r = 0; r < rounds; ++r) {
    double F[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) F[q] = poly4(C.K[q], fx, fy);
    implicit_num(u0, v0, w0, F, nx, ny, nz, rc);
    if (r + 1 < rounds) {
      // kernels.cpp:92: a non-finite predictor is a fault (z included)
      if (!finite3(nz, rc, rc)) bad = 1u;
      fx = fma(nx * U.dc[0], rc, fx0);
      fy = fma(ny * U.dc[1], rc, fy0);
      const bool cross = !(in_unit(fx) & in_unit(fy));
      if (cross) {
        const double bx = nx * rc, by = ny * rc;
        const double cx = lds_f64(&buf[0][p]) * g.rdx, cy = lds_f64(&buf[1][p]) * g.rdy;
        double tx = fma(bx, U.dc[0], cx), ty = fma(by, U.dc[1], cy);
        if ((dbits(tx) >= dbits(g.nxd)) | (dbits(ty) >= dbits(g.nyd))) {
          tx = fold_fast(tx, g.nxd, dbits(g.nxd), g.rnx, bad);
          ty = fold_fast(ty, g.nyd, dbits(g.nyd), g.rny, bad);
        }
        fast_enter2<PRED>(g, cols, C, tx, ty, fx, fy);
        fx0 = fma(-bx, U.dc[0], fx);
        fy0 = fma(-by, U.dc[1], fy);
      }
    }
  }
  const double bx = nx * rc, by = ny * rc, bz = nz * rc;
  double x1 = fma(bx, U.dt, lds_f64(&buf[0][p]));
  double y1 = fma(by, U.dt, lds_f64(&buf[1][p]));
  double z1 = fma(bz, U.dt, lds_f64(&buf[2][p]));
  const double u1 = fma(2.0, bx, -u0);
  const double v1 = fma(2.0, by, -v0);
  const double w1 = fma(2.0, bz, -w0);
  const bool fin_v = finite3(u1, v1, w1);
  if (!((dbits(x1) <= dbits(g.ax.hi0)) & (dbits(y1) <= dbits(g.ay.hi0)) &
        (dbits(z1) <= dbits(g.az.hi0)))) {
    x1 = wrap_exact_bits(x1, g.ax, dbits(g.ax.hi0), dbits(g.ax.hi1), dbits(g.ax.lom1) & kAbs);
    y1 = wrap_exact_bits(y1, g.ay, dbits(g.ay.hi0), dbits(g.ay.hi1), dbits(g.ay.lom1) & kAbs);
    z1 = wrap_exact_bits(z1, g.az, dbits(g.az.hi0), dbits(g.az.hi1), dbits(g.az.lom1) & kAbs);
    if (!finite3(x1, y1, z1)) bad = 1u;
  }
  if (y_out) *y_out = y1;
  if ((bad == 0u) & fin_v) {
    buf[0][p] = x1; buf[1][p] = y1; buf[2][p] = z1;
    buf[3][p] = u1; buf[4][p] = v1; buf[5][p] = w1;
    return 0u;
  }
  return p < cnt ? 1u : 0u;
}

// ---- two particles per lane (ILP 2) on one column cache ------------------
//
// The lane's particles j and j+1 of a tile (32 apart in a cell-sorted
// species, i.e. nearly always in the same column: a C2 column holds ~7000
// particles per species) are advanced together, their dependency chains
// interleaved.  Each particle keeps its own cell frame (corner, column,
// fractions) exactly as fast_particle_2d does, so its arithmetic -- and
// result -- is the same bit for bit; the shared cache is (re)loaded for a
// particle's column before that particle's gather when it is not the cached
// one (load-only branches, rare), so two particles in different columns
// still move correctly, only with reloads.
struct PairP {
  double u0, v0, w0;
  double fx0, fy0, fx, fy;  // fractions in the particle's own cell frame
  double ci, cj;            // that cell's corner (cell units)
  double nx, ny, nz, rc;
  int col;
  unsigned bad;
};

__device__ __forceinline__ void pair_locate2(const FastGrid& g, double tx, double ty, PairP& P) {
  const int i = max(min(__double2int_rz(tx), g.nx - 1), 0);
  const int j = max(min(__double2int_rz(ty), g.ny - 1), 0);
  P.ci = static_cast<double>(i);
  P.cj = static_cast<double>(j);
  P.fx = tx - P.ci;
  P.fy = ty - P.cj;
  P.col = i + g.nx * j;
}

__device__ __forceinline__ void pair_cache(FastCol& C, const double* __restrict__ cols,
                                           const PairP& P) {
  if (P.col != C.col) {
    const double* c = cols + static_cast<long long>(P.col) * 24;
#pragma unroll
    for (int q = 0; q < 6; ++q) C.K[q] = load_coef4(c + 4 * q);
    C.col = P.col;
    C.ci = P.ci;
    C.cj = P.cj;
  }
}

template <int TILE>
__device__ __forceinline__ void pair_start(const FastGrid& g, const FastCol& C,
                                           double (*buf)[TILE], int p, int cnt, PairP& P) {
  const double x0 = buf[0][p], y0 = buf[1][p], z0 = buf[2][p];
  P.u0 = buf[3][p];
  P.v0 = buf[4][p];
  P.w0 = buf[5][p];
  P.bad = 0u;
  const double cx = x0 * g.rdx, cy = y0 * g.rdy;
  P.fx = cx - C.ci;
  P.fy = cy - C.cj;
  P.ci = C.ci;
  P.cj = C.cj;
  P.col = C.col;
  if (!((p < cnt) & below_bits(x0, dbits(g.lx)) & below_bits(y0, dbits(g.ly)) &
        below_bits(z0, dbits(g.lz)) & in_unit(P.fx) & in_unit(P.fy))) {
    const bool inside = (p < cnt) && in_range(x0, dbits(g.lx)) && in_range(y0, dbits(g.ly)) &&
                        in_range(z0, dbits(g.lz));
    P.bad = inside ? 0u : 1u;
    pair_locate2(g, inside ? cx : 0.0, inside ? cy : 0.0, P);
  }
  P.fx0 = P.fx;
  P.fy0 = P.fy;
}

template <int TILE>
__device__ __forceinline__ void pair_predict(const FastGrid& g, const FastUniform& U,
                                             double (*buf)[TILE], int p, PairP& P) {
  // kernels.cpp:92: a non-finite predictor is a fault (z included)
  if (!finite3(P.nz, P.rc, P.rc)) P.bad = 1u;
  P.fx = fma(P.nx * U.dc[0], P.rc, P.fx0);
  P.fy = fma(P.ny * U.dc[1], P.rc, P.fy0);
  if (!(in_unit(P.fx) & in_unit(P.fy))) {
    const double bx = P.nx * P.rc, by = P.ny * P.rc;
    const double cx = lds_f64(&buf[0][p]) * g.rdx, cy = lds_f64(&buf[1][p]) * g.rdy;
    double tx = fma(bx, U.dc[0], cx), ty = fma(by, U.dc[1], cy);
    if ((dbits(tx) >= dbits(g.nxd)) | (dbits(ty) >= dbits(g.nyd))) {
      tx = fold_fast(tx, g.nxd, dbits(g.nxd), g.rnx, P.bad);
      ty = fold_fast(ty, g.nyd, dbits(g.nyd), g.rny, P.bad);
    }
    pair_locate2(g, tx, ty, P);
    P.fx0 = fma(-bx, U.dc[0], P.fx);
    P.fy0 = fma(-by, U.dc[1], P.fy);
  }
}

template <int TILE>
__device__ __forceinline__ unsigned pair_finish(const FastGrid& g, const FastUniform& U,
                                                double (*buf)[TILE], int p, int cnt, PairP& P) {
  const double bx = P.nx * P.rc, by = P.ny * P.rc, bz = P.nz * P.rc;
  double x1 = fma(bx, U.dt, lds_f64(&buf[0][p]));
  double y1 = fma(by, U.dt, lds_f64(&buf[1][p]));
  double z1 = fma(bz, U.dt, lds_f64(&buf[2][p]));
  const double u1 = fma(2.0, bx, -P.u0);
  const double v1 = fma(2.0, by, -P.v0);
  const double w1 = fma(2.0, bz, -P.w0);
  const bool fin_v = finite3(u1, v1, w1);
  if (!((dbits(x1) <= dbits(g.ax.hi0)) & (dbits(y1) <= dbits(g.ay.hi0)) &
        (dbits(z1) <= dbits(g.az.hi0)))) {
    x1 = wrap_exact_bits(x1, g.ax, dbits(g.ax.hi0), dbits(g.ax.hi1), dbits(g.ax.lom1) & kAbs);
    y1 = wrap_exact_bits(y1, g.ay, dbits(g.ay.hi0), dbits(g.ay.hi1), dbits(g.ay.lom1) & kAbs);
    z1 = wrap_exact_bits(z1, g.az, dbits(g.az.hi0), dbits(g.az.hi1), dbits(g.az.lom1) & kAbs);
    if (!finite3(x1, y1, z1)) P.bad = 1u;
  }
  if ((P.bad == 0u) & fin_v) {
    buf[0][p] = x1; buf[1][p] = y1; buf[2][p] = z1;
    buf[3][p] = u1; buf[4][p] = v1; buf[5][p] = w1;
    return 0u;
  }
  return p < cnt ? 1u : 0u;
}

// Particles pa and pb of the tile; returns the fault bits (1: pa, 2: pb).
template <int TILE, int ROUNDS>
__device__ __forceinline__ unsigned fast_pair_2d(const FastGrid& g, const FastUniform& U,
                                                 const double* __restrict__ cols,
                                                 double (*buf)[TILE], int pa, int pb, int cnt,
                                                 FastCol& C) {
  PairP A, B;
  pair_start<TILE>(g, C, buf, pa, cnt, A);
  pair_start<TILE>(g, C, buf, pb, cnt, B);
  const int rounds = ROUNDS > 0 ? ROUNDS : U.rounds;
#pragma unroll
  for (int r = 0; r < rounds; ++r) {
    double Fa[6], Fb[6];
    pair_cache(C, cols, A);
#pragma unroll
    for (int q = 0; q < 6; ++q) Fa[q] = poly4(C.K[q], A.fx, A.fy);
    pair_cache(C, cols, B);
#pragma unroll
    for (int q = 0; q < 6; ++q) Fb[q] = poly4(C.K[q], B.fx, B.fy);
    implicit_num(A.u0, A.v0, A.w0, Fa, A.nx, A.ny, A.nz, A.rc);
    implicit_num(B.u0, B.v0, B.w0, Fb, B.nx, B.ny, B.nz, B.rc);
    if (r + 1 < rounds) {
      pair_predict<TILE>(g, U, buf, pa, A);
      pair_predict<TILE>(g, U, buf, pb, B);
    }
  }
  return pair_finish<TILE>(g, U, buf, pa, cnt, A) | (pair_finish<TILE>(g, U, buf, pb, cnt, B) << 1);
}

// ---------------------------------------------------------------------------
// STRICT: the reference's operation order, every rounding separate
// ---------------------------------------------------------------------------

struct PState {
  double x0, y0, z0, u0, v0, w0;
  double tx, ty, tz;   // predictor position (FAST: cell units, STRICT: physical)
  double cx0, cy0, cz0;  // FAST: x0 in cell units
  double bx, by, bz;   // time-centred velocity
  bool ok;
};

// Cell field cache.  FAST: 24 double2 polynomial pairs (b2m_mover.cuh
// layout).  STRICT: the 8 corner nodes' (E, B) in corner order.
#ifndef B2M_STRICT_PRED_RELOAD
#define B2M_STRICT_PRED_RELOAD 1  // STRICT cache reload as predicated loads (3.077 -> 3.064 ms)
#endif
struct CellCache {
  double2 c[24];
  int cell;
};

// The 8 corner nodes' E and B of a cell: 48 doubles laid out by
// strict_nodes_kernel in exactly the cache's order (corner c: Ex Ey Ez Bx By
// Bz), so the reload is twelve 256-bit loads -- the same values the
// reference reads from the node mesh, bit for bit.
// DIM 2 (z-invariant field: corners 4-7 equal corners 0-3 bit for bit): the
// first 24 doubles of the column's k = 0 cell, corners 0-3.
template <int DIM = 3>
__device__ __forceinline__ void cache_load_strict(CellCache& cc, const double* __restrict__ nodes,
                                                  int cell) {
  const double* c = nodes + static_cast<long long>(cell) * 48;
#pragma unroll
  for (int q = 0; q < (DIM == 2 ? 6 : 12); ++q) {
    double a, b, d, e;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(a), "=d"(b), "=d"(d), "=d"(e)
        : "l"(c + 4 * q));
    cc.c[2 * q] = make_double2(a, b);
    cc.c[2 * q + 1] = make_double2(d, e);
  }
  cc.cell = cell;
}

// The same reload as predicated loads (no divergent branch): the cache is
// replaced only where `diff` is set.
template <int DIM = 3>
__device__ __forceinline__ void cache_load_strict_pred(CellCache& cc,
                                                       const double* __restrict__ nodes, int cell,
                                                       bool diff) {
  const double* c = nodes + static_cast<long long>(cell) * 48;
  const int d = diff;
#pragma unroll
  for (int q = 0; q < (DIM == 2 ? 6 : 12); ++q)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %5, 0;\n\t"
        "@p ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];\n\t}"
        : "+d"(cc.c[2 * q].x), "+d"(cc.c[2 * q].y), "+d"(cc.c[2 * q + 1].x),
          "+d"(cc.c[2 * q + 1].y)
        : "l"(c + 4 * q), "r"(d));
  cc.cell = cell;
}

__device__ __forceinline__ void begin(PState& P, const double* p) {
  P.x0 = p[0]; P.y0 = p[1]; P.z0 = p[2];
  P.u0 = p[3]; P.v0 = p[4]; P.w0 = p[5];
  P.tx = P.x0; P.ty = P.y0; P.tz = P.z0;
  P.bx = P.u0; P.by = P.v0; P.bz = P.w0;
  P.ok = true;
}

__device__ __forceinline__ int strict_locate(PState& P, const DevGrid& g, double* wt,
                                             int* column = nullptr) {
  if (!(P.tx >= 0.0 && P.tx < g.lx && P.ty >= 0.0 && P.ty < g.ly && P.tz >= 0.0 && P.tz < g.lz)) {
    P.ok = false;
    return -1;
  }
  const double sx = div_axis(P.tx, g.dx, g.rdx), sy = div_axis(P.ty, g.dy, g.rdy),
               sz = div_axis(P.tz, g.dz, g.rdz);
  int i = __double2int_rz(sx), j = __double2int_rz(sy), k = __double2int_rz(sz);
  if (i >= g.nx) i = g.nx - 1;
  if (j >= g.ny) j = g.ny - 1;
  if (k >= g.nz) k = g.nz - 1;
  double fx = __dsub_rn(sx, static_cast<double>(i));
  double fy = __dsub_rn(sy, static_cast<double>(j));
  double fz = __dsub_rn(sz, static_cast<double>(k));
  if (fx > 1.0) fx = 1.0;
  if (fy > 1.0) fy = 1.0;
  if (fz > 1.0) fz = 1.0;
  const double wx[2] = {__dsub_rn(1.0, fx), fx};
  const double wy[2] = {__dsub_rn(1.0, fy), fy};
  const double wz[2] = {__dsub_rn(1.0, fz), fz};
#pragma unroll
  for (int c = 0; c < 8; ++c)
    wt[c] = __dmul_rn(__dmul_rn(wx[c & 1], wy[(c >> 1) & 1]), wz[(c >> 2) & 1]);
  if (column) *column = i + g.nx * j;
  return i + g.nx * (j + g.ny * k);
}

template <int DIM = 3>
__device__ __forceinline__ void strict_round(PState& P, const CellCache& cc, const double* wt,
                                             double beta) {
  double ex = 0.0, ey = 0.0, ez = 0.0, fbx = 0.0, fby = 0.0, fbz = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double w = wt[c];
    const int n = DIM == 2 ? (c & 3) : c;  // z-invariant: corner c + 4 holds corner c's values
    ex = __dadd_rn(ex, __dmul_rn(w, cc.c[3 * n + 0].x));
    ey = __dadd_rn(ey, __dmul_rn(w, cc.c[3 * n + 0].y));
    ez = __dadd_rn(ez, __dmul_rn(w, cc.c[3 * n + 1].x));
    fbx = __dadd_rn(fbx, __dmul_rn(w, cc.c[3 * n + 1].y));
    fby = __dadd_rn(fby, __dmul_rn(w, cc.c[3 * n + 2].x));
    fbz = __dadd_rn(fbz, __dmul_rn(w, cc.c[3 * n + 2].y));
  }
  const double vtx = __dadd_rn(P.u0, __dmul_rn(beta, ex));
  const double vty = __dadd_rn(P.v0, __dmul_rn(beta, ey));
  const double vtz = __dadd_rn(P.w0, __dmul_rn(beta, ez));
  const double ox = __dmul_rn(beta, fbx), oy = __dmul_rn(beta, fby), oz = __dmul_rn(beta, fbz);
  const double omsq = __dadd_rn(__dadd_rn(__dmul_rn(ox, ox), __dmul_rn(oy, oy)), __dmul_rn(oz, oz));
  const double denom = __ddiv_rn(1.0, __dadd_rn(1.0, omsq));
  const double vdot = __dadd_rn(__dadd_rn(__dmul_rn(vtx, ox), __dmul_rn(vty, oy)), __dmul_rn(vtz, oz));
  P.bx = __dmul_rn(__dadd_rn(__dadd_rn(vtx, __dsub_rn(__dmul_rn(vty, oz), __dmul_rn(vtz, oy))),
                             __dmul_rn(vdot, ox)), denom);
  P.by = __dmul_rn(__dadd_rn(__dadd_rn(vty, __dsub_rn(__dmul_rn(vtz, ox), __dmul_rn(vtx, oz))),
                             __dmul_rn(vdot, oy)), denom);
  P.bz = __dmul_rn(__dadd_rn(__dadd_rn(vtz, __dsub_rn(__dmul_rn(vtx, oy), __dmul_rn(vty, ox))),
                             __dmul_rn(vdot, oz)), denom);
}

// wrap_len (grid.hpp:45-50) bit for bit: the quotient's floor read off the
// WrapAxis thresholds instead of an IEEE division (same result, see WrapAxis)
__device__ __forceinline__ double wrap_strict(double v, const WrapAxis& a) {
  // common case v in [+0, hi0]: floor(RN(v/l)) = 0, w = v, no fix-up applies
  if (dbits(v) <= dbits(a.hi0)) return v;
  return wrap_exact_bits(v, a, dbits(a.hi0), dbits(a.hi1), dbits(a.lom1) & kAbs);
}

__device__ __forceinline__ void strict_predict(PState& P, const FastGrid& w, double dto2) {
  P.tx = wrap_strict(__dadd_rn(P.x0, __dmul_rn(P.bx, dto2)), w.ax);
  P.ty = wrap_strict(__dadd_rn(P.y0, __dmul_rn(P.by, dto2)), w.ay);
  P.tz = wrap_strict(__dadd_rn(P.z0, __dmul_rn(P.bz, dto2)), w.az);
}

__device__ __forceinline__ bool strict_finish(PState& P, const FastGrid& w, double dt, double* out) {
  if (!P.ok) return false;
  const double x1 = wrap_strict(__dadd_rn(P.x0, __dmul_rn(P.bx, dt)), w.ax);
  const double y1 = wrap_strict(__dadd_rn(P.y0, __dmul_rn(P.by, dt)), w.ay);
  const double z1 = wrap_strict(__dadd_rn(P.z0, __dmul_rn(P.bz, dt)), w.az);
  const double u1 = __dsub_rn(__dmul_rn(2.0, P.bx), P.u0);
  const double v1 = __dsub_rn(__dmul_rn(2.0, P.by), P.v0);
  const double w1 = __dsub_rn(__dmul_rn(2.0, P.bz), P.w0);
  if (!(isfinite(x1) && isfinite(y1) && isfinite(z1) && isfinite(u1) && isfinite(v1) &&
        isfinite(w1)))
    return false;
  out[0] = x1; out[1] = y1; out[2] = z1;
  out[3] = u1; out[4] = v1; out[5] = w1;
  return true;
}

// ---------------------------------------------------------------------------
// STRICT, one particle per thread at a time with a register node cache
// ---------------------------------------------------------------------------
//
// Bit-identical to the reference: every round locates with IEEE divisions,
// computes the 8 weights and accumulates the corners in the reference's
// order with separate roundings.  The 8 corner nodes' E and B (48 doubles)
// stay in registers while the particle -- and the lane's next particles --
// remain in the same cell: a bitwise-identical reuse of values the reference
// would re-read.
// DIM 2: the field is z-invariant (zinv_check_kernel, bitwise), so the cache
// holds the column's 4 corner nodes -- the reference's 8 products and sums are
// all still formed, in its order, from the same values -- and z crossings do
// not reload.
template <int TILE, int ROUNDS = 0, int DIM = 3>
__device__ __forceinline__ unsigned strict_tile_thread_p1(const DevGrid& g, const FastGrid& wg,
                                                          const double* __restrict__ nodes,
                                                          const SpeciesLaunch& sp,
                                                          double (*buf)[TILE], int p, int cnt,
                                                          CellCache& cc) {
  if (p >= cnt) return 0u;
  PState P;
  const double in[6] = {buf[0][p], buf[1][p], buf[2][p], buf[3][p], buf[4][p], buf[5][p]};
  begin(P, in);
  const int rounds = ROUNDS > 0 ? ROUNDS : sp.rounds;
#pragma unroll
  for (int r = 0; r < rounds; ++r) {
    double wt[8];
    int column;
    const int cell = strict_locate(P, g, wt, DIM == 2 ? &column : nullptr);
    if (!P.ok) return 1u;  // the reference's DomainError -> NumericalFault
    const int key = DIM == 2 ? column : cell;
    if (B2M_STRICT_PRED_RELOAD) cache_load_strict_pred<DIM>(cc, nodes, key, key != cc.cell);
    else if (key != cc.cell) cache_load_strict<DIM>(cc, nodes, key);
    strict_round<DIM>(P, cc, wt, sp.beta);
    if (r + 1 < rounds) strict_predict(P, wg, sp.dto2);
  }
  double out[6];
  if (!strict_finish(P, wg, sp.dt, out)) return 1u;
#pragma unroll
  for (int a = 0; a < 6; ++a) buf[a][p] = out[a];
  return 0u;
}
}  // namespace b2m
