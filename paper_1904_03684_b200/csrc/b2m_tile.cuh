// b2m_tile.cuh — the production mover: persistent, TMA-staged, two particles
// per thread sharing a register-resident cell cache.
//
// Why this shape (profiles/r01_fast_v1.md): a thread-per-particle gather pulls
// 48 doubles of field per particle per predictor round into registers, and on
// sm_100a the L1->register writeback (128 B/clk/SM) saturates long before the
// FP64 pipe or HBM do.  The field of a cell is identical for every round in
// which the particle stays in that cell (>99% of rounds: |v| dt/2 is a few
// percent of a cell) and for both particles of a thread after the cell sort,
// so the 48 values are loaded into registers once per (thread, cell) and
// reused: 3 rounds x 2 particles per load instead of 1.
//
// Particle tiles (256 particles x 6 SoA arrays = 12 KB) stream through shared
// memory with 1-D bulk TMA copies (cp.async.bulk + mbarrier, 3 stages), and
// results leave through bulk TMA stores, so HBM latency hides behind the
// FP64 work of the previous tiles without spending registers on prefetch.
// Partial tail tiles (and unaligned spans) use plain loads/stores.
#pragma once

#include <cuda.h>

#include "b2m_mover.cuh"

namespace b2m {

#ifndef B2M_TPB
#define B2M_TPB 128
#endif
#ifndef B2M_WARP_STAGES
#define B2M_WARP_STAGES 3
#endif
constexpr int kTileThreads = 128;        // block-tile (STRICT legacy) kernel
constexpr int kWarpThreads = B2M_TPB;     // warp-tile kernels
constexpr int kTileStages = 2;
constexpr int kWarpStages = B2M_WARP_STAGES;
constexpr int kTileMinBlocks = 3;
// particles per thread: FAST streams coefficients to 4 particles, STRICT
// keeps a register cell cache shared by 2
// FAST kernel shape (tuned on B200, tools/sweep.py): each lane moves 4
// particles one after the other with a register cell cache (SEQ), 3 blocks
// of 128 threads per SM.  SEQ=0 selects the older pair-sharing variant.
#ifndef B2M_FAST_PPT
#define B2M_FAST_PPT 4
#endif
#ifndef B2M_FAST_SEQ
#define B2M_FAST_SEQ 1
#endif
#ifndef B2M_FAST_MINBLOCKS
#define B2M_FAST_MINBLOCKS 3
#endif
template <bool STRICT>
struct TileShape {
  static constexpr int ppt = STRICT ? 2 : B2M_FAST_PPT;
  static constexpr int tile = kTileThreads * ppt;
  static constexpr int smem = kTileStages * 6 * tile * 8 + 64;
};
constexpr int kMaxTileSpans = 8;

struct TileSpans {
  SpeciesLaunch sp[kMaxTileSpans];
  unsigned long long tile_start[kMaxTileSpans + 1];
  int tma_ok[kMaxTileSpans];
  int n;
};

// FAST launch: per span a 2-D tensor map over the species' [6][stride]
// block (dims {col0 + n, 6}), so one TMA box moves all six arrays of a tile
// and the hardware clips partial tiles.
struct alignas(64) TensorSpans {
  CUtensorMap tmap[kMaxTileSpans];
  SpeciesLaunch sp[kMaxTileSpans];
  unsigned long long tile_start[kMaxTileSpans + 1];
  uint8_t* flags[kMaxTileSpans];  // migration: per-particle destination flag (or null)
  int n;
};

// ---------------------------------------------------------------------------
// TMA / mbarrier primitives (PTX ISA 8.x, sm_90+; SASS: UBLKCP, SYNCS)
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

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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

__device__ __forceinline__ void tma_load_1d_hint(void* smem_dst, const void* gmem_src,
                                                 uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void tma_store_1d_hint(void* gmem_dst, const void* smem_src,
                                                  uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                   gmem_dst),
               "r"(smem_u32(smem_src)), "r"(bytes), "l"(pol)
               : "memory");
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

__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_store_1d(void* gmem_dst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
               "r"(smem_u32(smem_src)), "r"(bytes)
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
// per-particle state machines
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
struct CellCache {
  double2 c[24];
  int cell;
};

__device__ __forceinline__ void cache_load_fast(CellCache& cc, const double2* __restrict__ cells,
                                                int cell) {
  const double2* src = cells + static_cast<long long>(cell) * 24;
#pragma unroll
  for (int q = 0; q < 24; ++q) cc.c[q] = __ldg(src + q);
  cc.cell = cell;
}

__device__ __forceinline__ void cache_load_strict(CellCache& cc, const DevGrid& g,
                                                  const double* __restrict__ E,
                                                  const double* __restrict__ B, int cell) {
  const int i = cell % g.nx;
  const int j = (cell / g.nx) % g.ny;
  const int k = cell / (g.nx * g.ny);
  const long long sx1 = g.nx + 1, sy1 = g.ny + 1;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int di = c & 1, dj = (c >> 1) & 1, dk = (c >> 2) & 1;
    const long long n = 3 * ((i + di) + sx1 * ((j + dj) + sy1 * (k + dk)));
    cc.c[3 * c + 0] = make_double2(__ldg(E + n + 0), __ldg(E + n + 1));
    cc.c[3 * c + 1] = make_double2(__ldg(E + n + 2), __ldg(B + n + 0));
    cc.c[3 * c + 2] = make_double2(__ldg(B + n + 1), __ldg(B + n + 2));
  }
  cc.cell = cell;
}

__device__ __forceinline__ void begin(PState& P, const double* p) {
  P.x0 = p[0]; P.y0 = p[1]; P.z0 = p[2];
  P.u0 = p[3]; P.v0 = p[4]; P.w0 = p[5];
  P.tx = P.x0; P.ty = P.y0; P.tz = P.z0;
  P.bx = P.u0; P.by = P.v0; P.bz = P.w0;
  P.ok = true;
}

// ---- FAST -----------------------------------------------------------------

__device__ __forceinline__ void fast_begin(PState& P, const FastGrid& g, const double* p) {
  begin(P, p);
  // grid.hpp:65-67: the first locate rejects x0 outside [0,l)
  P.ok = (P.x0 >= 0.0 && P.x0 < g.lx && P.y0 >= 0.0 && P.y0 < g.ly && P.z0 >= 0.0 && P.z0 < g.lz);
  P.cx0 = P.x0 * g.rdx; P.cy0 = P.y0 * g.rdy; P.cz0 = P.z0 * g.rdz;
  P.tx = P.cx0; P.ty = P.cy0; P.tz = P.cz0;
}

// Returns the cell and fractions; clears P.ok on a non-finite position.
__device__ __forceinline__ int fast_locate(PState& P, const FastGrid& g, double& fx, double& fy,
                                           double& fz) {
  if (!(P.tx >= 0.0 && P.tx <= g.nxd && P.ty >= 0.0 && P.ty <= g.nyd && P.tz >= 0.0 &&
        P.tz <= g.nzd)) {
    P.ok = false;
    return -1;
  }
  const int i = min(__double2int_rz(P.tx), g.nx - 1);
  const int j = min(__double2int_rz(P.ty), g.ny - 1);
  const int k = min(__double2int_rz(P.tz), g.nz - 1);
  fx = P.tx - static_cast<double>(i);
  fy = P.ty - static_cast<double>(j);
  fz = P.tz - static_cast<double>(k);
  return i + g.nx * (j + g.ny * k);
}

__device__ __forceinline__ double fast_comp(const double2* c, double fx, double fy, double fz) {
  const double p0 = fma(fz, c[0].y, c[0].x);
  const double p1 = fma(fz, c[1].y, c[1].x);
  const double p2 = fma(fz, c[2].y, c[2].x);
  const double p3 = fma(fz, c[3].y, c[3].x);
  return fma(fx, fma(fy, p3, p2), fma(fy, p1, p0));
}

__device__ __forceinline__ void fast_round(PState& P, const CellCache& cc, double fx, double fy,
                                           double fz, double beta) {
  const double ex = fast_comp(cc.c + 0, fx, fy, fz);
  const double ey = fast_comp(cc.c + 4, fx, fy, fz);
  const double ez = fast_comp(cc.c + 8, fx, fy, fz);
  const double ox = beta * fast_comp(cc.c + 12, fx, fy, fz);
  const double oy = beta * fast_comp(cc.c + 16, fx, fy, fz);
  const double oz = beta * fast_comp(cc.c + 20, fx, fy, fz);
  const double vtx = fma(beta, ex, P.u0);
  const double vty = fma(beta, ey, P.v0);
  const double vtz = fma(beta, ez, P.w0);
  const double den = 1.0 + fma(oz, oz, fma(oy, oy, ox * ox));
  double rc;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(den));
  double e = fma(-den, rc, 1.0);
  rc = fma(rc, e, rc);
  e = fma(-den, rc, 1.0);
  rc = fma(rc, e, rc);
  e = fma(-den, rc, 1.0);
  rc = fma(rc, e, rc);
  const double vdot = fma(vtz, oz, fma(vty, oy, vtx * ox));
  P.bx = fma(vdot, ox, vtx + fma(vty, oz, -vtz * oy)) * rc;
  P.by = fma(vdot, oy, vty + fma(vtz, ox, -vtx * oz)) * rc;
  P.bz = fma(vdot, oz, vtz + fma(vtx, oy, -vty * ox)) * rc;
}

__device__ __forceinline__ void fast_predict(PState& P, const FastGrid& g, const double* dto2c) {
  P.tx = fold_cells(fma(P.bx, dto2c[0], P.cx0), g.nxd, g.rnx);
  P.ty = fold_cells(fma(P.by, dto2c[1], P.cy0), g.nyd, g.rny);
  P.tz = fold_cells(fma(P.bz, dto2c[2], P.cz0), g.nzd, g.rnz);
}

__device__ __forceinline__ bool fast_finish(PState& P, const FastGrid& g, double dt, double* out) {
  if (!P.ok) return false;
  const double x1 = wrap_len_exact(fma(P.bx, dt, P.x0), g.ax);
  const double y1 = wrap_len_exact(fma(P.by, dt, P.y0), g.ay);
  const double z1 = wrap_len_exact(fma(P.bz, dt, P.z0), g.az);
  const double u1 = fma(2.0, P.bx, -P.u0);
  const double v1 = fma(2.0, P.by, -P.v0);
  const double w1 = fma(2.0, P.bz, -P.w0);
  if (!(isfinite(x1) && isfinite(y1) && isfinite(z1) && isfinite(u1) && isfinite(v1) &&
        isfinite(w1)))
    return false;
  out[0] = x1; out[1] = y1; out[2] = z1;
  out[3] = u1; out[4] = v1; out[5] = w1;
  return true;
}

// ---- STRICT (reference order, separate roundings) -------------------------

__device__ __forceinline__ int strict_locate(PState& P, const DevGrid& g, double* wt) {
  if (!(P.tx >= 0.0 && P.tx < g.lx && P.ty >= 0.0 && P.ty < g.ly && P.tz >= 0.0 && P.tz < g.lz)) {
    P.ok = false;
    return -1;
  }
  const double sx = __ddiv_rn(P.tx, g.dx), sy = __ddiv_rn(P.ty, g.dy), sz = __ddiv_rn(P.tz, g.dz);
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
  return i + g.nx * (j + g.ny * k);
}

__device__ __forceinline__ void strict_round(PState& P, const CellCache& cc, const double* wt,
                                             double beta) {
  double ex = 0.0, ey = 0.0, ez = 0.0, fbx = 0.0, fby = 0.0, fbz = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double w = wt[c];
    ex = __dadd_rn(ex, __dmul_rn(w, cc.c[3 * c + 0].x));
    ey = __dadd_rn(ey, __dmul_rn(w, cc.c[3 * c + 0].y));
    ez = __dadd_rn(ez, __dmul_rn(w, cc.c[3 * c + 1].x));
    fbx = __dadd_rn(fbx, __dmul_rn(w, cc.c[3 * c + 1].y));
    fby = __dadd_rn(fby, __dmul_rn(w, cc.c[3 * c + 2].x));
    fbz = __dadd_rn(fbz, __dmul_rn(w, cc.c[3 * c + 2].y));
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

__device__ __forceinline__ void strict_predict(PState& P, const DevGrid& g, double dto2) {
  P.tx = wrap_len_strict(__dadd_rn(P.x0, __dmul_rn(P.bx, dto2)), g.lx);
  P.ty = wrap_len_strict(__dadd_rn(P.y0, __dmul_rn(P.by, dto2)), g.ly);
  P.tz = wrap_len_strict(__dadd_rn(P.z0, __dmul_rn(P.bz, dto2)), g.lz);
}

__device__ __forceinline__ bool strict_finish(PState& P, const DevGrid& g, double dt, double* out) {
  if (!P.ok) return false;
  const double x1 = wrap_len_strict(__dadd_rn(P.x0, __dmul_rn(P.bx, dt)), g.lx);
  const double y1 = wrap_len_strict(__dadd_rn(P.y0, __dmul_rn(P.by, dt)), g.ly);
  const double z1 = wrap_len_strict(__dadd_rn(P.z0, __dmul_rn(P.bz, dt)), g.lz);
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
// two particles, one cell cache
// ---------------------------------------------------------------------------

struct TileField {
  FastGrid fg;
  DevGrid dg;
  const double2* cells;  // FAST
  const double* E;       // STRICT
  const double* B;
};

// Advances P consecutive particles p[i] (only those with has[i]).  They share
// one register cell cache; when every live particle of the group sits in the
// same cell (the common case after the cell sort) the P evaluations run as
// independent instruction streams -- P-fold ILP for the FP64 chains.
// Results overwrite p[i] on success; ok[i] reports success.
template <bool STRICT, int P>
__device__ __forceinline__ void push_group(const TileField& F, const SpeciesLaunch& sp,
                                           double (&p)[P][6], const bool (&has)[P],
                                           bool (&ok)[P]) {
  PState S[P];
#pragma unroll
  for (int i = 0; i < P; ++i) {
    if (STRICT)
      begin(S[i], p[i]);
    else
      fast_begin(S[i], F.fg, p[i]);
    S[i].ok = S[i].ok && has[i];
  }
  CellCache cc;
  cc.cell = -1;
  for (int r = 0; r < sp.rounds; ++r) {
    const bool pred = r + 1 < sp.rounds;
    int cell[P];
    double w[P][8];  // STRICT: trilinear weights; FAST: w[i][0..2] = fractions
#pragma unroll
    for (int i = 0; i < P; ++i) {
      cell[i] = -1;
      if (S[i].ok) {
        if (STRICT)
          cell[i] = strict_locate(S[i], F.dg, w[i]);
        else
          cell[i] = fast_locate(S[i], F.fg, w[i][0], w[i][1], w[i][2]);
      }
    }
    int ref = -1;
    bool same = true;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      if (!S[i].ok) continue;
      if (ref < 0) ref = cell[i];
      same = same && (cell[i] == ref);
    }
    if (ref < 0) break;  // every particle of the group faulted
    if (same) {
      if (ref != cc.cell) {
        if (STRICT)
          cache_load_strict(cc, F.dg, F.E, F.B, ref);
        else
          cache_load_fast(cc, F.cells, ref);
      }
#pragma unroll
      for (int i = 0; i < P; ++i) {
        if (!S[i].ok) continue;
        if (STRICT) {
          strict_round(S[i], cc, w[i], sp.beta);
          if (pred) strict_predict(S[i], F.dg, sp.dto2);
        } else {
          fast_round(S[i], cc, w[i][0], w[i][1], w[i][2], sp.beta);
          if (pred) fast_predict(S[i], F.fg, sp.dto2_cell);
        }
      }
    } else {
#pragma unroll 1
      for (int i = 0; i < P; ++i) {
        if (!S[i].ok) continue;
        if (cell[i] != cc.cell) {
          if (STRICT)
            cache_load_strict(cc, F.dg, F.E, F.B, cell[i]);
          else
            cache_load_fast(cc, F.cells, cell[i]);
        }
        if (STRICT) {
          strict_round(S[i], cc, w[i], sp.beta);
          if (pred) strict_predict(S[i], F.dg, sp.dto2);
        } else {
          fast_round(S[i], cc, w[i][0], w[i][1], w[i][2], sp.beta);
          if (pred) fast_predict(S[i], F.fg, sp.dto2_cell);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < P; ++i) {
    if (STRICT)
      ok[i] = has[i] && strict_finish(S[i], F.dg, sp.dt, p[i]);
    else
      ok[i] = has[i] && fast_finish(S[i], F.fg, sp.dt, p[i]);
  }
}

// ---------------------------------------------------------------------------
// FAST, coefficient streaming: P particles per thread, no register cache
// ---------------------------------------------------------------------------
//
// Each round, each of the 24 coefficient pairs of a cell is loaded once (L1
// hit) and applied to all P particles of the thread when they share that cell
// (the common case after the cell sort): L1->register traffic per particle is
// 3 rounds x 384 B / P, and the P particles give P independent FP64 chains.
//
// Control flow is kept off the FP64 pipe and out of the warp: every range
// check is an unsigned compare of the IEEE bit pattern (for x >= +0 the bit
// patterns order like the values; negatives, -0, NaN and Inf all land above
// any positive bound), invalid lanes compute on harmless data and are masked
// at the store, and cell indices are clamped so a NaN can never address
// memory.  A sticky per-particle flag records every event the reference
// would have thrown on (x0 outside [0,l), a non-finite predictor position,
// a non-finite result), so faults name the same particles.

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

#ifndef B2M_LDG256
#define B2M_LDG256 1
#endif
#ifndef B2M_L2HINT
#define B2M_L2HINT 1
#endif
__device__ __forceinline__ Coef8 load_coef8(const double2* c) {
  Coef8 k;
#if B2M_L2HINT && B2M_LDG256
  const uint64_t pol = policy_evict_last();
  asm("ld.global.nc.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
      : "=d"(k.p0), "=d"(k.q0), "=d"(k.p1), "=d"(k.q1)
      : "l"(c), "l"(pol));
  asm("ld.global.nc.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
      : "=d"(k.p2), "=d"(k.q2), "=d"(k.p3), "=d"(k.q3)
      : "l"(c + 2), "l"(pol));
  return k;
#endif
#if !B2M_LDG256
  const double2 a = __ldg(c), b = __ldg(c + 1), cc = __ldg(c + 2), d = __ldg(c + 3);
  k.p0 = a.x; k.q0 = a.y; k.p1 = b.x; k.q1 = b.y;
  k.p2 = cc.x; k.q2 = cc.y; k.p3 = d.x; k.q3 = d.y;
  return k;
#endif
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(k.p0), "=d"(k.q0), "=d"(k.p1), "=d"(k.q1)
      : "l"(c));
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(k.p2), "=d"(k.q2), "=d"(k.p3), "=d"(k.q3)
      : "l"(c + 2));
  return k;
}

__device__ __forceinline__ double poly8(const Coef8& k, double fx, double fy, double fz) {
  return fma(fx, fma(fy, fma(fz, k.q3, k.p3), fma(fz, k.q2, k.p2)),
             fma(fy, fma(fz, k.q1, k.p1), fma(fz, k.q0, k.p0)));
}

__device__ __forceinline__ double poly(const double2& a, const double2& b, const double2& c,
                                       const double2& d, double fx, double fy, double fz) {
  return fma(fx, fma(fy, fma(fz, d.y, d.x), fma(fz, c.y, c.x)),
             fma(fy, fma(fz, b.y, b.x), fma(fz, a.y, a.x)));
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
  double beta, dt, dcx, dcy, dcz;         // dcx = 0.5*dt/dx
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
  k.beta = sp.beta; k.dt = sp.dt;
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

// Implicit velocity (kernels.cpp:83-90), FMA form: vt = v0 + beta*E,
// W = beta*B, vbar = (vt + vt x W + (vt.W) W) / (1 + |W|^2).  The reciprocal
// is the MUFU.RCP64H seed (~2^-23) refined by two Newton steps (~2^-92).
__device__ __forceinline__ void implicit_v(double beta, double u0, double v0, double w0,
                                           const double* F, double& bx, double& by, double& bz) {
  const double ox = beta * F[3], oy = beta * F[4], oz = beta * F[5];
  const double vtx = fma(beta, F[0], u0);
  const double vty = fma(beta, F[1], v0);
  const double vtz = fma(beta, F[2], w0);
  const double den = 1.0 + fma(oz, oz, fma(oy, oy, ox * ox));
  double rc;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(den));
  double e = fma(-den, rc, 1.0);
  rc = fma(rc, e, rc);
  e = fma(-den, rc, 1.0);
  rc = fma(rc, e, rc);
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

// One thread's P particles of a staged tile: buf[a][i0 + i] holds input a of
// particle i (x,y,z,u,v,w); results overwrite it for particles that finish
// clean.  Returns a bit mask of particles that must be reported as faulted.
template <int P, int TILE>
__device__ __forceinline__ unsigned fast_tile_thread(const FastGrid& g,
                                                     const double2* __restrict__ cells,
                                                     const FastConst& k, double (*buf)[TILE],
                                                     int i0, int cnt) {
  static_assert(P % 2 == 0 || P == 1, "pairs of particles are read with 128-bit shared loads");
  double u0[P], v0[P], w0[P], cx0[P], cy0[P], cz0[P], fx[P], fy[P], fz[P];
  int cell[P];
  unsigned bad[P];
#pragma unroll
  for (int i = 0; i < P; i += 2) {
    const double2 X = *reinterpret_cast<const double2*>(&buf[0][i0 + i]);
    const double2 Y = *reinterpret_cast<const double2*>(&buf[1][i0 + i]);
    const double2 Z = *reinterpret_cast<const double2*>(&buf[2][i0 + i]);
    const double2 U = *reinterpret_cast<const double2*>(&buf[3][i0 + i]);
    const double2 V = *reinterpret_cast<const double2*>(&buf[4][i0 + i]);
    const double2 W = *reinterpret_cast<const double2*>(&buf[5][i0 + i]);
    const double xs[2] = {X.x, X.y}, ys[2] = {Y.x, Y.y}, zs[2] = {Z.x, Z.y};
    u0[i] = U.x; u0[i + 1] = U.y;
    v0[i] = V.x; v0[i + 1] = V.y;
    w0[i] = W.x; w0[i + 1] = W.y;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = i + h;
      // grid.hpp:65-67: the first locate rejects x0 outside [0,l)
      const bool inside = (i0 + q < cnt) && in_range(xs[h], k.lxb) && in_range(ys[h], k.lyb) &&
                          in_range(zs[h], k.lzb);
      bad[q] = inside ? 0u : 1u;
      cx0[q] = inside ? xs[h] * k.rdx : 0.0;
      cy0[q] = inside ? ys[h] * k.rdy : 0.0;
      cz0[q] = inside ? zs[h] * k.rdz : 0.0;
      cell[q] = locate_fast(k, cx0[q], cy0[q], cz0[q], fx[q], fy[q], fz[q]);
    }
  }
#ifndef B2M_FAST_CACHE
#define B2M_FAST_CACHE 0
#endif
#if B2M_FAST_CACHE
  // Register cell cache: the 48 coefficients of one cell stay in registers
  // across the predictor rounds and are shared by the P particles; it is
  // refilled only when fewer than half of the live particles sit in it.
  Coef8 K[6];
  int kcell = -1;
#endif
  for (int r = 0; r < k.rounds; ++r) {
    double F[P][6];
#if B2M_FAST_CACHE
    {
      int hits = 0;
#pragma unroll
      for (int i = 0; i < P; ++i) hits += (cell[i] == kcell) ? 1 : 0;
      if (2 * hits < P) {
        kcell = cell[0];
        const double2* c = cells + static_cast<long long>(kcell) * 24;
#pragma unroll
        for (int q = 0; q < 6; ++q) K[q] = load_coef8(c + 4 * q);
      }
    }
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
      for (int i = 0; i < P; ++i) F[i][q] = poly8(K[q], fx[i], fy[i], fz[i]);
#pragma unroll
    for (int i = 0; i < P; ++i) {
      if (cell[i] != kcell) {
        const double2* c = cells + static_cast<long long>(cell[i]) * 24;
#pragma unroll
        for (int q = 0; q < 6; ++q) F[i][q] = poly8(load_coef8(c + 4 * q), fx[i], fy[i], fz[i]);
      }
    }
#elif defined(B2M_DIAG_NOGATHER)
    // DIAGNOSTIC BUILD ONLY (tools/build_variants.sh): no field loads at all
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
      for (int i = 0; i < P; ++i) F[i][q] = fma(fx[i], fy[i], fz[i] * (0.001 * q));
#else
    // every particle is gathered with the coefficients of particle 0's cell
    // (one L1 load per pair, shared by the group); a particle that sits in
    // another cell is re-gathered from its own.  A warp pays the fix-up only
    // when one of its lanes needs it, instead of running a second full path.
    {
      const double2* c = cells + static_cast<long long>(cell[0]) * 24;
      Coef8 K[6];
#pragma unroll
      for (int q = 0; q < 6; ++q) K[q] = load_coef8(c + 4 * q);
#pragma unroll
      for (int q = 0; q < 6; ++q)
#pragma unroll
        for (int i = 0; i < P; ++i) F[i][q] = poly8(K[q], fx[i], fy[i], fz[i]);
    }
#pragma unroll
    for (int i = 1; i < P; ++i) {
      if (cell[i] != cell[0]) {
        const double2* c = cells + static_cast<long long>(cell[i]) * 24;
#pragma unroll
        for (int q = 0; q < 6; ++q) F[i][q] = poly8(load_coef8(c + 4 * q), fx[i], fy[i], fz[i]);
      }
    }
#endif
    if (r + 1 < k.rounds) {
#pragma unroll
      for (int i = 0; i < P; ++i) {
        double bx, by, bz;
        implicit_v(k.beta, u0[i], v0[i], w0[i], F[i], bx, by, bz);
        double tx = fma(bx, k.dcx, cx0[i]);
        double ty = fma(by, k.dcy, cy0[i]);
        double tz = fma(bz, k.dcz, cz0[i]);
        fold3(tx, ty, tz, k, bad[i]);
        cell[i] = locate_fast(k, tx, ty, tz, fx[i], fy[i], fz[i]);
      }
    } else {
      unsigned faults = 0u;
#pragma unroll
      for (int i = 0; i < P; ++i) {
        double bx, by, bz;
        implicit_v(k.beta, u0[i], v0[i], w0[i], F[i], bx, by, bz);
        // kernels.cpp:95-99
        const int p = i0 + i;
        double x1 = fma(bx, k.dt, buf[0][p]);
        double y1 = fma(by, k.dt, buf[1][p]);
        double z1 = fma(bz, k.dt, buf[2][p]);
        // common case: every coordinate stayed in [+0, hi0] -> wrap_len is the
        // identity; otherwise the exact per-axis wrap
        if ((dbits(x1) > dbits(g.ax.hi0)) | (dbits(y1) > dbits(g.ay.hi0)) |
            (dbits(z1) > dbits(g.az.hi0))) {
          x1 = wrap_exact_bits(x1, g.ax, dbits(g.ax.hi0), dbits(g.ax.hi1),
                               dbits(g.ax.lom1) & kAbs);
          y1 = wrap_exact_bits(y1, g.ay, dbits(g.ay.hi0), dbits(g.ay.hi1),
                               dbits(g.ay.lom1) & kAbs);
          z1 = wrap_exact_bits(z1, g.az, dbits(g.az.hi0), dbits(g.az.hi1),
                               dbits(g.az.lom1) & kAbs);
        }
        const double u1 = fma(2.0, bx, -u0[i]);
        const double v1 = fma(2.0, by, -v0[i]);
        const double w1 = fma(2.0, bz, -w0[i]);
        const bool fin = finite_bits(x1) && finite_bits(y1) && finite_bits(z1) &&
                         finite_bits(u1) && finite_bits(v1) && finite_bits(w1);
        if (bad[i] == 0u && fin) {
          buf[0][p] = x1; buf[1][p] = y1; buf[2][p] = z1;
          buf[3][p] = u1; buf[4][p] = v1; buf[5][p] = w1;
        } else if (p < cnt) {
          faults |= 1u << i;
        }
      }
      return faults;
    }
  }
  return 0u;
}

// ---------------------------------------------------------------------------
// FAST, one particle per thread with a register cell cache
// ---------------------------------------------------------------------------
//
// The 48 coefficients of the particle's cell stay in registers for all
// predictor rounds and are reloaded only when the predictor position moves to
// another cell (~2 % of rounds in GEM).  The reload branch contains loads
// only, so a warp whose lanes disagree never runs two evaluation paths, and
// performance does not depend on particles sharing cells (no cell sort
// needed).  L1->register traffic: 384 B per particle per cycle.
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
    implicit_v(k.beta, u0, v0, w0, F, bx, by, bz);
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
// STRICT, one particle per thread at a time with a register node cache
// ---------------------------------------------------------------------------
//
// Bit-identical to the reference: every round locates with IEEE divisions,
// computes the 8 weights and accumulates the corners in the reference's
// order with separate roundings.  The 8 corner nodes' E and B (48 doubles)
// stay in registers while the particle -- and the lane's next particles --
// remain in the same cell: a bitwise-identical reuse of values the reference
// would re-read.
template <int TILE>
__device__ __forceinline__ unsigned strict_tile_thread_p1(const DevGrid& g,
                                                          const double* __restrict__ E,
                                                          const double* __restrict__ B,
                                                          const SpeciesLaunch& sp,
                                                          double (*buf)[TILE], int p, int cnt,
                                                          CellCache& cc) {
  if (p >= cnt) return 0u;
  PState P;
  const double in[6] = {buf[0][p], buf[1][p], buf[2][p], buf[3][p], buf[4][p], buf[5][p]};
  begin(P, in);
  for (int r = 0; r < sp.rounds; ++r) {
    double wt[8];
    const int cell = strict_locate(P, g, wt);
    if (!P.ok) return 1u;  // the reference's DomainError -> NumericalFault
    if (cell != cc.cell) cache_load_strict(cc, g, E, B, cell);
    strict_round(P, cc, wt, sp.beta);
    if (r + 1 < sp.rounds) strict_predict(P, g, sp.dto2);
  }
  double out[6];
  if (!strict_finish(P, g, sp.dt, out)) return 1u;
#pragma unroll
  for (int a = 0; a < 6; ++a) buf[a][p] = out[a];
  return 0u;
}

}  // namespace b2m
