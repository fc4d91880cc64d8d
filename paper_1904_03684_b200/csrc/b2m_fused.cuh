// b2m_fused.cuh — moment deposition fused into the FAST mover's tile loop
// (deposit_moments, kernels.cpp:147-183, of the state the
// mover just produced, without re-reading the particles from HBM).
//
// After a row of 32 particles (one per lane) has been moved in the tile's
// shared-memory stage, the warp deposits rho and J of the NEW positions and
// velocities.  The per-cell sums are a small matrix product: for the particles
// of one cell,
//     D[c][m] = sum_p W[c][p] * Mom[p][m],   c = corner 0..7, m = {1, u, v, w}
// with W[c][p] = qv * wx * wy * wz the corner weight (kernels.cpp:168).  That
// is an FP64 mma.sync m8n8k4 (DMMA, the tensor-core FP64 path of sm_100a)
// over k = 4 particles at a time -- 8 per row of 32 -- with the 8x8 f64
// accumulator held in TWO registers per lane.  That register economy is the
// point: a per-lane register carry of the 32 sums (the separate deposit
// kernel's design, 64 registers) does not fit beside the mover's column cache
// at the mover's residency, and a shared-memory transpose of 32 terms per
// particle costs 512 B of shared traffic per particle.
//
// The 8 accumulator columns hold two cells: columns 0-3 the warp's CARRIED
// cell (the row's largest group; kept across rows and tiles while it stays
// the largest), columns 4-7 the row's largest other group, flushed (one FP64
// atomic per corner and moment) right after the pass.  Every row is ONE pass
// of 8 DMMAs; particles in neither cell (strays drifted out of the sorted
// order) add their 32 terms with direct atomics, all such lanes at once.  A
// row whose particles all sit in the carried cell -- the common case after a
// sort -- costs no atomics at all.
//
// Per lane, the A fragment (row c = lane/4, k = lane%4) is the corner-c weight
// of particle 4k' + lane%4, built from 6 staged factors (qv*wx*wy for the 4
// (dx, dy) corners, wz for the 2 dz) -- 1.5 KB of shared memory per warp; the
// B fragment (k = lane%4, n = lane/4) is that particle's moment n%4 (1, or its
// new u, v, w read from the tile stage), or 0 when it is not in the column
// half's cell.  Locate and weights follow the FAST deposit (1/d scaling,
// trunc, clamp, min(f, 1)); sums are in DMMA order, so the mesh matches the
// separate deposit to rounding of the sums.
#pragma once

#include "b2m_tile.cuh"

namespace b2m {

#ifndef B2M_DEP_PASSES
#define B2M_DEP_PASSES 3  // extra DMMA passes per row for groups of >= 2 beyond the first
#endif
// Staging rows are kDepRow doubles apart: with 36, the 16 (row, lane%4)
// pairs a DMMA fragment load touches fall in 16 distinct 64-bit bank pairs
// (2 * (36 r + q) mod 32 = 8 r + 2 q) -- rows of 32 would put every row on
// the same banks (4-way conflicts).
constexpr int kDepRow = 36;
#ifndef B2M_DEP_STAGE_UVW
#define B2M_DEP_STAGE_UVW 1  // fused mover: stage u, v, w too (conflict-free B rows), 96-particle tiles
#endif
// fused mover: six staged weight factors (+ u, v, w) per warp
constexpr int kDepStage = (B2M_DEP_STAGE_UVW ? 9 : 6) * kDepRow;
// fused mover tile width in rows of 32 (the staging has to fit beside the TMA
// ring at 4 blocks per SM)
constexpr int kDepPPT = B2M_DEP_STAGE_UVW ? 3 : 4;

struct DepCarry {
  double d0, d1;   // DMMA accumulator: D[lane/4][2*(lane%4) + {0, 1}]
  long long key;   // carried cell (warp-uniform), -1: none
  int ci, cj, ck;  // its indices
};

__device__ __forceinline__ void dep_reset(DepCarry& C) {
  C.d0 = C.d1 = 0.0;
  C.key = -1;
  C.ci = C.cj = C.ck = 0;
}

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Add one half of the accumulator (columns 4h..4h+3: m = 0..3 of cell
// (ci, cj, ck)) to the mesh and clear it.  Lane l holds D[c][n] for c = l/4,
// n = 2(l%4) + e; the half's values sit on the lanes with (l%4)/2 == h.
template <class G>
__device__ __forceinline__ void dep_flush_half(double& d0, double& d1, int h, int ci, int cj,
                                               int ck, const G& g, double* const* mom,
                                               int lane) {
  const int q = lane & 3;
  if ((q >> 1) != h) return;
  const int c = lane >> 2;
  const int ii = (c & 1) ? (ci + 1 == g.nx ? 0 : ci + 1) : ci;
  const int jj = (c & 2) ? (cj + 1 == g.ny ? 0 : cj + 1) : cj;
  const int kk = (c & 4) ? (ck + 1 == g.nz ? 0 : ck + 1) : ck;
  const long long node = ii + static_cast<long long>(g.nx) * (jj + static_cast<long long>(g.ny) * kk);
  const int m0 = (2 * q) & 3;  // moment of d0 (d1: m0 + 1)
  atomicAdd(mom[m0] + node, d0);
  atomicAdd(mom[m0 + 1] + node, d1);
  d0 = 0.0;
  d1 = 0.0;
}

// One pass: D[:, 0:4] += carried-cell members' terms, D[:, 4:8] += group
// `g1` members' terms (masks over the row's 32 particles).  mrow[(m - 1) *
// MS + l] is moment m (u, v, w) of the row's particle l.  W8: sw holds the 8
// corner weights (row c = corner c); else the 6 factors (rows 0-3: qv wx wy
// per (dx, dy) corner, rows 4-5: wz), multiplied here.
template <int MS, bool W8>
__device__ __forceinline__ void dep_pass(DepCarry& C, const double* sw, const double* mrow,
                                         unsigned carry_mask, unsigned g1_mask, int lane) {
  const int q = lane & 3;     // A: k column / B: k row
  const int n = lane >> 2;    // A: corner row / B: column
  const int m = n & 3;        // moment of the B column
  const unsigned mask = (n >> 2) ? g1_mask : carry_mask;
  const int cxy = n & 3, cz = n >> 2;  // A: corner n = cxy + 4 cz
  const double* mr = mrow + (m == 0 ? 0 : (m - 1) * MS);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int pl = 4 * k + q;  // particle of this fragment element, within the row
    const double a = W8 ? sw[n * kDepRow + pl]
                        : sw[cxy * kDepRow + pl] * sw[(4 + cz) * kDepRow + pl];
    double b = 0.0;
    if ((mask >> pl) & 1u) b = m == 0 ? 1.0 : mr[pl];
    dmma_8x8x4(C.d0, C.d1, a, b);
  }
}

// (px, py, pz): this lane's particle's position; mrow as in dep_pass.
// Used by the fused mover (the row in the tile stage, MS = tile width) and by
// the standalone FAST deposit (u, v, w staged per lane, MS = 32).
template <int MS, bool W8 = false, class G>
__device__ __forceinline__ void dep_row(DepCarry& C, const G& g, double qv, double* const* mom,
                                        double* sw, const double* mrow, double px, double py,
                                        double pz, bool ok, int lane) {
  constexpr unsigned FULL = 0xffffffffu;
  // FAST deposit locate (b2m_moments.cu, grid.hpp:64-82 with 1/d scaling)
  const double sx = px * g.rdx, sy = py * g.rdy, sz = pz * g.rdz;
  int i = min(__double2int_rz(sx), g.nx - 1), j = min(__double2int_rz(sy), g.ny - 1),
      k = min(__double2int_rz(sz), g.nz - 1);
  i = max(i, 0);
  j = max(j, 0);
  k = max(k, 0);
  const double fx = fmin(sx - static_cast<double>(i), 1.0);
  const double fy = fmin(sy - static_cast<double>(j), 1.0);
  const double fz = fmin(sz - static_cast<double>(k), 1.0);
  // a particle that is not deposited stages zeros (B masks it, but 0 * NaN
  // from a faulted particle's weights would still poison the accumulator)
  const double qw = ok ? qv : 0.0, ow = ok ? 1.0 : 0.0;
  const double wx0 = qw * (1.0 - fx), wx1 = qw * fx;
  const double wxy[4] = {wx0 * (1.0 - fy), wx1 * (1.0 - fy), wx0 * fy, wx1 * fy};
  const double wz[2] = {ow * (1.0 - fz), ow * fz};
  if (W8) {
#pragma unroll
    for (int c = 0; c < 8; ++c) sw[c * kDepRow + lane] = wxy[c & 3] * wz[c >> 2];
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) sw[c * kDepRow + lane] = wxy[c];
    sw[4 * kDepRow + lane] = wz[0];
    sw[5 * kDepRow + lane] = wz[1];
  }
  const long long key =
      ok ? i + static_cast<long long>(g.nx) * (j + static_cast<long long>(g.ny) * k) : -1;
  const unsigned okm = __ballot_sync(FULL, ok);
  __syncwarp();
  if (okm == 0) return;
  const unsigned grp = __match_any_sync(FULL, key);
  // the carried cell: kept while it still holds the row's largest group (or
  // ties it), else the largest group's cell takes over (ties: the group of
  // the row's last particle -- the sorted order continues there)
  const unsigned score = ok ? (static_cast<unsigned>(__popc(grp)) << 6) |
                                  (((grp >> 31) & 1u) << 5) | static_cast<unsigned>(lane)
                            : 0u;
  const unsigned best = __reduce_max_sync(FULL, score);
  const int bl = best & 31;
  const int ncar = __popc(__ballot_sync(FULL, ok && key == C.key));
  if (ncar < static_cast<int>(best >> 6)) {
    if (C.key >= 0) dep_flush_half(C.d0, C.d1, 0, C.ci, C.cj, C.ck, g, mom, lane);
    C.key = __shfl_sync(FULL, key, bl);
    C.ci = __shfl_sync(FULL, i, bl);
    C.cj = __shfl_sync(FULL, j, bl);
    C.ck = __shfl_sync(FULL, k, bl);
  }
  const unsigned carry = __ballot_sync(FULL, ok && key == C.key);
  unsigned rest = okm & ~carry;
  // the largest other group rides in columns 4-7 of the same pass
  unsigned g1 = 0u;
  int gi = 0, gj = 0, gk = 0;
  if (rest) {
    const unsigned s2 = ((rest >> lane) & 1u)
                            ? (static_cast<unsigned>(__popc(grp)) << 6) | static_cast<unsigned>(lane)
                            : 0u;
    const int leader = __reduce_max_sync(FULL, s2) & 31;
    g1 = __shfl_sync(FULL, grp, leader);
    gi = __shfl_sync(FULL, i, leader);
    gj = __shfl_sync(FULL, j, leader);
    gk = __shfl_sync(FULL, k, leader);
    rest &= ~g1;
  }
  dep_pass<MS, W8>(C, sw, mrow, carry, g1, lane);
  if (g1) dep_flush_half(C.d0, C.d1, 1, gi, gj, gk, g, mom, lane);
  // further passes for groups of >= 2 (B2M_DEP_PASSES of them, largest first)
#pragma unroll 1
  for (int x = 0; x < B2M_DEP_PASSES && rest; ++x) {
    const unsigned s2 = ((rest >> lane) & 1u)
                            ? (static_cast<unsigned>(__popc(grp & rest)) << 6) |
                                  static_cast<unsigned>(lane)
                            : 0u;
    const unsigned b2 = __reduce_max_sync(FULL, s2);
    if ((b2 >> 6) < 2) break;
    const int leader = b2 & 31;
    const unsigned gm = __shfl_sync(FULL, grp, leader);
    gi = __shfl_sync(FULL, i, leader);
    gj = __shfl_sync(FULL, j, leader);
    gk = __shfl_sync(FULL, k, leader);
    rest &= ~gm;
    dep_pass<MS, W8>(C, sw, mrow, 0u, gm, lane);
    dep_flush_half(C.d0, C.d1, 1, gi, gj, gk, g, mom, lane);
  }
  if (rest) {
    // everything else (strays drifted out of the sorted order): each lane
    // adds its own particle's 32 terms to the mesh, all lanes at once
    if ((rest >> lane) & 1u) {
      const double u = mrow[lane], v = mrow[MS + lane], w = mrow[2 * MS + lane];
      const int i1 = i + 1 == g.nx ? 0 : i + 1, j1 = j + 1 == g.ny ? 0 : j + 1,
                k1 = k + 1 == g.nz ? 0 : k + 1;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double wq = wxy[c & 3] * wz[c >> 2];
        const long long node =
            ((c & 1) ? i1 : i) +
            static_cast<long long>(g.nx) *
                (((c & 2) ? j1 : j) + static_cast<long long>(g.ny) * ((c & 4) ? k1 : k));
        atomicAdd(mom[0] + node, wq);
        atomicAdd(mom[1] + node, wq * u);
        atomicAdd(mom[2] + node, wq * v);
        atomicAdd(mom[3] + node, wq * w);
      }
    }
  }
  __syncwarp();  // the stage is rewritten by the next row
}

// ---- the pressure tensor (set 1: p_ab = sum w u_a u_b) ------------------
// Same fragments, 6 of the 8 accumulator columns: {uu, uv, uw, vv, vw, ww} of
// the members of one cell; the carried cell keeps D across rows, every other
// group of >= 2 takes a pass into the temporary E, strays add their 48 terms
// with direct atomics.
__device__ __forceinline__ void dep_pass_p(double& d0, double& d1, const double* sw,
                                           const double* mrow, int ms, unsigned mask, int lane) {
  const int q = lane & 3, n = lane >> 2;
  const int a = n < 3 ? 0 : (n < 5 ? 1 : 2);               // u_a of column n
  const int b = n < 3 ? n : (n < 5 ? n - 2 : 2);           // u_b of column n
  const double* ma = mrow + a * ms;
  const double* mb = mrow + b * ms;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int pl = 4 * k + q;
    const double av = sw[n * kDepRow + pl];
    double bv = 0.0;
    if (n < 6 && ((mask >> pl) & 1u)) bv = ma[pl] * mb[pl];
    dmma_8x8x4(d0, d1, av, bv);
  }
}

// flush columns 0-5 of a pressure accumulator to mom[4..9] at cell (ci, cj, ck)
template <class G>
__device__ __forceinline__ void dep_flush_p(double& d0, double& d1, int ci, int cj, int ck,
                                            const G& g, double* const* mom, int lane) {
  const int q = lane & 3;
  if (q < 3) {
    const int c = lane >> 2;
    const int ii = (c & 1) ? (ci + 1 == g.nx ? 0 : ci + 1) : ci;
    const int jj = (c & 2) ? (cj + 1 == g.ny ? 0 : cj + 1) : cj;
    const int kk = (c & 4) ? (ck + 1 == g.nz ? 0 : ck + 1) : ck;
    const long long node =
        ii + static_cast<long long>(g.nx) * (jj + static_cast<long long>(g.ny) * kk);
    atomicAdd(mom[4 + 2 * q] + node, d0);
    atomicAdd(mom[4 + 2 * q + 1] + node, d1);
  }
  d0 = 0.0;
  d1 = 0.0;
}

// One row of the pressure deposit; the 8 corner weights staged in sw rows
// 0-7 (W8 layout) and u, v, w in mrow (stride ms).
template <class G>
__device__ __forceinline__ void dep_row_p(DepCarry& C, const G& g, double qv, double* const* mom,
                                          double* sw, const double* mrow, int ms, double px,
                                          double py, double pz, bool ok, int lane) {
  constexpr unsigned FULL = 0xffffffffu;
  const double sx = px * g.rdx, sy = py * g.rdy, sz = pz * g.rdz;
  int i = max(min(__double2int_rz(sx), g.nx - 1), 0), j = max(min(__double2int_rz(sy), g.ny - 1), 0),
      k = max(min(__double2int_rz(sz), g.nz - 1), 0);
  const double fx = fmin(sx - static_cast<double>(i), 1.0);
  const double fy = fmin(sy - static_cast<double>(j), 1.0);
  const double fz = fmin(sz - static_cast<double>(k), 1.0);
  const double qw = ok ? qv : 0.0, ow = ok ? 1.0 : 0.0;
  const double wx0 = qw * (1.0 - fx), wx1 = qw * fx;
  const double wxy[4] = {wx0 * (1.0 - fy), wx1 * (1.0 - fy), wx0 * fy, wx1 * fy};
  const double wz[2] = {ow * (1.0 - fz), ow * fz};
#pragma unroll
  for (int c = 0; c < 8; ++c) sw[c * kDepRow + lane] = wxy[c & 3] * wz[c >> 2];
  const long long key =
      ok ? i + static_cast<long long>(g.nx) * (j + static_cast<long long>(g.ny) * k) : -1;
  const unsigned okm = __ballot_sync(FULL, ok);
  __syncwarp();
  if (okm == 0) return;
  const unsigned grp = __match_any_sync(FULL, key);
  const unsigned score = ok ? (static_cast<unsigned>(__popc(grp)) << 6) |
                                  (((grp >> 31) & 1u) << 5) | static_cast<unsigned>(lane)
                            : 0u;
  const unsigned best = __reduce_max_sync(FULL, score);
  const int bl = best & 31;
  const int ncar = __popc(__ballot_sync(FULL, ok && key == C.key));
  if (ncar < static_cast<int>(best >> 6)) {
    if (C.key >= 0) dep_flush_p(C.d0, C.d1, C.ci, C.cj, C.ck, g, mom, lane);
    C.key = __shfl_sync(FULL, key, bl);
    C.ci = __shfl_sync(FULL, i, bl);
    C.cj = __shfl_sync(FULL, j, bl);
    C.ck = __shfl_sync(FULL, k, bl);
  }
  const unsigned carry = __ballot_sync(FULL, ok && key == C.key);
  unsigned rest = okm & ~carry;
  if (carry) dep_pass_p(C.d0, C.d1, sw, mrow, ms, carry, lane);
#pragma unroll 1
  for (int x = 0; x < 1 + B2M_DEP_PASSES && rest; ++x) {
    const unsigned s2 = ((rest >> lane) & 1u)
                            ? (static_cast<unsigned>(__popc(grp & rest)) << 6) |
                                  static_cast<unsigned>(lane)
                            : 0u;
    const unsigned b2 = __reduce_max_sync(FULL, s2);
    if ((b2 >> 6) < 2) break;
    const int leader = b2 & 31;
    const unsigned gm = __shfl_sync(FULL, grp, leader);
    const int gi = __shfl_sync(FULL, i, leader), gj = __shfl_sync(FULL, j, leader),
              gk = __shfl_sync(FULL, k, leader);
    rest &= ~gm;
    double e0 = 0.0, e1 = 0.0;
    dep_pass_p(e0, e1, sw, mrow, ms, gm, lane);
    dep_flush_p(e0, e1, gi, gj, gk, g, mom, lane);
  }
  if ((rest >> lane) & 1u) {
    const double u = mrow[lane], v = mrow[ms + lane], w = mrow[2 * ms + lane];
    const double m6[6] = {u * u, u * v, u * w, v * v, v * w, w * w};
    const int i1 = i + 1 == g.nx ? 0 : i + 1, j1 = j + 1 == g.ny ? 0 : j + 1,
              k1 = k + 1 == g.nz ? 0 : k + 1;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double wq = wxy[c & 3] * wz[c >> 2];
      const long long node =
          ((c & 1) ? i1 : i) +
          static_cast<long long>(g.nx) *
              (((c & 2) ? j1 : j) + static_cast<long long>(g.ny) * ((c & 4) ? k1 : k));
#pragma unroll
      for (int m = 0; m < 6; ++m) atomicAdd(mom[4 + m] + node, wq * m6[m]);
    }
  }
  __syncwarp();
}

// ---- rho, J and the pressure tensor in one pass over the particles -------
// dep_row's set-0 machinery and dep_row_p's set-1 passes on ONE staging of
// the row (locate, weights, groups computed once): the carried cell keeps both
// accumulators (C.d0/d1 for rho and J, P.d0/d1 for the pressure), every other
// group of >= 2 takes a set-0 pass (columns 4-7) and a set-1 pass into a
// temporary, strays add their 32 + 48 terms with direct atomics.
template <class G>
__device__ __forceinline__ void dep_row_all(DepCarry& C, DepCarry& P, const G& g, double qv,
                                            double* const* mom, double* sw, const double* mrow,
                                            double px, double py, double pz, bool ok, int lane) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int MS = kDepRow;
  const double sx = px * g.rdx, sy = py * g.rdy, sz = pz * g.rdz;
  int i = max(min(__double2int_rz(sx), g.nx - 1), 0), j = max(min(__double2int_rz(sy), g.ny - 1), 0),
      k = max(min(__double2int_rz(sz), g.nz - 1), 0);
  const double fx = fmin(sx - static_cast<double>(i), 1.0);
  const double fy = fmin(sy - static_cast<double>(j), 1.0);
  const double fz = fmin(sz - static_cast<double>(k), 1.0);
  const double qw = ok ? qv : 0.0, ow = ok ? 1.0 : 0.0;
  const double wx0 = qw * (1.0 - fx), wx1 = qw * fx;
  const double wxy[4] = {wx0 * (1.0 - fy), wx1 * (1.0 - fy), wx0 * fy, wx1 * fy};
  const double wz[2] = {ow * (1.0 - fz), ow * fz};
#pragma unroll
  for (int c = 0; c < 8; ++c) sw[c * kDepRow + lane] = wxy[c & 3] * wz[c >> 2];
  const long long key =
      ok ? i + static_cast<long long>(g.nx) * (j + static_cast<long long>(g.ny) * k) : -1;
  const unsigned okm = __ballot_sync(FULL, ok);
  __syncwarp();
  if (okm == 0) return;
  const unsigned grp = __match_any_sync(FULL, key);
  const unsigned score = ok ? (static_cast<unsigned>(__popc(grp)) << 6) |
                                  (((grp >> 31) & 1u) << 5) | static_cast<unsigned>(lane)
                            : 0u;
  const unsigned best = __reduce_max_sync(FULL, score);
  const int bl = best & 31;
  const int ncar = __popc(__ballot_sync(FULL, ok && key == C.key));
  if (ncar < static_cast<int>(best >> 6)) {
    if (C.key >= 0) {
      dep_flush_half(C.d0, C.d1, 0, C.ci, C.cj, C.ck, g, mom, lane);
      dep_flush_p(P.d0, P.d1, C.ci, C.cj, C.ck, g, mom, lane);
    }
    C.key = __shfl_sync(FULL, key, bl);
    C.ci = __shfl_sync(FULL, i, bl);
    C.cj = __shfl_sync(FULL, j, bl);
    C.ck = __shfl_sync(FULL, k, bl);
  }
  const unsigned carry = __ballot_sync(FULL, ok && key == C.key);
  unsigned rest = okm & ~carry;
  unsigned g1 = 0u;
  int gi = 0, gj = 0, gk = 0;
  if (rest) {
    const unsigned s2 = ((rest >> lane) & 1u)
                            ? (static_cast<unsigned>(__popc(grp)) << 6) | static_cast<unsigned>(lane)
                            : 0u;
    const int leader = __reduce_max_sync(FULL, s2) & 31;
    g1 = __shfl_sync(FULL, grp, leader);
    gi = __shfl_sync(FULL, i, leader);
    gj = __shfl_sync(FULL, j, leader);
    gk = __shfl_sync(FULL, k, leader);
    rest &= ~g1;
  }
  dep_pass<MS, true>(C, sw, mrow, carry, g1, lane);
  dep_pass_p(P.d0, P.d1, sw, mrow, MS, carry, lane);
  if (g1) {
    dep_flush_half(C.d0, C.d1, 1, gi, gj, gk, g, mom, lane);
    double e0 = 0.0, e1 = 0.0;
    dep_pass_p(e0, e1, sw, mrow, MS, g1, lane);
    dep_flush_p(e0, e1, gi, gj, gk, g, mom, lane);
  }
#pragma unroll 1
  for (int x = 0; x < B2M_DEP_PASSES && rest; ++x) {
    const unsigned s2 = ((rest >> lane) & 1u)
                            ? (static_cast<unsigned>(__popc(grp & rest)) << 6) |
                                  static_cast<unsigned>(lane)
                            : 0u;
    const unsigned b2 = __reduce_max_sync(FULL, s2);
    if ((b2 >> 6) < 2) break;
    const int leader = b2 & 31;
    const unsigned gm = __shfl_sync(FULL, grp, leader);
    gi = __shfl_sync(FULL, i, leader);
    gj = __shfl_sync(FULL, j, leader);
    gk = __shfl_sync(FULL, k, leader);
    rest &= ~gm;
    dep_pass<MS, true>(C, sw, mrow, 0u, gm, lane);
    dep_flush_half(C.d0, C.d1, 1, gi, gj, gk, g, mom, lane);
    double e0 = 0.0, e1 = 0.0;
    dep_pass_p(e0, e1, sw, mrow, MS, gm, lane);
    dep_flush_p(e0, e1, gi, gj, gk, g, mom, lane);
  }
  if ((rest >> lane) & 1u) {
    const double u = mrow[lane], v = mrow[MS + lane], w = mrow[2 * MS + lane];
    const double m10[10] = {1.0, u, v, w, u * u, u * v, u * w, v * v, v * w, w * w};
    const int i1 = i + 1 == g.nx ? 0 : i + 1, j1 = j + 1 == g.ny ? 0 : j + 1,
              k1 = k + 1 == g.nz ? 0 : k + 1;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double wq = wxy[c & 3] * wz[c >> 2];
      const long long node =
          ((c & 1) ? i1 : i) +
          static_cast<long long>(g.nx) *
              (((c & 2) ? j1 : j) + static_cast<long long>(g.ny) * ((c & 4) ? k1 : k));
#pragma unroll
      for (int m = 0; m < 10; ++m) atomicAdd(mom[m] + node, wq * m10[m]);
    }
  }
  __syncwarp();
}

template <class G>
__device__ __forceinline__ void dep_finish(DepCarry& C, const G& g, double* const* mom,
                                           int lane) {
  if (C.key >= 0) dep_flush_half(C.d0, C.d1, 0, C.ci, C.cj, C.ck, g, mom, lane);
  C.key = -1;
}

}  // namespace b2m
