// b2m_kernels.cu — sm_100a kernels and their launchers.
//
//   warp_tile_kernel<PPT, STRICT>  the mover (b2m_tile.cuh): FAST (FMA,
//                         1e-12 contract) or STRICT (bit-identical to
//                         kernels.cpp:52-104); optionally fused with the
//                         y-slab owner scan (partition_outgoing,
//                         runtime.cpp:46-62) writing migration flags
//   field_to_cells_kernel node-layout E/B (field_mesh.hpp:13-60) -> per-cell
//                         trilinear polynomial for the FAST gather
//   bin_count / bin_scatter   the cell sort (a counting sort by cell; the CUB
//                         radix sort + gather is the low-memory fallback)
//   compact_* / fill_*       outbox compaction (scan of the mover's per-tile
//                         counts) and hole filling (merge_incoming,
//                         runtime.cpp:64-76)
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include <cub/cub.cuh>
#include <cudaTypedefs.h>

#include "b2m_internal.hpp"
#include "b2m_tile.cuh"
#include "b2m_fused.cuh"

namespace b2m {

namespace {

__device__ __forceinline__ void load6(const SpeciesLaunch& sp, unsigned long long i, double* p) {
  p[0] = sp.x[i]; p[1] = sp.y[i]; p[2] = sp.z[i];
  p[3] = sp.u[i]; p[4] = sp.v[i]; p[5] = sp.w[i];
}

__device__ __forceinline__ void store6(const SpeciesLaunch& sp, unsigned long long i,
                                       const double* p) {
  sp.x[i] = p[0]; sp.y[i] = p[1]; sp.z[i] = p[2];
  sp.u[i] = p[3]; sp.v[i] = p[4]; sp.w[i] = p[5];
}

// Migration flag of a (wrapped, finite) new y: 0 stays, 1 prev, 2 next,
// 3 another slab (CflViolation).  owner_of (runtime.cpp:39-44) evaluated
// through the exact thresholds of trunc(RN(y/dy)) -- no division.
// Integer compares of the IEEE bit patterns, branch-free (a wrapped y is
// finite and >= 0, where bit patterns order like values; the sign is cleared
// so -0 compares as +0, as `y >= 0.0` does): the FP64-pipe DSETPs and
// branches of the plain form cost ~7 % of the mover.
__device__ __forceinline__ int slab_flag(double y, const SlabLaunch& sl) {
  const unsigned long long b = dbits(y) & kAbs;
  // the common case, one unsigned range test: y in [own_lo, own_hi)
  if (b - dbits(sl.own_lo) < dbits(sl.own_hi) - dbits(sl.own_lo)) return 0;
  const bool own = (b >= dbits(sl.own_lo)) & (b < dbits(sl.own_hi));
  const bool prv = (b >= dbits(sl.prev_lo)) & (b < dbits(sl.prev_hi));
  const bool nxt = (b >= dbits(sl.next_lo)) & (b < dbits(sl.next_hi));
  return own ? 0 : (prv ? 1 : (nxt ? 2 : 3));
}

// Owner scan, per particle: does the new y stay in this rank's slab (one
// unsigned compare of the bit pattern; slab_flag's fast path)?
__device__ __forceinline__ bool stays_in_slab(double y, const SlabLaunch& sl) {
  const unsigned long long b = dbits(y) & kAbs;
  return b - dbits(sl.own_lo) < dbits(sl.own_hi) - dbits(sl.own_lo);
}

// Owner scan, per tile with a leaver: bit j of `leave` marks this lane's
// row-j particle (its new y in yrow[32 j + lane]); classify them (1 prev,
// 2 next, 3 CflViolation) and add the warp's counts per direction.
template <int P>
__device__ __forceinline__ void classify_leavers(unsigned leave, const double* yrow,
                                                 const SlabLaunch& sl, FaultWord* fault,
                                                 int species, unsigned long long base, int lane,
                                                 unsigned& n_prev, unsigned& n_next) {
#pragma unroll 1
  for (int j = 0; j < P; ++j) {
    int flag = 0;
    if ((leave >> j) & 1u) {
      flag = slab_flag(yrow[lane + 32 * j], sl);
      if (flag == 3) {
        atomicMin(&fault->cfl, fault_key(species, base + lane + 32 * j));
        flag = 0;
      }
    }
    n_prev += __popc(__ballot_sync(0xffffffffu, flag == 1));
    n_next += __popc(__ballot_sync(0xffffffffu, flag == 2));
  }
}

// The mover with warp-private TMA pipelines: every warp streams its own
// tiles of 32*P particles (kWarpStages deep) through its slice of shared
// memory with its own mbarriers -- no block-wide barrier anywhere.  One 2-D
// tensor-map box per tile carries all six SoA arrays in (and one out); the
// TMA unit zero-fills / clips partial tiles, so there is a single code path.
#ifndef B2M_ABL_STREAM_ONLY
#define B2M_ABL_STREAM_ONLY 0
#endif
#ifndef B2M_FAST_V
#define B2M_FAST_V 2   // FAST body: 2 = cached-cell frame (fast_particle_v2), 1 = round-1 kernel
#endif
#ifndef B2M_J_UNROLL
#define B2M_J_UNROLL 1
#endif
constexpr int kJUnroll = B2M_J_UNROLL;  // unroll of the per-lane particle loop
#ifndef B2M_SORT_ZFAST
#define B2M_SORT_ZFAST 1       // cell sort order: 1 = z fastest (column-contiguous), 0 = x fastest
#endif
#ifndef B2M_2D_RDISPATCH
#define B2M_2D_RDISPATCH 1     // pc_iterations dispatched once per tile (not per particle)
#endif
#ifndef B2M_2D_UNROLL
#define B2M_2D_UNROLL 2        // unroll of the column kernel's particle loop (2: 1.15 -> 1.12 ms; 4: 1.19)
#endif
constexpr int kUnroll2D = B2M_2D_UNROLL;
#ifndef B2M_3D_UNROLL
#define B2M_3D_UNROLL 1        // unroll of the general FAST kernel's particle loop
#endif
constexpr int kUnroll3D = B2M_3D_UNROLL;
#ifndef B2M_TILE_RUN_2D
#define B2M_TILE_RUN_2D 4      // column kernels: consecutive tiles per warp (1.180 -> 1.156 ms)
#endif
#ifndef B2M_TILE_RUN_3D
#define B2M_TILE_RUN_3D 1      // 3-D kernels (runs of 2 and 4 measured 1 % slower)
#endif
#ifndef B2M_2D_R45
#define B2M_2D_R45 1           // column kernel bodies specialised for pc_iterations 4 and 5 too (C5 pc 4: 43.3k -> 45.7k)
#endif
#ifndef B2M_TILE_PREFETCH
#define B2M_TILE_PREFETCH 0    // 1: L1 prefetch of the next tile's first-row columns
#endif
#ifndef B2M_COL_PREFETCH
#define B2M_COL_PREFETCH 0     // 1: L1 prefetch of the next particle's column (measured slower: 1.31 vs 1.16 ms)
#endif
#ifndef B2M_2D_PAIR
#define B2M_2D_PAIR 0          // 1: two particles per lane at a time (measured slower: spills)
#endif
#ifndef B2M_2D_MINBLOCKS
#define B2M_2D_MINBLOCKS (B2M_2D_PAIR ? 3 : 4)  // z-invariant FAST kernel: 24-double column cache
#endif
// DIM: 3 = general FAST (or STRICT), 2 = z-invariant FAST.  The two FAST
// kernels are launched back to back; each reads the field's z-invariance
// flag (zinv_check_kernel) and the one that does not apply exits at once.
// DEP: FAST only -- deposit rho and J of the moved particles in the tile loop
// (b2m_fused.cuh) into F.mom.
template <int P, bool STRICT, int DIM, bool DEP>
__global__ void __launch_bounds__(kWarpThreads, DIM == 2 ? B2M_2D_MINBLOCKS : B2M_FAST_MINBLOCKS)
    warp_tile_kernel(const __grid_constant__ TileField F, const __grid_constant__ TensorSpans S,
                     const __grid_constant__ SlabLaunch sl, unsigned long long total_tiles,
                     FaultWord* fault) {
  if (F.zvar && ((*F.zvar == 0) != (DIM == 2))) return;
  constexpr int WT = 32 * P;
  constexpr int WARPS = kWarpThreads / 32;
  extern __shared__ __align__(128) unsigned char wt_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto buf = reinterpret_cast<double(*)[6][WT]>(wt_smem) + warp * kWarpStages;
  uint64_t* bar = reinterpret_cast<uint64_t*>(wt_smem + WARPS * kWarpStages * 6 * WT * 8) +
                  warp * kWarpStages;
  double* const sw = reinterpret_cast<double*>(wt_smem + WARPS * kWarpStages * (6 * WT * 8 + 8)) +
                     warp * kDepStage;  // DEP only
  DepCarry dc;
  if (DEP) dep_reset(dc);
  const unsigned long long gw = static_cast<unsigned long long>(blockIdx.x) * WARPS + warp;
  const unsigned long long GW = static_cast<unsigned long long>(gridDim.x) * WARPS;
  // tiles round-robin over all warps of the grid in runs of kTileRun
  // consecutive tiles: at any moment the whole GPU streams one contiguous
  // window of the particle arrays (DRAM-friendly; one contiguous run per warp
  // measured 1.2x slower), and a cell-ordered species keeps the lanes' cached
  // cell from one tile of a run to the next
  constexpr unsigned long long kTileRun = DIM == 2 ? B2M_TILE_RUN_2D : B2M_TILE_RUN_3D;
  const unsigned long long t_begin = gw * kTileRun, t_end = total_tiles;
  auto t_next = [&](unsigned long long t) {
    return (t + 1) % kTileRun ? t + 1 : t + 1 + (GW - 1) * kTileRun;
  };
  const uint64_t stream_pol = policy_evict_first();

  // Tiles are visited in increasing order, so the span index only advances.
  auto advance_span = [&](int& s, unsigned long long tile) {
    while (s + 1 < S.n && tile >= S.tile_start[s + 1]) ++s;
  };
  // lane 0's load cursor: the next tile to load, its span and ring stage
  unsigned long long ld_tile = t_begin;
  int ld_span = 0, ld_stage = 0;
  auto issue = [&]() {  // lane 0
    if (ld_tile >= t_end) return;
    advance_span(ld_span, ld_tile);
    const int c0 =
        static_cast<int>(S.sp[ld_span].col0 + (ld_tile - S.tile_start[ld_span]) * WT);
    mbar_arrive_tx(&bar[ld_stage], 6 * WT * sizeof(double));
    tma_load_2d(buf[ld_stage], &S.tmap[ld_span], c0, 0, &bar[ld_stage], stream_pol);
    ld_tile = t_next(ld_tile);
    ld_stage = ld_stage + 1 == kWarpStages ? 0 : ld_stage + 1;
  };

  if (lane == 0) {
    for (int s = 0; s < kWarpStages; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
    for (int k = 0; k < kWarpStages; ++k) issue();  // fill every stage
  }
  __syncwarp();

  int s = 0, st = 0;
  uint32_t phase = 0;
  for (unsigned long long tile = t_begin, k = 0; tile < t_end; tile = t_next(tile), ++k) {
    advance_span(s, tile);
    const SpeciesLaunch& sp = S.sp[s];
    const unsigned long long off = (tile - S.tile_start[s]) * WT;
    const unsigned long long left = sp.n - off;
    const int cnt = left < static_cast<unsigned long long>(WT) ? static_cast<int>(left) : WT;
    mbar_wait(&bar[st], phase);
    unsigned n_prev = 0, n_next = 0;  // the warp's leavers in the tile (ballot totals)
    if (STRICT) {
      CellCache cc;
      cc.cell = -1;
      uint8_t* flags = S.flags[s];
      unsigned leave = 0;  // bit j: this lane's row-j particle left the slab
#pragma unroll 1
      for (int j = 0; j < P; ++j) {
        const int p = lane + 32 * j;
        // pc_iterations = 3 (the reference default) gets a fully unrolled body
        const unsigned bad =
            sp.rounds == 3
                ? strict_tile_thread_p1<WT, 3, DIM>(F.dg, F.fg, F.nodes, sp, buf[st], p, cnt, cc)
                : strict_tile_thread_p1<WT, 0, DIM>(F.dg, F.fg, F.nodes, sp, buf[st], p, cnt, cc);
        if (bad) atomicMin(&fault->numerical, fault_key(sp.species, sp.base + off + p));
        // owner scan (partition_outgoing, runtime.cpp:46-62): the stay test per
        // particle, the tile's leavers classified after its last row; the
        // compaction re-derives each leaver from its y
        if (flags && (p < cnt) & !bad & !stays_in_slab(buf[st][1][p], sl)) leave |= 1u << j;
      }
      if (flags && __any_sync(0xffffffffu, leave))
        classify_leavers<P>(leave, buf[st][1], sl, fault, sp.species, sp.base + off, lane, n_prev,
                            n_next);
    } else if (B2M_ABL_STREAM_ONLY) {
      // ablation: the tile pipeline without the mover arithmetic
      if (lane < cnt) buf[st][0][lane] += 0.0;
    } else if (DIM == 2) {
      // z-invariant field (b2m_tile.cuh): bilinear column gather
      FastCol C;
      fast_col_reset(C);
      uint8_t* flags = S.flags[s];
      unsigned leave = 0;  // bit j: this lane's row-j particle left the slab
      const double* cols = reinterpret_cast<const double*>(sp.cells);
      // per moved particle: fault record, fused deposit, migration flag
      auto after = [&](int j, unsigned bad, double y1) {
        const int p = lane + 32 * j;
        if (bad) atomicMin(&fault->numerical, fault_key(sp.species, sp.base + off + p));
        if (DEP) {
          if (B2M_DEP_STAGE_UVW) {
            // u, v, w into padded rows: the DMMA B fragments read them without
            // the tile rows' 3-way bank conflicts
            sw[6 * kDepRow + lane] = buf[st][3][p];
            sw[7 * kDepRow + lane] = buf[st][4][p];
            sw[8 * kDepRow + lane] = buf[st][5][p];
            dep_row<kDepRow>(dc, F.fg, sp.qv, F.mom, sw, sw + 6 * kDepRow, buf[st][0][p],
                             buf[st][1][p], buf[st][2][p], p < cnt && !bad, lane);
          } else {
            dep_row<WT>(dc, F.fg, sp.qv, F.mom, sw, &buf[st][3][32 * j], buf[st][0][p],
                        buf[st][1][p], buf[st][2][p], p < cnt && !bad, lane);
          }
        }
        // owner scan (partition_outgoing, runtime.cpp:46-62): the stay test per
        // particle, the tile's leavers classified after its last row (the fused
        // launch never migrates)
        if (!DEP && flags && (p < cnt) & !bad & !stays_in_slab(y1, sl)) leave |= 1u << j;
      };
      if (B2M_2D_PAIR && (P % 2) == 0) {
        // two particles per lane at a time (ILP 2, b2m_tile.cuh fast_pair_2d)
#pragma unroll 1
        for (int j = 0; j < P; j += 2) {
          const int pa = lane + 32 * j, pb = pa + 32;
          const unsigned bad2 =
              F.U.rounds == 3
                  ? fast_pair_2d<WT, 3>(F.fg, F.U, cols, buf[st], pa, pb, cnt, C)
                  : fast_pair_2d<WT, 0>(F.fg, F.U, cols, buf[st], pa, pb, cnt, C);
          after(j, bad2 & 1u, buf[st][1][pa]);
          after(j + 1, bad2 >> 1, buf[st][1][pb]);
        }
      } else if (B2M_2D_RDISPATCH && !B2M_COL_PREFETCH) {
        // pc_iterations dispatched once per tile, the particle loop inside
        auto run = [&](auto rounds_tag) {
          constexpr int R = decltype(rounds_tag)::value;
#pragma unroll (DEP ? 1 : kUnroll2D)
          for (int j = 0; j < P; ++j) {
            const int p = lane + 32 * j;
            if (B2M_TILE_PREFETCH && j == P - 2) {
              // the next tile's first-row columns into L1 once its load landed
              const int nst = st + 1 == kWarpStages ? 0 : st + 1;
              const uint32_t nph = nst == 0 ? phase ^ 1u : phase;
              const unsigned long long nt = t_next(tile);
              if (nt < t_end && mbar_test(&bar[nst], nph)) {
                int s2 = s;
                advance_span(s2, nt);
                col_prefetch(F.fg, reinterpret_cast<const double*>(S.sp[s2].cells), C,
                             buf[nst][0][lane], buf[nst][1][lane]);
              }
            }
            double y1 = 0.0;
            const unsigned bad = fast_particle_2d<WT, R, !DEP && B2M_2D_PRED_RELOAD>(
                F.fg, F.U, cols, buf[st], p, cnt, C, &y1);
            after(j, bad, y1);
          }
        };
        if (F.U.rounds == 3) run(std::integral_constant<int, 3>{});
#if B2M_2D_R45
        else if (!DEP && F.U.rounds == 4) run(std::integral_constant<int, 4>{});
        else if (!DEP && F.U.rounds == 5) run(std::integral_constant<int, 5>{});
#endif
        else run(std::integral_constant<int, 0>{});
      } else {
#pragma unroll 1
        for (int j = 0; j < P; ++j) {
          const int p = lane + 32 * j;
          if (B2M_COL_PREFETCH) {
            // the column of this lane's next particle: the next row of this
            // tile, or the first row of the next tile once its load landed
            if (j + 1 < P) {
              col_prefetch(F.fg, cols, C, buf[st][0][p + 32], buf[st][1][p + 32]);
            } else {
              const int nst = st + 1 == kWarpStages ? 0 : st + 1;
              const uint32_t nph = nst == 0 ? phase ^ 1u : phase;
              const unsigned long long nt = t_next(tile);
              if (nt < t_end && mbar_test(&bar[nst], nph)) {
                int s2 = s;
                advance_span(s2, nt);
                col_prefetch(F.fg, reinterpret_cast<const double*>(S.sp[s2].cells), C,
                             buf[nst][0][lane], buf[nst][1][lane]);
              }
            }
          }
          double y1 = 0.0;
          const unsigned bad =
              F.U.rounds == 3 ? fast_particle_2d<WT, 3>(F.fg, F.U, cols, buf[st], p, cnt, C, &y1)
                              : fast_particle_2d<WT, 0>(F.fg, F.U, cols, buf[st], p, cnt, C, &y1);
          after(j, bad, y1);
        }
      }
      if (!DEP && flags && __any_sync(0xffffffffu, leave))
        classify_leavers<P>(leave, buf[st][1], sl, fault, sp.species, sp.base + off, lane, n_prev,
                            n_next);
    } else if (B2M_FAST_V == 2) {
      // FAST v2 (b2m_tile.cuh): fractions relative to the lane's cached cell
      FastCell C;
      fast_cell_reset(C);
      uint8_t* flags = S.flags[s];
      unsigned leave = 0;  // bit j: this lane's row-j particle left the slab
      const double2* cells = sp.cells;
      auto run3 = [&](auto rounds_tag) {
      constexpr int R = decltype(rounds_tag)::value;
#pragma unroll (kUnroll3D)
      for (int j = 0; j < P; ++j) {
        const int p = lane + 32 * j;
        const unsigned bad = fast_particle_v2<WT, R, !DEP && B2M_3D_PRED_RELOAD>(F.fg, F.U, cells,
                                                                                buf[st], p, cnt, C);
        if (bad) atomicMin(&fault->numerical, fault_key(sp.species, sp.base + off + p));
        if (DEP) {
          if (B2M_DEP_STAGE_UVW) {
            // u, v, w into padded rows: the DMMA B fragments read them without
            // the tile rows' 3-way bank conflicts
            sw[6 * kDepRow + lane] = buf[st][3][p];
            sw[7 * kDepRow + lane] = buf[st][4][p];
            sw[8 * kDepRow + lane] = buf[st][5][p];
            dep_row<kDepRow>(dc, F.fg, sp.qv, F.mom, sw, sw + 6 * kDepRow, buf[st][0][p],
                             buf[st][1][p], buf[st][2][p], p < cnt && !bad, lane);
          } else {
            dep_row<WT>(dc, F.fg, sp.qv, F.mom, sw, &buf[st][3][32 * j], buf[st][0][p],
                        buf[st][1][p], buf[st][2][p], p < cnt && !bad, lane);
          }
        }
        // owner scan (partition_outgoing, runtime.cpp:46-62): the stay test per
        // particle, the tile's leavers classified after its last row
        if (!DEP && flags && (p < cnt) & !bad & !stays_in_slab(buf[st][1][p], sl))
          leave |= 1u << j;
      }
      };
      // pc_iterations dispatched once per tile
      if (F.U.rounds == 3) run3(std::integral_constant<int, 3>{});
      else run3(std::integral_constant<int, 0>{});
      if (!DEP && flags && __any_sync(0xffffffffu, leave))
        classify_leavers<P>(leave, buf[st][1], sl, fault, sp.species, sp.base + off, lane, n_prev,
                            n_next);
    } else {
      const FastConst kc = make_const(F.fg, sp);
      // particles lane + 32*j, j < P, one after the other, sharing the
      // register cell cache (consecutive particles of a cell-ordered species
      // mostly share a cell, so the cache is usually filled once per tile);
      // consecutive lanes read consecutive shared-memory words
      Coef8 K[6];
      int kcell = -1;
      uint8_t* flags = S.flags[s];
#pragma unroll (kJUnroll)
      for (int j = 0; j < P; ++j) {
        const int p = lane + 32 * j;
        // pc_iterations = 3 (the reference default) gets a fully unrolled body
        const unsigned bad =
            kc.rounds == 3
                ? fast_tile_thread_p1<WT, 3>(F.fg, sp.cells, kc, buf[st], p, cnt, K, kcell)
                : fast_tile_thread_p1<WT, 0>(F.fg, sp.cells, kc, buf[st], p, cnt, K, kcell);
        if (bad) atomicMin(&fault->numerical, fault_key(sp.species, sp.base + off + p));
        if (flags) {
          // migration scan fused into the mover (partition_outgoing,
          // runtime.cpp:46-62): 0 stay, 1 prev, 2 next; a non-neighbour
          // destination records a CflViolation
          int flag = 0;
          if (p < cnt && !bad) {
            flag = slab_flag(buf[st][1][p], sl);
            if (flag == 3) {
              atomicMin(&fault->cfl, fault_key(sp.species, sp.base + off + p));
              flag = 0;
            }
          }
          n_prev += __popc(__ballot_sync(0xffffffffu, flag == 1));
          n_next += __popc(__ballot_sync(0xffffffffu, flag == 2));
        }
      }
    }
    if (S.tcnt[s]) {  // per-tile leaver counts (warp totals): the compaction's scan input
      if (lane == 0)
        S.tcnt[s][tile - S.tile_start[s]] =
            (static_cast<unsigned long long>(n_next) << 32) | n_prev;
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(&S.tmap[s], static_cast<int>(sp.col0 + off), 0, buf[st], stream_pol);
      tma_commit();
      if (kWarpStages >= 3) {
        // refill the stage of tile k-1, whose store was issued a whole tile
        // ago (its shared-memory read is long done): no wait on this store
        if (k > 0) {
          tma_wait_read<1>();
          issue();  // tile k-1+stages into the stage of tile k-1
        }
      } else {
        tma_wait_read<0>();  // two stages: this tile's stage is the next refill
        issue();             // tile k+2 into it
      }
    }
    __syncwarp();
    if (++st == kWarpStages) {
      st = 0;
      phase ^= 1u;
    }
  }
  if (DEP) dep_finish(dc, F.fg, F.mom, lane);
  if (lane == 0) tma_wait_all();
}

// STRICT: per cell, the 8 corner nodes' (Ex, Ey, Ez, Bx, By, Bz) in corner
// order c = di + 2dj + 4dk (kernels.cpp:10-22) -- 48 doubles the mover's cell
// cache loads with twelve 256-bit loads.  Thread = (cell, corner).
__global__ void strict_nodes_kernel(int nx, int ny, int nz, const double* __restrict__ E,
                                    const double* __restrict__ B, double* __restrict__ out) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long ncell = static_cast<long long>(nx) * ny * nz;
  if (t >= 8 * ncell) return;
  const long long cell = t / 8;
  const int c = static_cast<int>(t % 8);
  const int i = static_cast<int>(cell % nx);
  const int j = static_cast<int>((cell / nx) % ny);
  const int k = static_cast<int>(cell / (static_cast<long long>(nx) * ny));
  const long long n = 3 * ((i + (c & 1)) + static_cast<long long>(nx + 1) *
                                               ((j + ((c >> 1) & 1)) +
                                                static_cast<long long>(ny + 1) * (k + (c >> 2))));
  double* o = out + 6 * t;
  o[0] = __ldg(E + n); o[1] = __ldg(E + n + 1); o[2] = __ldg(E + n + 2);
  o[3] = __ldg(B + n); o[4] = __ldg(B + n + 1); o[5] = __ldg(B + n + 2);
}

// Per-cell trilinear polynomials of (beta*E, beta*B) for up to kMaxTables
// species at once (one read of the field).  Thread = (cell, component q):
// the 8 corner values -> 4 {P, Q} pairs (b2m_mover.cuh, kCellDoubles), so
// consecutive threads write consecutive 64-byte pieces of the tables.
struct CellTables {
  double2* out[kMaxTables];
  double scale[kMaxTables];
  int n;
};

// Is the field z-invariant: every node plane k >= 1 of E and B equal to plane
// 0 bit for bit?  *flag must be 0 on entry; any difference sets it.
__global__ void zinv_check_kernel(long long plane, long long nodes, const double* __restrict__ E,
                                  const double* __restrict__ B, int* flag) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= 3 * (nodes - plane)) return;
  const long long a = 3 * plane + t, b = t % (3 * plane);
  const bool same = __double_as_longlong(E[a]) == __double_as_longlong(E[b]) &&
                    __double_as_longlong(B[a]) == __double_as_longlong(B[b]);
  if (!same) *flag = 1;
}

// z-invariant field: the bilinear column polynomial of plane k = 0 per x-y
// column (the same P values as the 3-D table below, whose Q are all exactly
// zero).  Thread = (column, component q); exits at once for a z-varying field.
__global__ void field_to_cols_kernel(int nx, int ny, const double* __restrict__ E,
                                     const double* __restrict__ B,
                                     const __grid_constant__ CellTables T,
                                     const int* __restrict__ zvar) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= 6LL * nx * ny || *zvar != 0) return;
  const long long col = t / 6;
  const int q = static_cast<int>(t % 6);
  const int i = static_cast<int>(col % nx), j = static_cast<int>(col / nx);
  const long long sx = nx + 1;
  const double* F = (q < 3 ? E : B) + q % 3;
  const double f00 = __ldg(F + 3 * (i + sx * j)), f10 = __ldg(F + 3 * (i + 1 + sx * j));
  const double f01 = __ldg(F + 3 * (i + sx * (j + 1))), f11 = __ldg(F + 3 * (i + 1 + sx * (j + 1)));
  for (int m = 0; m < T.n; ++m) {
    const double c = T.scale[m];
    const double g00 = c * f00, g10 = c * f10, g01 = c * f01, g11 = c * f11;
    double* out = reinterpret_cast<double*>(T.out[m]) + col * 24 + 4 * q;
    reinterpret_cast<double4*>(out)[0] =
        make_double4(g00, g01 - g00, g10 - g00, (g11 - g10) - (g01 - g00));
  }
}

// The general per-cell tables; a grid-stride loop over (cell, q), so for a
// z-invariant field (zvar set and 0) the whole grid exits after one load.
__global__ void field_to_cells_kernel(int nx, int ny, int nz, const double* __restrict__ E,
                                      const double* __restrict__ B,
                                      const __grid_constant__ CellTables T,
                                      const int* __restrict__ zvar) {
  if (zvar && *zvar == 0) return;
  const long long ncell = static_cast<long long>(nx) * ny * nz;
  const long long sx = nx + 1, sy = ny + 1;
  for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < 6 * ncell;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long cell = t / 6;
    const int q = static_cast<int>(t % 6);
    const int i = static_cast<int>(cell % nx);
    const int j = static_cast<int>((cell / nx) % ny);
    const int k = static_cast<int>(cell / (static_cast<long long>(nx) * ny));
    const double* F = (q < 3 ? E : B) + q % 3;
    auto f = [&](int di, int dj, int dk) {
      return __ldg(F + 3 * ((i + di) + sx * ((j + dj) + sy * (k + dk))));
    };
    // f<di dj dk>
    const double f000 = f(0, 0, 0), f100 = f(1, 0, 0), f010 = f(0, 1, 0), f110 = f(1, 1, 0);
    const double f001 = f(0, 0, 1), f101 = f(1, 0, 1), f011 = f(0, 1, 1), f111 = f(1, 1, 1);
    for (int m = 0; m < T.n; ++m) {
      const double c = T.scale[m];
      const double g000 = c * f000, g100 = c * f100, g010 = c * f010, g110 = c * f110;
      const double g001 = c * f001, g101 = c * f101, g011 = c * f011, g111 = c * f111;
      const double d00 = g001 - g000, d10 = g101 - g100, d01 = g011 - g010, d11 = g111 - g110;
      double2* out = T.out[m] + cell * (kCellDoubles / 2) + 4 * q;
      out[0] = make_double2(g000, d00);
      out[1] = make_double2(g010 - g000, d01 - d00);
      out[2] = make_double2(g100 - g000, d10 - d00);
      out[3] = make_double2((g110 - g100) - (g010 - g000), (d11 - d10) - (d01 - d00));
    }
  }
}

__global__ void fault_reset_kernel(FaultWord* f) {
  f->numerical = ~0ull;
  f->cfl = ~0ull;
  f->domain = ~0ull;
}

__global__ void cell_keys_kernel(const __grid_constant__ FastGrid g, const double* __restrict__ x,
                                 const double* __restrict__ y, const double* __restrict__ z,
                                 unsigned long long n, uint32_t* keys, uint32_t* vals) {
  const unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double cx = x[i] * g.rdx, cy = y[i] * g.rdy, cz = z[i] * g.rdz;
  uint32_t key = static_cast<uint32_t>(static_cast<long long>(g.nx) * g.ny * g.nz);
  if (cx >= 0.0 && cx <= g.nxd && cy >= 0.0 && cy <= g.nyd && cz >= 0.0 && cz <= g.nzd) {
    const int ci = min(__double2int_rz(cx), g.nx - 1);
    const int cj = min(__double2int_rz(cy), g.ny - 1);
    const int ck = min(__double2int_rz(cz), g.nz - 1);
    key = B2M_SORT_ZFAST ? static_cast<uint32_t>(ck + g.nz * (ci + g.nx * cj))  // see cell_key
                         : static_cast<uint32_t>(ci + g.nx * (cj + g.ny * ck));
  }
  keys[i] = key;
  vals[i] = static_cast<uint32_t>(i);
}

// ---- counting sort by cell (b2m_sort_species) -----------------------------
// Cell order is all the mover needs, not a stable order, so the sort is a
// counting sort: (1) the cell key of every particle and per-cell counts,
// (2) an exclusive scan of the counts, (3) every particle written straight to
// its cell's segment of the ping-pong arrays.  Both atomic passes aggregate
// over the lanes of a warp that share a cell (__match_any_sync), so a
// cell-ordered species costs a few atomics per warp.  One read of the
// positions, one read and one write of the six arrays: HBM-bound.
//
// Sort order: z fastest, then x, then y -- key k + nz*(i + nx*j).  Any cell
// order keeps a cell's particles together (all the deposit and the 3-D cell
// cache need); this one also keeps an x-y column's nz cells together, so the
// z-invariant mover's column cache (b2m_tile.cuh) meets a new column once per
// column (~7000 particles per species at C2) instead of once per cell (~216):
// with cells in the reference's index order (x fastest) a lane's next
// particle changed column ~15 % of the time and nearly every warp took the
// reload path.  y slowest also groups a y-slab's particles.
__device__ __forceinline__ uint32_t cell_key(const FastGrid& g, double x, double y, double z) {
  const double cx = x * g.rdx, cy = y * g.rdy, cz = z * g.rdz;
  uint32_t key = static_cast<uint32_t>(static_cast<long long>(g.nx) * g.ny * g.nz);
  if (cx >= 0.0 && cx <= g.nxd && cy >= 0.0 && cy <= g.nyd && cz >= 0.0 && cz <= g.nzd) {
    const int ci = min(__double2int_rz(cx), g.nx - 1);
    const int cj = min(__double2int_rz(cy), g.ny - 1);
    const int ck = min(__double2int_rz(cz), g.nz - 1);
    key = B2M_SORT_ZFAST ? static_cast<uint32_t>(ck + g.nz * (ci + g.nx * cj))
                         : static_cast<uint32_t>(ci + g.nx * (cj + g.ny * ck));
  }
  return key;
}

__global__ void bin_count_kernel(const __grid_constant__ FastGrid g, const double* __restrict__ x,
                                 const double* __restrict__ y, const double* __restrict__ z,
                                 unsigned long long n, uint32_t* __restrict__ keys,
                                 uint32_t* __restrict__ count) {
  const unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const unsigned active = __ballot_sync(0xffffffffu, i < n);
  if (i >= n) return;
  const uint32_t key = cell_key(g, x[i], y[i], z[i]);
  keys[i] = key;
  const unsigned peers = __match_any_sync(active, key);
  if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&count[key], __popc(peers));
}

struct Ptr6 {
  const double* in[6];
  double* out[6];
};

__global__ void bin_scatter_kernel(const __grid_constant__ Ptr6 P, const uint32_t* __restrict__ keys,
                                   unsigned long long n, const uint32_t* __restrict__ offs,
                                   uint32_t* __restrict__ cursor) {
  const unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const unsigned active = __ballot_sync(0xffffffffu, i < n);
  if (i >= n) return;
  const int lane = threadIdx.x & 31;
  const uint32_t key = keys[i];
  const unsigned peers = __match_any_sync(active, key);
  const int leader = __ffs(peers) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(&cursor[key], __popc(peers));
  base = __shfl_sync(peers, base, leader);
  const uint32_t slot = offs[key] + base + __popc(peers & ((1u << lane) - 1u));
#pragma unroll
  for (int a = 0; a < 6; ++a) P.out[a][slot] = __ldcs(P.in[a] + i);
}

__global__ void gather_kernel(const double* __restrict__ in, const uint32_t* __restrict__ perm,
                              unsigned long long n, double* __restrict__ out) {
  const unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[perm[i]];
}

// ---- migration ------------------------------------------------------------

// ---- migration compaction (partition_outgoing, runtime.cpp:46-62) ---------
// The mover wrote a flag per particle (0 stay, 1 prev, 2 next) and, per
// 128-particle tile, the packed counts (next << 32 | prev).  An exclusive scan
// of the packed counts gives every tile its outbox offsets (prev, next) and
// hole offset (prev + next); one block per tile then writes its leavers in
// scan order.  Tiles without leavers (most of them) return after one load.
constexpr int kTileParticles = 32 * B2M_FAST_PPT;

__global__ void fill_in_kernel(const __grid_constant__ SpeciesLaunch sp,
                               const unsigned long long* __restrict__ holes,
                               unsigned long long n_holes, const double* __restrict__ in_recs,
                               unsigned long long n_in) {
  const unsigned long long t = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n_in) return;
  const unsigned long long dst = t < n_holes ? holes[t] : sp.n + (t - n_holes);
  double p[6];
#pragma unroll
  for (int a = 0; a < 6; ++a) p[a] = in_recs[6 * t + a];
  store6(sp, dst, p);
}

// Phase C (m < L): the k-th surviving particle of [n', n) fills the k-th
// remaining hole below n'.  Single CTA; the tail is ~L-m particles long.
__global__ void __launch_bounds__(1024)
    fill_tail_kernel(const __grid_constant__ SpeciesLaunch sp,
                     const unsigned long long* __restrict__ holes, unsigned long long n_in,
                     const __grid_constant__ SlabLaunch sl, unsigned long long new_n) {
  typedef cub::BlockScan<int, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (unsigned long long base = new_n; base < sp.n; base += 1024) {
    const unsigned long long i = base + threadIdx.x;
    // tail positions still hold their own moved particles (arrivals only
    // fill holes below new_n): a leaver by the owner scan of its y
    int f = i < sp.n ? slab_flag(sp.y[i], sl) : 1;
    if (f == 3) f = 0;
    const int keep = (i < sp.n && f == 0) ? 1 : 0;
    int rank, total;
    Scan(tmp).ExclusiveSum(keep, rank, total);
    if (keep) {
      const unsigned long long dst = holes[n_in + carry + rank];
      double p[6];
      load6(sp, i, p);
      store6(sp, dst, p);
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
}

}  // namespace

int device_sms() {
  static const int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 1;
  }();
  return sms;
}

namespace {

unsigned grid_for(uint64_t n, int threads) {
  return static_cast<unsigned>((n + threads - 1) / threads);
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

namespace {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

bool encode_species_map(CUtensorMap* map, const SpeciesLaunch& sp, int box_cols) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  // the species block starts at x - col0; rows are the six arrays
  const double* base = sp.x - sp.col0;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(sp.col0 + sp.n), 6};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(sp.stride * sizeof(double))};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), 6};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool STRICT, int DIM, bool DEP = false>
bool launch_warp_tiles(const TileField& F, const SpeciesLaunch* sp, int n_spans, FaultWord* fault,
                       cudaStream_t st, const SlabLaunch* sl, uint8_t* const* flags,
                       unsigned long long* const* tcnt) {
  constexpr int P = DEP ? kDepPPT : B2M_FAST_PPT;
  constexpr int WT = 32 * P;
  constexpr int smem = (kWarpThreads / 32) * (kWarpStages * (6 * WT * 8 + 8) +
                                              (DEP ? kDepStage * 8 : 0));
  static_assert(smem <= 227 * 1024, "warp tiles exceed shared memory");
  // resident grid, computed once (thread-safe static initialisation: engines
  // on several host threads may launch concurrently)
  static const int grid_cap = [] {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(warp_tile_kernel<P, STRICT, DIM, DEP>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, warp_tile_kernel<P, STRICT, DIM, DEP>,
                                                  kWarpThreads, smem);
    int cap = sms * (per_sm > 0 ? per_sm : 1);
    // diagnostics: B2M_BLOCKS_PER_SM=k runs the persistent grid with k blocks per SM
    if (const char* e = std::getenv("B2M_BLOCKS_PER_SM")) {
      const int k = std::atoi(e);
      if (k > 0 && k < per_sm) cap = sms * k;
    }
    cudaGetLastError();  // a failed query above falls back, it is not the caller's error
    return cap;
  }();
  // FAST launches share dt / pc_iterations across their spans (FastUniform):
  // a batch whose species differ there is launched in runs of equal values
  auto same_uniform = [&](int a, int b) {
    return sp[a].dt == sp[b].dt && sp[a].rounds == sp[b].rounds &&
           sp[a].dto2_cell[0] == sp[b].dto2_cell[0] && sp[a].dto2_cell[1] == sp[b].dto2_cell[1] &&
           sp[a].dto2_cell[2] == sp[b].dto2_cell[2];
  };
  for (int base = 0; base < n_spans;) {
    TensorSpans S{};
    unsigned long long tiles = 0;
    TileField FL = F;
    FL.U.dt = sp[base].dt;
    FL.U.dc[0] = sp[base].dto2_cell[0];
    FL.U.dc[1] = sp[base].dto2_cell[1];
    FL.U.dc[2] = sp[base].dto2_cell[2];
    FL.U.rounds = sp[base].rounds;
    int s = base;
    for (; s < n_spans && S.n < kMaxTileSpans && (STRICT || same_uniform(base, s)); ++s) {
      if (sp[s].n == 0) continue;
      if (sp[s].col0 + sp[s].n > 0x7fffffffull) return false;  // 32-bit TMA coordinates
      S.sp[S.n] = sp[s];
      S.flags[S.n] = flags ? flags[s] : nullptr;
      S.tcnt[S.n] = flags && tcnt ? tcnt[s] : nullptr;
      if (!encode_species_map(&S.tmap[S.n], sp[s], WT)) return false;
      S.tile_start[S.n] = tiles;
      tiles += (sp[s].n + WT - 1) / WT;
      ++S.n;
    }
    base = s;
    S.tile_start[S.n] = tiles;
    if (S.n == 0) continue;
    constexpr unsigned long long WPB = kWarpThreads / 32;
    const unsigned long long blocks = (tiles + WPB - 1) / WPB;
    const int grid = static_cast<int>(blocks < static_cast<unsigned long long>(grid_cap) ? blocks : grid_cap);
    warp_tile_kernel<P, STRICT, DIM, DEP><<<grid, kWarpThreads, smem, st>>>(FL, S, sl ? *sl : SlabLaunch{},
                                                                   tiles, fault);
    note_launch();
  }
  return true;
}

bool launch_move_fast(const FastGrid& g, const SpeciesLaunch* sp, int n_spans, FaultWord* fault,
                      cudaStream_t st, const SlabLaunch* sl, uint8_t* const* flags,
                      unsigned long long* const* tcnt, const int* zvar, double* const* mom) {
  TileField F{};
  F.fg = g;
  F.zvar = zvar;
  if (mom) {
    // the fused mover + deposit (b2m_move_deposit_all) never migrates: its
    // kernels carry no owner scan
    if (flags) return false;
    for (int m = 0; m < 4; ++m) F.mom[m] = mom[m];
    if (zvar && !launch_warp_tiles<false, 2, true>(F, sp, n_spans, fault, st, sl, nullptr, nullptr))
      return false;
    return launch_warp_tiles<false, 3, true>(F, sp, n_spans, fault, st, sl, nullptr, nullptr);
  }
  // both FAST kernels; the one the field's z-invariance flag rules out exits
  // at its first instruction (no host round trip to decide)
  if (zvar && !launch_warp_tiles<false, 2>(F, sp, n_spans, fault, st, sl, flags, tcnt))
    return false;
  return launch_warp_tiles<false, 3>(F, sp, n_spans, fault, st, sl, flags, tcnt);
}

bool launch_move_strict_tiles(const DevGrid& g, const FastGrid& fg, const double* nodes,
                              const SpeciesLaunch* sp, int n_spans, FaultWord* fault,
                              cudaStream_t st, const SlabLaunch* sl, uint8_t* const* flags,
                              unsigned long long* const* tcnt, const int* zvar) {
  TileField F{};
  F.dg = g;
  F.fg = fg;  // wrap thresholds (WrapAxis)
  F.nodes = nodes;
  F.zvar = zvar;
  // as FAST: the column kernel for a z-invariant field, the general one else
  if (zvar && !launch_warp_tiles<true, 2>(F, sp, n_spans, fault, st, sl, flags, tcnt))
    return false;
  return launch_warp_tiles<true, 3>(F, sp, n_spans, fault, st, sl, flags, tcnt);
}

void launch_zinv_check(int nx, int ny, int nz, const double* E, const double* B, int* zvar,
                       cudaStream_t st) {
  const long long plane = static_cast<long long>(nx + 1) * (ny + 1);
  const long long nodes = plane * (nz + 1);
  cudaMemsetAsync(zvar, 0, sizeof(int), st);
  zinv_check_kernel<<<grid_for(3 * (nodes - plane), 256), 256, 0, st>>>(plane, nodes, E, B, zvar);
  note_launch();
}

void launch_strict_nodes(int nx, int ny, int nz, const double* E, const double* B, double* out,
                         cudaStream_t st) {
  const long long ncell = static_cast<long long>(nx) * ny * nz;
  strict_nodes_kernel<<<grid_for(8 * ncell, 256), 256, 0, st>>>(nx, ny, nz, E, B, out);
  note_launch();
}

void launch_field_to_cells(int nx, int ny, int nz, const double* E, const double* B,
                           const double* scale, double2* const* tables, int n_tables,
                           cudaStream_t st, int* zvar) {
  const long long ncell = static_cast<long long>(nx) * ny * nz;
  if (zvar) launch_zinv_check(nx, ny, nz, E, B, zvar, st);
  for (int base = 0; base < n_tables; base += kMaxTables) {
    CellTables T{};
    for (T.n = 0; T.n < kMaxTables && base + T.n < n_tables; ++T.n) {
      T.out[T.n] = tables[base + T.n];
      T.scale[T.n] = scale[base + T.n];
    }
    if (zvar) {
      field_to_cols_kernel<<<grid_for(6LL * nx * ny, 192), 192, 0, st>>>(nx, ny, E, B, T, zvar);
      note_launch();
    }
    const long long blocks = std::min<long long>(grid_for(6 * ncell, 192), 8LL * device_sms());
    field_to_cells_kernel<<<static_cast<int>(blocks), 192, 0, st>>>(nx, ny, nz, E, B, T, zvar);
    note_launch();
  }
}

void launch_fault_reset(FaultWord* fault, cudaStream_t st) {
  fault_reset_kernel<<<1, 1, 0, st>>>(fault);
  note_launch();
}

size_t bin_scan_temp_bytes(uint64_t n_bins) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<const uint32_t*>(nullptr),
                                static_cast<uint32_t*>(nullptr), n_bins);
  return bytes;
}

void launch_bin_sort(const FastGrid& g, double* const* in, double* const* out, uint64_t n,
                     uint32_t* keys, uint32_t* count, uint32_t* offs, void* temp,
                     size_t temp_bytes, cudaStream_t st) {
  if (n == 0) return;
  const uint64_t n_bins = static_cast<uint64_t>(g.nx) * g.ny * g.nz + 1;  // + out-of-domain bin
  cudaMemsetAsync(count, 0, n_bins * sizeof(uint32_t), st);
  bin_count_kernel<<<grid_for(n, 256), 256, 0, st>>>(g, in[0], in[1], in[2], n, keys, count);
  note_launch();
  size_t b = temp_bytes;
  cub::DeviceScan::ExclusiveSum(temp, b, count, offs, n_bins, st);
  note_launch();
  cudaMemsetAsync(count, 0, n_bins * sizeof(uint32_t), st);  // reused as the cursors
  Ptr6 P;
  for (int a = 0; a < 6; ++a) {
    P.in[a] = in[a];
    P.out[a] = out[a];
  }
  bin_scatter_kernel<<<grid_for(n, 256), 256, 0, st>>>(P, keys, n, offs, count);
  note_launch();
}


void launch_cell_keys(const FastGrid& g, const double* x, const double* y, const double* z,
                      uint64_t n, uint32_t* keys, uint32_t* vals, cudaStream_t st) {
  if (n == 0) return;
  cell_keys_kernel<<<grid_for(n, 256), 256, 0, st>>>(g, x, y, z, n, keys, vals);
  note_launch();
}

void launch_gather(const double* in, const uint32_t* perm, uint64_t n, double* out,
                   cudaStream_t st) {
  if (n == 0) return;
  gather_kernel<<<grid_for(n, 256), 256, 0, st>>>(in, perm, n, out);
  note_launch();
}

size_t sort_temp_bytes(uint64_t n, int key_bits) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr),
                                  static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), static_cast<int>(n), 0,
                                  key_bits);
  return bytes;
}

void launch_sort_pairs(void* temp, size_t temp_bytes, const uint32_t* kin, uint32_t* kout,
                       const uint32_t* vin, uint32_t* vout, uint64_t n, int key_bits,
                       cudaStream_t st) {
  if (n == 0) return;
  cub::DeviceRadixSort::SortPairs(temp, temp_bytes, kin, kout, vin, vout, static_cast<int>(n), 0,
                                  key_bits, st);
  note_launch((key_bits + 7) / 8 + 1);
}

// Native slab world (b2m_world_step): the per-species outbox counts
// (totals[s] = {prev, next, holes}) packed into one [2][ns] send buffer for
// the counts exchange, all zero when this rank faulted or an outbox
// overflowed -- a faulted rank keeps running the protocol with empty
// outboxes (runtime.cpp:283-288 drops it from the barrier instead).
__global__ void pack_counts_kernel(const unsigned long long* const* totals, int ns,
                                   const unsigned long long* cap, const FaultWord* fault,
                                   unsigned long long* out) {
  if (threadIdx.x != 0) return;
  bool bad = fault->numerical != ~0ull || fault->cfl != ~0ull || fault->domain != ~0ull;
  for (int s = 0; s < ns; ++s) {
    const unsigned long long p = totals[s][0], n = totals[s][1];
    bad = bad || p > cap[s] || n > cap[s];
    out[s] = p;
    out[ns + s] = n;
  }
  if (bad)
    for (int i = 0; i < 2 * ns; ++i) out[i] = 0;
}

void launch_pack_counts(const unsigned long long* const* totals, int ns,
                        const unsigned long long* cap, const FaultWord* fault,
                        unsigned long long* out, cudaStream_t st) {
  pack_counts_kernel<<<1, 32, 0, st>>>(totals, ns, cap, fault, out);
  note_launch();
}

// The rank's contribution to the step's all-reduce, {count after the merge,
// failed}: failed when the rank was already failing (own_bad), the mover
// faulted, an outbox overflowed, or the arrivals the counts round announced
// would overflow the exchange buffer or the species' capacity -- the same
// tests the host then repeats for its typed error (world_counts), so every
// failure a rank can see before the records round is in the sum every rank
// reads at the same sync.
__global__ void world_verdict_kernel(const unsigned long long* const* totals, int ns,
                                     const unsigned long long* cap, const FaultWord* fault,
                                     const unsigned long long* cnt_recv,
                                     const unsigned long long* vin, int own_bad, long long* red) {
  if (threadIdx.x != 0) return;
  bool bad = own_bad != 0 || fault->numerical != ~0ull || fault->cfl != ~0ull ||
             fault->domain != ~0ull;
  long long n = 0;
  for (int s = 0; s < ns; ++s) {
    const unsigned long long in = cnt_recv[s] + cnt_recv[ns + s];
    const unsigned long long pre = vin[s], holes = totals[s][2];
    bad = bad || totals[s][0] > cap[s] || totals[s][1] > cap[s] || in > vin[2 * ns + s] ||
          holes > pre || pre - holes + in > vin[ns + s];
    n += static_cast<long long>(pre - holes + in);
  }
  red[0] = bad ? 0 : n;
  red[1] = bad ? 1 : 0;
}

void launch_world_verdict(const unsigned long long* const* totals, int ns,
                          const unsigned long long* cap, const FaultWord* fault,
                          const unsigned long long* cnt_recv, const unsigned long long* vin,
                          int own_bad, long long* red, cudaStream_t st) {
  world_verdict_kernel<<<1, 32, 0, st>>>(totals, ns, cap, fault, cnt_recv, vin, own_bad, red);
  note_launch();
}

uint64_t migrate_tiles(uint64_t n) { return (n + kTileParticles - 1) / kTileParticles; }

size_t scan_temp_bytes(uint64_t n_tiles) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<const unsigned long long*>(nullptr),
                                static_cast<unsigned long long*>(nullptr), n_tiles);
  return bytes;
}



namespace {

// Fused compaction of several species whose tile counts sit side by side in
// one array: one scan over all of them, then every species' offsets are taken
// relative to the scan value at its first tile (unsigned arithmetic, so
// whatever the tiles before it hold cancels exactly).
__device__ __forceinline__ int compact_species_of(const CompactSet& C, unsigned long long t) {
  for (int i = 0; i < C.n; ++i)
    if (t >= C.s[i].tile0 && t < C.s[i].tile0 + C.s[i].n_tiles) return i;
  return -1;
}

__global__ void compact_totals_kernel(const __grid_constant__ CompactSet C,
                                      const unsigned long long* __restrict__ cnt,
                                      const unsigned long long* __restrict__ off) {
  const int i = threadIdx.x;
  if (i >= C.n) return;
  const CompactSpecies& c = C.s[i];
  unsigned long long t = 0;
  if (c.n_tiles) {
    const unsigned long long last = c.tile0 + c.n_tiles - 1;
    t = off[last] + cnt[last] - off[c.tile0];
  }
  c.totals[0] = t & 0xffffffffull;  // prev
  c.totals[1] = t >> 32;            // next
  c.totals[2] = c.totals[0] + c.totals[1];
}

__global__ void __launch_bounds__(kTileParticles)
    compact_scatter_kernel(const __grid_constant__ CompactSet C,
                           const unsigned long long* __restrict__ cnt,
                           const unsigned long long* __restrict__ off, unsigned long long t_end) {
  __shared__ int warp_tot[2][kTileParticles / 32];
  __shared__ unsigned active[kTileParticles];
  __shared__ int n_active;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (unsigned long long g0 = static_cast<unsigned long long>(blockIdx.x) * kTileParticles;
       g0 < t_end; g0 += static_cast<unsigned long long>(gridDim.x) * kTileParticles) {
    __syncthreads();
    if (threadIdx.x == 0) n_active = 0;
    __syncthreads();
    const unsigned long long tt = g0 + threadIdx.x;
    if (tt < t_end && compact_species_of(C, tt) >= 0 && cnt[tt] != 0)
      active[atomicAdd(&n_active, 1)] = threadIdx.x;
    __syncthreads();
    const int na = n_active;
    for (int a = 0; a < na; ++a) {
      const unsigned long long t = g0 + active[a];
      const CompactSpecies& c = C.s[compact_species_of(C, t)];
      const unsigned long long i = (t - c.tile0) * kTileParticles + threadIdx.x;
      // the mover's owner scan again, from the new y (bad particles were
      // left in place, in this slab: 0; a CflViolation stays: 3 -> 0)
      int flag = i < c.sp.n ? slab_flag(c.sp.y[i], C.sl) : 0;
      if (flag == 3) flag = 0;
      const unsigned bp = __ballot_sync(~0u, flag == 1);
      const unsigned bn = __ballot_sync(~0u, flag == 2);
      __syncthreads();
      if (lane == 0) {
        warp_tot[0][wid] = __popc(bp);
        warp_tot[1][wid] = __popc(bn);
      }
      __syncthreads();
      if (flag == 0) continue;
      int rp = __popc(bp & lt), rn = __popc(bn & lt);
      for (int w = 0; w < wid; ++w) {
        rp += warp_tot[0][w];
        rn += warp_tot[1][w];
      }
      const unsigned long long o = off[t] - off[c.tile0];
      const unsigned long long op = o & 0xffffffffull, on = o >> 32;
      const unsigned long long hp = op + rp, hn = on + rn;
      c.holes[op + on + rp + rn] = i;  // all leavers in index order
      double* dst = nullptr;
      if (flag == 1 && hp < c.cap_out) dst = c.out_prev + 6 * hp;
      if (flag == 2 && hn < c.cap_out) dst = c.out_next + 6 * hn;
      if (dst) {
        double p[6];
        load6(c.sp, i, p);
#pragma unroll
        for (int a6 = 0; a6 < 6; ++a6) dst[a6] = p[a6];
      }
    }
  }
}

}  // namespace

void launch_compact(const CompactSet& C, void* temp, size_t temp_bytes,
                    const unsigned long long* cnt, unsigned long long* off, cudaStream_t st) {
  unsigned long long t_end = 0;
  for (int i = 0; i < C.n; ++i) t_end = std::max(t_end, C.s[i].tile0 + C.s[i].n_tiles);
  if (t_end > 0) {
    size_t b = temp_bytes;
    cub::DeviceScan::ExclusiveSum(temp, b, cnt, off, t_end, st);
    note_launch();
  }
  compact_totals_kernel<<<1, 32, 0, st>>>(C, cnt, off);
  note_launch();
  if (t_end == 0) return;
  const uint64_t groups = (t_end + kTileParticles - 1) / kTileParticles;
  const uint64_t cap = static_cast<uint64_t>(device_sms()) * 16;
  compact_scatter_kernel<<<static_cast<unsigned>(groups < cap ? groups : cap), kTileParticles, 0,
                           st>>>(C, cnt, off, t_end);
  note_launch();
}

void launch_fill(const SpeciesLaunch& sp, const unsigned long long* holes, uint64_t n_holes,
                 const double* in_recs, uint64_t n_in, const SlabLaunch& sl, cudaStream_t st) {
  if (n_in > 0) {
    fill_in_kernel<<<grid_for(n_in, 256), 256, 0, st>>>(sp, holes, n_holes, in_recs, n_in);
    note_launch();
  }
  if (n_in < n_holes) {
    const unsigned long long new_n = sp.n - n_holes + n_in;
    fill_tail_kernel<<<1, 1024, 0, st>>>(sp, holes, n_in, sl, new_n);
    note_launch();
  }
}

}  // namespace b2m
