// b2m_internal.hpp — host-side declarations shared by the libb2m translation
// units (kernel launchers, context, GEM generator).  Not part of the ABI.
#pragma once

#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "b2m.h"
#include "b2m_mover.cuh"

namespace b2m {

// Thread-local last-error text (b2m_last_error).
void set_error(const std::string& msg);
b2m_status fail(b2m_status s, const std::string& msg);

// SM count of the device (queried once; every GPU of the process is a B200).
int device_sms();
// Count of kernel launches issued by this process (b2m_launch_count).
void note_launch(int n = 1);

// Host computation of the exact-wrap thresholds for one axis length.
WrapAxis make_wrap_axis(double l);
DevGrid to_dev(const b2m_grid& g);
FastGrid to_fast(const b2m_grid& g);

// ---- launchers (b2m_kernels.cu) -------------------------------------------
// All launches are asynchronous on `st`.

// FAST mover on a batch of species spans (one launch).  Returns false when a
// TMA tensor map cannot be built (driver entry point missing, >2^31 columns).
struct SlabLaunch;
bool launch_move_fast(const FastGrid& g, const SpeciesLaunch* sp,
                      int n_spans, FaultWord* fault, cudaStream_t st,
                      const SlabLaunch* sl = nullptr, uint8_t* const* flags = nullptr,
                      unsigned long long* const* tcnt = nullptr, const int* zvar = nullptr,
                      double* const* mom = nullptr);
// STRICT mover on the same warp-tile pipeline (bit-identical to the reference)
bool launch_move_strict_tiles(const DevGrid& g, const FastGrid& fg, const double* nodes,
                              const SpeciesLaunch* sp, int n_spans, FaultWord* fault,
                              cudaStream_t st, const SlabLaunch* sl = nullptr,
                              uint8_t* const* flags = nullptr,
                              unsigned long long* const* tcnt = nullptr,
                              const int* zvar = nullptr);
// The field's z-invariance flag alone (0 = every node plane equals plane 0
// bit for bit); launch_field_to_cells runs it too.
void launch_zinv_check(int nx, int ny, int nz, const double* E, const double* B, int* zvar,
                       cudaStream_t st);
// STRICT cell table: per cell the 8 corner nodes' E, B (48 doubles).
void launch_strict_nodes(int nx, int ny, int nz, const double* E, const double* B, double* out,
                         cudaStream_t st);
// Node AoS E/B -> per-cell polynomial coefficients of (scale[m]*E,
// scale[m]*B) into tables[m] (48 doubles per cell), one field read per
// kMaxTables tables.
constexpr int kMaxTables = 8;
// With `zvar` (device int): first set it to 0 when the field is z-invariant
// (every node plane k equal to plane 0 bit for bit), else 1; when 0, the tables
// are written in the column layout of the z-invariant kernel (nx*ny columns
// of 24 doubles: per component p0..p3 of the bilinear polynomial).
void launch_field_to_cells(int nx, int ny, int nz, const double* E, const double* B,
                           const double* scale, double2* const* tables, int n_tables,
                           cudaStream_t st, int* zvar = nullptr);
// Moment deposition (b2m_moments.cu, deposit_moments kernels.cpp:147-183) of
// one species span, qv = q_per_particle / cell volume, accumulated into
// mesh[0..3] = rho, jx, jy, jz (+ mesh[4..9] = pxx..pzz with pressure).
// exact: bit-identical per-particle terms (STRICT); else FAST arithmetic.
void launch_deposit(const DevGrid& g, const SpeciesLaunch& sp, double qv, double* const* mesh,
                    bool pressure, bool exact, FaultWord* fault, cudaStream_t st);
// field_phase_stub (b2m_field.cu, kernels.cpp:185-215) on the node AoS E/B:
// `passes` stencil rounds ping-ponging between E and scratch, then the seam
// mirror of E and B.  Returns the buffer that holds the result (E or scratch).
double* launch_field_stub(int nx, int ny, int nz, double* E, double* B, double* scratch,
                          int passes, cudaStream_t st);
// Reset the fault words to "clean".
void launch_fault_reset(FaultWord* fault, cudaStream_t st);
void launch_pack_counts(const unsigned long long* const* totals, int ns,
                        const unsigned long long* cap, const FaultWord* fault,
                        unsigned long long* out, cudaStream_t st);
// Native slab world: this rank's verdict for the closing all-reduce, from
// device state after the counts round (b2m_world_step).  vin = [3][ns]:
// count before the step, capacity, exchange-buffer records per species.
void launch_world_verdict(const unsigned long long* const* totals, int ns,
                          const unsigned long long* cap, const FaultWord* fault,
                          const unsigned long long* cnt_recv, const unsigned long long* vin,
                          int own_bad, long long* red, cudaStream_t st);

// Cell keys of the current positions (cell-unit locate), for sorting.
void launch_cell_keys(const FastGrid& g, const double* x, const double* y, const double* z,
                      uint64_t n, uint32_t* keys, uint32_t* vals, cudaStream_t st);
// Counting sort of the six SoA arrays by cell (unstable within a cell) from
// `in` into `out`; keys: n scratch, count / offs: nx*ny*nz + 1 scratch each.
size_t bin_scan_temp_bytes(uint64_t n_bins);
void launch_bin_sort(const FastGrid& g, double* const* in, double* const* out, uint64_t n,
                     uint32_t* keys, uint32_t* count, uint32_t* offs, void* temp,
                     size_t temp_bytes, cudaStream_t st);
// out[i] = in[perm[i]]
void launch_gather(const double* in, const uint32_t* perm, uint64_t n, double* out,
                   cudaStream_t st);
// Temp bytes needed by the radix sort of n (key,value) pairs.
size_t sort_temp_bytes(uint64_t n, int key_bits);
void launch_sort_pairs(void* temp, size_t temp_bytes, const uint32_t* kin, uint32_t* kout,
                       const uint32_t* vin, uint32_t* vout, uint64_t n, int key_bits,
                       cudaStream_t st);

// ---- migration (y-slab partition layer) ----------------------------------
struct SlabLaunch {
  int rank, world, prev, next;
  int slab;        // ny / world
  double dy;       // owner_of divisor (grid.hpp Grid::dy)
  int ny;
  // owner_of(y) == r  <=>  y in [lo_r, hi_r): exact thresholds of the
  // reference's trunc(y / dy) (b2m_slab_config), for this rank, prev, next
  double own_lo, own_hi, prev_lo, prev_hi, next_lo, next_hi;
};

// The movers above, given `sl`, `flags` and `tcnt`, also run the owner_of
// scan: flags[i] (0 stay, 1 prev, 2 next) and, per 128-particle tile t,
// tcnt[t] = next << 32 | prev.
uint64_t migrate_tiles(uint64_t n);
// one species of a fused migration compaction (its tile counts start at
// tile0 of the shared count array)
constexpr int kMaxCompactSpecies = 16;
struct CompactSpecies {
  SpeciesLaunch sp;
  const uint8_t* flags;
  double* out_prev;
  double* out_next;
  unsigned long long cap_out;
  unsigned long long* holes;
  unsigned long long* totals;  // device [3]: prev, next, holes
  unsigned long long tile0, n_tiles;
};
struct CompactSet {
  CompactSpecies s[kMaxCompactSpecies];
  SlabLaunch sl;  // the owner scan's thresholds: leavers re-derived from the new y
  int n;
};
// scan of the shared tile counts, every species' totals, outbox + hole scatter
void launch_compact(const CompactSet& C, void* temp, size_t temp_bytes,
                    const unsigned long long* cnt, unsigned long long* off, cudaStream_t st);
// CUB temp bytes of the tile-count scan
size_t scan_temp_bytes(uint64_t n_tiles);

// Fill holes with incoming records, then append / compact the tail.
void launch_fill(const SpeciesLaunch& sp, const unsigned long long* holes, uint64_t n_holes,
                 const double* in_recs, uint64_t n_in, const SlabLaunch& sl, cudaStream_t st);

}  // namespace b2m
