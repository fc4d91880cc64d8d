// b2m_ctx.hpp — the context behind the C ABI's opaque b2m_ctx, shared by
// the ABI translation units (b2m_capi.cu: contexts, transfers, mover, sort,
// moments, migration steps; b2m_world.cu: the native slab world).  Not part
// of the ABI.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "b2m_internal.hpp"

namespace b2m {

constexpr int kEventSlots = 16;

struct Species {
  // the six SoA arrays live in one [6][stride] block (stride = capacity
  // rounded up to 32), so a tile of all six is a single 2-D TMA box
  double* a[6] = {};
  double* alt[6] = {};  // ping-pong set for the cell sort (allocated on first sort)
  uint64_t capacity = 0;
  uint64_t stride = 0;
  uint64_t count = 0;
  // migration scratch
  uint8_t* flags = nullptr;  // non-null: the owner scan is on (a 1-byte marker, nothing stored)
  unsigned long long* tcnt = nullptr;  // per-tile packed leaver counts (next << 32 | prev)
  unsigned long long* toff = nullptr;  // their exclusive scan
  double* out[2] = {};
  uint64_t cap_out = 0;
  unsigned long long* holes = nullptr;
  unsigned long long* totals = nullptr;   // device [3]
  unsigned long long* totals_h = nullptr; // pinned [3]
  uint64_t n_out[2] = {0, 0};
  uint64_t n_holes = 0;
  uint64_t pre_count = 0;  // count before the last migration step
  bool migrate_pending = false;
  // FAST: the field as per-cell polynomials pre-scaled by this species' beta
  // (qom*dt/2), rebuilt when the field or beta changes
  double2* cells = nullptr;
  double cells_beta = 0.0;
  uint64_t cells_gen = 0;
};


// NCCL is resolved at run time, not linked: a process that already loaded
// one (torch bundles its own libnccl.so.2) keeps using it, and loading this
// library never pins a different NCCL under the same soname before torch.
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl();  // b2m_world.cu


}  // namespace b2m

struct b2m_ctx {
  int device = 0;
  b2m_grid grid{};
  int mode = B2M_MODE_FAST;
  std::vector<b2m::Species> sp;
  uint64_t n_nodes = 0;
  double* dE = nullptr;
  double* dE_alt = nullptr;  // field-stub ping-pong (allocated on first use)
  // field stub replayed as a CUDA graph: the `passes` launches are captured
  // once per (passes, buffers, stream) and replayed with one cudaGraphLaunch
  // (two entries: an odd pass count alternates the ping-pong buffers)
  struct StubGraph {
    cudaGraphExec_t exec = nullptr;
    int passes = 0;
    const double* in = nullptr;
    cudaStream_t stream = nullptr;
    double* out = nullptr;
  } stub[2];
  double* strict_nodes = nullptr;  // STRICT per-cell corner node table
  // FAST: device flag, 0 when the field is z-invariant (set with every table
  // build); null when the z-invariant kernel is disabled (B2M_FAST_3D=1)
  int* zvar = nullptr;
  uint64_t strict_gen = 0;
  double* dB = nullptr;
  bool field_ready = false;
  uint64_t field_gen = 0;  // bumped by every field upload
  b2m::FaultWord* fault = nullptr;
  b2m::FaultWord* fault_h = nullptr;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[b2m::kEventSlots] = {};
  bool poisoned = false;
  std::string poison_msg;
  // sort scratch (lazily sized to the largest species)
  void* sort_temp = nullptr;
  size_t sort_temp_bytes = 0;
  uint32_t* keys[2] = {};
  uint32_t* vals[2] = {};
  double* scratch = nullptr;
  uint64_t sort_cap = 0;
  // counting sort by cell: per-cell counts / offsets and the scan's temp
  uint32_t* bin_keys = nullptr;
  uint64_t bin_keys_cap = 0;
  uint32_t* bin_count = nullptr;
  uint32_t* bin_offs = nullptr;
  void* bin_temp = nullptr;
  size_t bin_temp_bytes = 0;
  void* scan_temp = nullptr;
  size_t scan_temp_bytes = 0;
  // host pipeline (b2m_run_mover_host)
  cudaStream_t up = nullptr, down = nullptr;
  std::vector<cudaEvent_t> pipe_ev;
  // moment mesh (b2m_moments_zero): 4 or 10 arrays of nx*ny*nz
  double* mom[10] = {};
  int mom_arrays = 0;
  bool mom_pressure = false;
  // slab partition
  bool slab_on = false;
  b2m::SlabLaunch sl{};
  // migration: every species' tile counts / offsets side by side (one scan),
  // their totals in one device block and one pinned block (one copy back)
  unsigned long long* mig_tcnt = nullptr;
  unsigned long long* mig_toff = nullptr;
  unsigned long long* mig_totals = nullptr;
  unsigned long long* mig_totals_h = nullptr;
  std::vector<uint64_t> mig_tile0;
  // native slab world (b2m_world_init / b2m_world_step)
  struct World {
    bool on = false;
    ncclComm_t comm = nullptr;            // null: loopback (tests) or world of 1
    unsigned long long** totals = nullptr;  // device [ns] -> each species' totals
    unsigned long long* cap = nullptr;      // device [ns] outbox capacities
    unsigned long long* cnt_send = nullptr;  // device [2][ns]: to prev, to next
    unsigned long long* cnt_recv = nullptr;  // device [2][ns]: from prev, from next
    unsigned long long* cnt_h = nullptr;     // pinned [4][ns]: send then recv rows
    std::vector<double*> stage;              // device per species: arrivals (AoS records)
    std::vector<uint64_t> stage_cap;         // records per species
    long long* red = nullptr;                // device [2]: count, faulted
    long long* red_h = nullptr;              // pinned [2]
    unsigned long long* vin = nullptr;       // device [3][ns]: pre-step count, capacity, stage cap
    unsigned long long* vin_h = nullptr;     // pinned [3][ns]
    double* bstage = nullptr;                // device: field broadcast header + plane 0 (E, B)
    double* bflag_h = nullptr;               // pinned: the broadcast header (z-invariance flag)
    double* mstage = nullptr;                // device [world][mesh]: gathered moment meshes
    uint64_t mstage_n = 0;                   // doubles per rank in mstage
    uint64_t total = 0;
    bool total_set = false;
  } w;
  std::vector<void*> allocations;
  // b2m_kernel_timing_begin / _read: per mover call a (start, end) event pair
  // around the mover launch(es) alone, for timing without host syncs
  std::vector<cudaEvent_t> kt_ev;
  int kt_cap = 0, kt_n = 0;
};

namespace b2m {

b2m_status cuda_fail(b2m_ctx* ctx, cudaError_t e, const char* what);
// b2m_world.cu: reserve the moment all-gather buffer for an n-double mesh
b2m_status world_reserve_moments(b2m_ctx* ctx, uint64_t n);
b2m_status check_ctx(b2m_ctx* ctx);
b2m_status check_species(b2m_ctx* ctx, int s);
b2m_status check_params(const b2m_mover_params* mp);
// the mover over n species in one launch fused with the owner scan, then
// each species' compaction (b2m_move_migrate[_all])
b2m_status move_migrate_species(b2m_ctx* ctx, const int* species, const b2m_mover_params* mp,
                                int n);

#define B2M_CUDA(ctx, call)                                   \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return cuda_fail((ctx), e_, #call); \
  } while (0)

template <class T>
inline b2m_status dalloc(b2m_ctx* ctx, T** p, size_t count, const char* what) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(B2M_ALLOC_ERROR, std::string("device allocation failed for ") + what + " (" +
                                     std::to_string(count * sizeof(T)) + " bytes): " +
                                     cudaGetErrorString(e));
  }
  ctx->allocations.push_back(*p);
  return B2M_OK;
}

}  // namespace b2m
