/*
 * b2m.h — C ABI of the B200-native particle mover (libb2m.so).
 *
 * Drop-in boundary for the reference "minipic" mover path
 * (/root/reference/proj).  Every entry point names the reference interface it
 * replaces.  Plain C: pointers, sizes and status codes; no exceptions and no
 * torch/CUDA types cross it (streams are passed as opaque `void*`).
 *
 * Threading: a b2m_ctx is single-owner (engines.hpp:9-11, "an engine is owned
 * by exactly one worker") but may be driven from any host thread; every call
 * binds the ctx's device first.
 *
 * Errors map one-to-one onto the reference taxonomy (errors.hpp:12-44).  The
 * message of the most recent failure on the calling thread is returned by
 * b2m_last_error().  A context that saw a NumericalFault, CflViolation or a
 * CUDA error is POISONED: every later call returns B2M_ENGINE_FAULT, like the
 * reference's queue (command_queue.cpp:45-49, :71-72) and Simulation
 * (runtime.cpp:192, :205-208).
 */
#ifndef B2M_H_
#define B2M_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B2M_ABI_VERSION 1

typedef enum b2m_status {
  B2M_OK = 0,
  B2M_CONFIG_ERROR = 1,     /* pic::ConfigError     errors.hpp:15-17 */
  B2M_DOMAIN_ERROR = 2,     /* pic::DomainError     errors.hpp:20-22 */
  B2M_ALLOC_ERROR = 3,      /* pic::AllocError      errors.hpp:25-27 */
  B2M_NUMERICAL_FAULT = 4,  /* pic::NumericalFault  errors.hpp:30-32 */
  B2M_CFL_VIOLATION = 5,    /* pic::CflViolation    errors.hpp:35-37 */
  B2M_ENGINE_FAULT = 6,     /* pic::EngineFault     errors.hpp:40-42 */
  B2M_METRIC_ERROR = 7,     /* pic::MetricError     errors.hpp:45-47 */
  B2M_CUDA_ERROR = 8,       /* device/runtime failure (adapters raise EngineFault) */
  B2M_INVALID_ARGUMENT = 9  /* null pointer, bad species id, ... */
} b2m_status;

/* Layout-identical to pic::Grid (grid.hpp:15-41): 64 bytes, offsets nx 0,
 * ny 4, nz 8, lx 16, ly 24, lz 32, dx 40, dy 48, dz 56. */
typedef struct b2m_grid {
  int32_t nx, ny, nz;
  int32_t pad_;
  double lx, ly, lz;
  double dx, dy, dz;
} b2m_grid;

/* Layout-identical to pic::MoverParams (kernels.hpp:30-39): 32 bytes,
 * dt 0, qom 8, pc_iterations 16, beta 24.  beta = qom*dt*0.5 is used as given. */
typedef struct b2m_mover_params {
  double dt;
  double qom;
  int32_t pc_iterations;
  int32_t pad_;
  double beta;
} b2m_mover_params;

/* Arithmetic mode of the mover kernel.
 *   STRICT: the reference's operation order with every product and sum
 *           rounded separately and IEEE division -> bit-identical to
 *           pic::move_batch (kernels.cpp:52-104).
 *   FAST:   fused multiply-add, per-cell polynomial gather and cell-unit
 *           predictor; positions/velocities within 1e-12 (vector-relative)
 *           of the reference, final periodic wrap bit-exact given the
 *           unwrapped coordinate. */
typedef enum b2m_mode { B2M_MODE_STRICT = 0, B2M_MODE_FAST = 1 } b2m_mode;

typedef struct b2m_ctx b2m_ctx;

/* ---- library ------------------------------------------------------------ */
int b2m_abi_version(void);
const char* b2m_status_name(b2m_status s);
/* Message of the last failing call on this thread ("" if none). */
const char* b2m_last_error(void);
/* Number of visible CUDA devices (0 when none); never fails. */
int b2m_device_count(void);
/* Number of kernel launches this process issued through libb2m. */
uint64_t b2m_launch_count(void);

/* ---- value types (grid.hpp:20-29 Grid::make, kernels.hpp:36-38) ---------- */
/* ConfigError unless n >= 2 and l > 0 per axis; dx = lx/nx etc. */
b2m_status b2m_grid_make(int nx, int ny, int nz, double lx, double ly, double lz,
                         b2m_grid* out);
/* MoverParams::make: beta = qom*dt*0.5. */
b2m_status b2m_mover_params_make(double dt, double qom, int pc_iterations,
                                 b2m_mover_params* out);

/* ---- kernel-level boundary ------------------------------------------------
 * Replaces  void pic::move_batch(ParticleSpan p, const FieldView& f,
 *                                const Grid& g, const MoverParams& mp)
 * (kernels.hpp:49, called at engines.cpp:24 and :97).
 *
 * Host pointers in the reference layouts: six SoA arrays of n doubles
 * (ParticleSpan, particle_batch.hpp:13-21) updated in place, and E/B as
 * 3 doubles per node, (nx+1)(ny+1)(nz+1) nodes with mirrored seams
 * (FieldView, field_mesh.hpp:13-16).  Synchronous.  On a non-finite result
 * returns B2M_NUMERICAL_FAULT with *first_bad = index of the first faulting
 * particle; particles [0, first_bad) are updated and [first_bad, n) left
 * untouched, exactly like the reference (kernels.cpp:98-99).
 * Runs on the current device (device 0 unless b2m_set_device was called).
 * Each host thread keeps one cached context (reused while grid, mode and
 * device match and the capacity suffices), so repeated calls cost the copies
 * and the kernel only. */
b2m_status b2m_move_batch_host(const b2m_grid* g, const b2m_mover_params* mp,
                               const double* E, const double* B, double* x, double* y,
                               double* z, double* u, double* v, double* w, uint64_t n,
                               int mode, int64_t* first_bad);
b2m_status b2m_set_device(int device);

/* ---- engine-level boundary ------------------------------------------------
 * Replaces pic::Engine (engines.hpp:20-48) + DeviceArena
 * (device_arena.hpp:23-75) + CommandQueue (command_queue.hpp:17-112): one
 * context = one GPU's device-resident particle store, field buffers and
 * stream.  All device memory is allocated here, so capacity errors surface at
 * creation as B2M_ALLOC_ERROR (device_arena.cpp:20-55), never mid-run. */
b2m_status b2m_ctx_create(int device, const b2m_grid* g, int n_species,
                          const uint64_t* capacity, int mode, b2m_ctx** out);
b2m_status b2m_ctx_destroy(b2m_ctx* ctx);
/* Run all work on an external stream (e.g. torch's current stream);
 * NULL restores the context's own stream. */
b2m_status b2m_ctx_set_stream(b2m_ctx* ctx, void* cuda_stream);
b2m_status b2m_ctx_set_mode(b2m_ctx* ctx, int mode);

/* Pin a host range so the copies below run asynchronously (cudaHostRegister). */
b2m_status b2m_host_register(void* ptr, size_t bytes);
b2m_status b2m_host_unregister(void* ptr);
/* Page-locked host allocation (cudaHostAlloc) for staging buffers. */
b2m_status b2m_host_alloc(size_t bytes, void** out);
b2m_status b2m_host_free(void* ptr);

/* Field upload (enqueue_field_h2d, engines.cpp:52-60): E/B in FieldView
 * layout from host memory; the device relayout for the gather is enqueued
 * behind the copy.  n_nodes must equal (nx+1)(ny+1)(nz+1). */
b2m_status b2m_field_upload(b2m_ctx* ctx, const double* E, const double* B, uint64_t n_nodes);
/* Same from device memory (e.g. after an NCCL broadcast).  Passing the
 * context's own buffers (b2m_field_device_ptrs) copies nothing and only marks
 * the field as changed: the derived gather tables rebuild on the next move. */
b2m_status b2m_field_upload_device(b2m_ctx* ctx, const double* dE, const double* dB,
                                   uint64_t n_nodes);
/* The context's device field buffers (FieldView layout), for a device-side
 * field phase writing the next cycle's field in place (the reference's field
 * update between mover calls, runtime.cpp:221-223). */
b2m_status b2m_field_device_ptrs(b2m_ctx* ctx, double** dE, double** dB);

/* Species transfers (enqueue_species_h2d/d2h, engines.cpp:62-93).  host6 =
 * {x,y,z,u,v,w}.  Upload sets the device count to n (AllocError above
 * capacity).  Download copies count() particles. */
b2m_status b2m_species_upload(b2m_ctx* ctx, int s, const double* const* host6, uint64_t n);
b2m_status b2m_species_download(b2m_ctx* ctx, int s, double* const* host6, uint64_t max_n,
                                uint64_t* n_out);
/* Partial transfers for chunked pipelines: [offset, offset+n). */
b2m_status b2m_species_upload_range(b2m_ctx* ctx, int s, const double* const* host6,
                                    uint64_t offset, uint64_t n);
b2m_status b2m_species_download_range(b2m_ctx* ctx, int s, double* const* host6,
                                      uint64_t offset, uint64_t n);
b2m_status b2m_species_set_count(b2m_ctx* ctx, int s, uint64_t n);
b2m_status b2m_species_count(b2m_ctx* ctx, int s, uint64_t* n);
b2m_status b2m_species_capacity(b2m_ctx* ctx, int s, uint64_t* cap);
/* Device addresses of the six SoA arrays of species s. */
b2m_status b2m_species_device_ptrs(b2m_ctx* ctx, int s, double** out6);

/* The mover kernel on device-resident species s (enqueue_kernel,
 * engines.cpp:95-99).  Asynchronous; a fault is recorded on the device and
 * reported by b2m_sync. */
b2m_status b2m_move(b2m_ctx* ctx, int s, const b2m_mover_params* mp);
/* All species in one launch: mp[n_species].  Records event slots 11 and 12
 * around the mover launch(es) alone -- after any gather-table rebuild the
 * call enqueues first -- so b2m_event_elapsed_ms(11, 12) is the kernel time. */
b2m_status b2m_move_all(b2m_ctx* ctx, const b2m_mover_params* mp);
/* Range variant for chunked pipelines. */
b2m_status b2m_move_range(b2m_ctx* ctx, int s, const b2m_mover_params* mp, uint64_t offset,
                          uint64_t n);

/* Engine-level mover cycle for HOST-resident batches (the whole
 * enqueue_species_h2d -> enqueue_kernel -> enqueue_species_d2h schedule of
 * engines.cpp:62-99 / :157-200 in one call): every species is cut into chunks
 * of `chunk` particles that flow H2D -> mover -> D2H on three streams, so both
 * PCIe directions and the kernel overlap.  host6_all[6*s + a] is array a of
 * species s (page-locked memory for full overlap), counts[s] its size, mp[s]
 * its parameters.  The field must have been uploaded.  Blocking: on return
 * the host arrays hold the moved particles; faults as b2m_sync. */
b2m_status b2m_run_mover_host(b2m_ctx* ctx, int n_species, double* const* host6_all,
                              const uint64_t* counts, const b2m_mover_params* mp,
                              uint64_t chunk);

/* Optional cell-sort pass for gather locality (north star): stable
 * reordering of species s by cell index of its current position.  The
 * particle multiset is unchanged (the reference's own exchange reorders too,
 * runtime.cpp:64-76). */
b2m_status b2m_sort_species(b2m_ctx* ctx, int s);

/* ---- field phase stand-in (field_phase_stub, kernels.cpp:185-215) ---------
 * `passes` rounds of 7-point averaging of E on the context's device field
 * (B untouched), then the seam mirror of E and B -- bit-identical to the
 * reference.  The result becomes the context's field (the FAST tables are
 * rebuilt on the next move), like Simulation's f_next (runtime.cpp:222).
 * b2m_field_download copies the device field to host (FieldView layout).
 * The _host form runs in place on host arrays (one-shot). */
b2m_status b2m_field_phase_stub(b2m_ctx* ctx, int passes);
b2m_status b2m_field_download(b2m_ctx* ctx, double* E, double* B);
b2m_status b2m_field_phase_stub_host(const b2m_grid* g, double* E, double* B, int passes);

/* ---- moments (deposit_moments, kernels.cpp:147-183; MomentMesh
 * kernels.hpp:54-69) -------------------------------------------------------
 * The context owns one device moment mesh of nx*ny*nz periodic nodes (index
 * i + nx*(j + ny*k)): rho, jx, jy, jz and, with pressure, pxx, pxy, pxz, pyy,
 * pyz, pzz.  b2m_moments_zero (re)allocates it for `with_pressure` and zeroes
 * it (MomentMesh::make / zero); b2m_deposit adds species s's particles with
 * charge q_per_particle each (asynchronous; a particle outside the domain is
 * reported by b2m_sync as B2M_DOMAIN_ERROR, the reference's grid_cell_of
 * DomainError); b2m_moments_download copies the 4 (or 10) arrays to host
 * out[0..] and synchronizes.  Sums are in a different order than the
 * reference's particle order: equal to rounding. */
b2m_status b2m_moments_zero(b2m_ctx* ctx, int with_pressure);
b2m_status b2m_deposit(b2m_ctx* ctx, int s, double q_per_particle);
/* One mover cycle of all species followed by the deposition of their new
 * state: the reference's move_batch per species then deposit_moments per
 * species (runtime.cpp:227-229, :251-262; kernels.cpp:52-104, :147-183).
 * FAST without pressure: ONE fused launch -- rho and J are deposited from the
 * tile the mover just wrote, in shared memory, by FP64 DMMA (b2m_fused.cuh),
 * so the particles are not re-read from HBM.  STRICT (bit-identical
 * per-particle terms) or with pressure: b2m_move_all then b2m_deposit per
 * species.  mp[n_species], q_per_particle[n_species]; b2m_moments_zero
 * first.  Event slots 11 / 12 bracket the launch(es) as in b2m_move_all. */
b2m_status b2m_move_deposit_all(b2m_ctx* ctx, const b2m_mover_params* mp,
                                const double* q_per_particle);
b2m_status b2m_moments_download(b2m_ctx* ctx, double* const* out, int n_arrays);
/* Device view of the moment mesh: one contiguous block of n_doubles =
 * (4 or 10) * nx*ny*nz, arrays in the order above -- for reducing the
 * per-rank meshes across GPUs (the reference sums per-worker meshes,
 * runtime.cpp:256-262). */
b2m_status b2m_moments_device_ptr(b2m_ctx* ctx, double** d_mesh, uint64_t* n_doubles);
/* One-shot pic::deposit_moments for host arrays: ADDS the n particles'
 * moments into out[0..3] (+ out[4..9] with pressure), nx*ny*nz each.
 * B2M_DOMAIN_ERROR (nothing added) if a particle lies outside the domain. */
b2m_status b2m_deposit_moments_host(const b2m_grid* g, const double* x, const double* y,
                                    const double* z, const double* u, const double* v,
                                    const double* w, uint64_t n, double q_per_particle,
                                    int with_pressure, double* const* out);

/* Wait for all enqueued work (CommandQueue::synchronize,
 * command_queue.cpp:45-49).  Returns B2M_NUMERICAL_FAULT with the species and
 * particle index of the first recorded fault (message text as
 * kernels.cpp:98-99), B2M_CFL_VIOLATION for an exchange violation, and
 * poisons the context. */
b2m_status b2m_sync(b2m_ctx* ctx, int* bad_species, int64_t* first_bad);
/* Kernel timing without host syncs: after b2m_kernel_timing_begin(ctx, n)
 * the next n b2m_move_all calls each record a CUDA event pair around their
 * mover launch(es) alone; b2m_kernel_timing_read waits for them and returns
 * the n durations in ms (*n = how many were recorded) and ends the log. */
b2m_status b2m_kernel_timing_begin(b2m_ctx* ctx, int capacity);
b2m_status b2m_kernel_timing_read(b2m_ctx* ctx, float* ms, int max_n, int* n);
/* Record / measure device time on the context's stream (CUDA events). */
b2m_status b2m_event_record(b2m_ctx* ctx, int slot);
b2m_status b2m_event_elapsed_ms(b2m_ctx* ctx, int slot_a, int slot_b, float* ms);

/* ---- partition layer (runtime.cpp:22-76; one context per GPU/rank) -------
 * y-slab decomposition exactly as pic::decompose / pic::owner_of
 * (runtime.cpp:22-44).  ConfigError unless world divides ny and slabs have
 * >= 2 cells. */
b2m_status b2m_slab_config(b2m_ctx* ctx, int rank, int world);
/* owner_of(y) (runtime.cpp:39-44), for host-side checks. */
int b2m_owner_of(const b2m_grid* g, int world, double y);
/* Mover fused with the migration scan of partition_outgoing
 * (runtime.cpp:46-62): particles whose new y belongs to the previous / next
 * slab are appended to that outbox (48-byte PartRec records
 * {x,y,z,u,v,w}, runtime.hpp:35-37) and removed; survivors are compacted in
 * place preserving scan order.  A particle landing in a non-neighbour slab
 * records a CflViolation.  Asynchronous. */
b2m_status b2m_move_migrate(b2m_ctx* ctx, int s, const b2m_mover_params* mp);
/* All species (mp[n_species]) in one mover launch, then each species'
 * compaction -- the per-cycle form of the above. */
b2m_status b2m_move_migrate_all(b2m_ctx* ctx, const b2m_mover_params* mp);
/* After b2m_sync: outbox of species s towards dir (0 = prev, 1 = next);
 * device pointer to count records. */
b2m_status b2m_outbox(b2m_ctx* ctx, int s, int dir, double** d_recs, uint64_t* count);
/* Append n received PartRec records (device memory) to species s
 * (merge_incoming, runtime.cpp:64-76).  AllocError above capacity. */
b2m_status b2m_inbox_append(b2m_ctx* ctx, int s, const double* d_recs, uint64_t n);

/* ---- native slab world over NCCL ------------------------------------------
 * Simulation's per-cycle protocol (runtime.cpp:218-288) for one rank per
 * GPU, replacing worker_loop's mover + partition_outgoing + exchange +
 * merge_incoming + count check (runtime.cpp:227-269).
 * b2m_world_id: the NCCL unique id (B2M_WORLD_ID_BYTES), made on one rank and
 * handed to all.  b2m_world_init: b2m_slab_config + ncclCommInitRank + the
 * exchange buffers (AllocError here, never mid-run); id == NULL builds the
 * buffers without a communicator (world of 1, or b2m_world_loopback_step).
 * b2m_world_set_total: the global particle count, the conservation reference
 * (runtime.cpp:150).  b2m_world_step: b2m_move_migrate_all, the outbox counts
 * exchanged with prev / next, one all-reduce of (count after the merge,
 * failed ranks) computed on the device from those counts, then -- when no
 * rank failed and the count is conserved -- the records exchanged (grouped
 * ncclSend/ncclRecv) and merged.  Returns this rank's typed fault
 * (NumericalFault / CflViolation / DomainError / AllocError) when it failed
 * -- it still takes part in the counts round and the all-reduce with empty
 * outboxes, so its peers do not hang (the analogue of arrive_and_drop,
 * runtime.cpp:283-288) --, EngineFault when a peer failed or the global count
 * drifted; every rank reads the same reduced verdict, so all take the same
 * branch.  One host synchronisation per step.  *sent = records this rank
 * sent.  The step records event slots 13 (start), 14 (mover + compaction
 * enqueued) and 15 (exchange and merge enqueued) on the context's stream, so
 * b2m_event_elapsed_ms(13, 14) / (14, 15) split its device time. */
#define B2M_WORLD_ID_BYTES 128
b2m_status b2m_world_id(void* id);
/* B2M_OK when NCCL resolved in this process (B2M_NCCL_LIB, the process's own
 * libnccl, or libnccl.so.2), else ConfigError with the reason: what every
 * rank checks -- and the ranks agree on -- before b2m_world_init. */
b2m_status b2m_world_nccl_available(void);
b2m_status b2m_world_init(b2m_ctx* ctx, const void* id, int rank, int world);
b2m_status b2m_world_set_total(b2m_ctx* ctx, uint64_t* total);
/* Replicate the root rank's device field on every rank (ncclBroadcast of E
 * and B): runtime.cpp:143 gives every worker the whole mesh.  A header with
 * the root's z-invariance flag and node plane 0 go first; a z-invariant field
 * is rebuilt from plane 0 on the other ranks (bitwise the root's field), any
 * other field is sent whole (B2M_BCAST_ZINV=0: always whole).  One host read
 * of the header per call. */
b2m_status b2m_world_broadcast_field(b2m_ctx* ctx, int root);
/* Sum every rank's moment mesh (b2m_moments_zero + b2m_deposit per rank) into
 * every rank's mesh, in place, in the reference's order: zero, then rank
 * 0's mesh added, then rank 1's, ... (moments_.add per worker,
 * runtime.cpp:256-262) -- an ncclAllGather of the meshes and one ordered,
 * separately rounded sum per element on every rank, so the reduction itself
 * is deterministic and identical on all ranks (unlike an ncclAllReduce,
 * whose order depends on the NCCL algorithm).  Each rank's own mesh still
 * sums its particles with FP64 atomics (equal to the reference to rounding).
 * The gather buffer (world x mesh) is reserved with the mesh
 * (b2m_moments_zero, or b2m_world_init when the mesh exists): the reduction
 * allocates nothing. */
b2m_status b2m_world_reduce_moments(b2m_ctx* ctx);
b2m_status b2m_world_step(b2m_ctx* ctx, const b2m_mover_params* mp, uint64_t* sent,
                          uint64_t* global_count);
/* The same protocol over the `world` contexts of ONE process (rank r =
 * ctxs[r], each b2m_world_init'ed with id NULL), the exchange done by device
 * copies: the protocol without NCCL, for tests on one GPU. */
b2m_status b2m_world_loopback_step(b2m_ctx* const* ctxs, int world, const b2m_mover_params* mp,
                                   uint64_t* sent);

/* ---- synthetic GEM input (init.cpp:62-102, rng.hpp:12-56) ----------------
 * Bit-identical to pic::init_gem for the default GEM parameters
 * (sim_config.hpp:30-39) on grid g: the 4 species (bg e-, bg i+, sheet e-,
 * sheet i+) and the Harris B field with E = 0.  Host memory; uses `threads`
 * host threads (0 = all). */
b2m_status b2m_gem_counts(const b2m_grid* g, int ppc, uint64_t* counts4);
b2m_status b2m_gem_species_params(const b2m_grid* g, int ppc, double* qom4, double* qpp4);
b2m_status b2m_gem_fill_species(const b2m_grid* g, int ppc, uint64_t seed, int s,
                                double* const* host6, int threads);
/* Background species s (0 or 1) particles [m0, m1) of the reference's
 * (k,j,i,p) emission order, written to host6[a][0 .. m1-m0): the counter RNG
 * jumps straight to particle m0, so a rank can generate just its slab. */
b2m_status b2m_gem_fill_species_range(const b2m_grid* g, int ppc, uint64_t seed, int s,
                                      uint64_t m0, uint64_t m1, double* const* host6,
                                      int threads);
b2m_status b2m_gem_field(const b2m_grid* g, double* E, double* B);
/* Test/bench field fixture with nonzero E (test_offload.cpp:60-71):
 * E=(0.01 sin y, 0, 0.02), B=(tanh((y-ly/2)/0.5), 0.05 sin x, 0). */
b2m_status b2m_gem_like_field(const b2m_grid* g, double* E, double* B);

#ifdef __cplusplus
}
#endif

#endif /* B2M_H_ */
