// world_example.cpp -- the per-rank cycle of INTEGRATION.md section 6 as a
// compilable function (tests/test_capi.py builds it against include/b2m.h and
// libb2m.so; running it needs one GPU per rank and an id exchange).
#include <cstdint>
#include <stdexcept>
#include <string>

#include "b2m.h"

namespace {
void check(b2m_status st) {
  if (st != B2M_OK) throw std::runtime_error(std::string(b2m_status_name(st)) + ": " + b2m_last_error());
}
}  // namespace

// `id` was made by b2m_world_id on rank 0 and handed to every rank.
void run_rank(int local_gpu, int rank, int world, const unsigned char* id, const b2m_grid& grid,
              int n_species, const uint64_t* caps, double* const* const* slab_arrays,
              const uint64_t* slab_counts, const double* E, const double* B, uint64_t n_nodes,
              const b2m_mover_params* params, int cycles) {
  b2m_ctx* ctx = nullptr;
  check(b2m_ctx_create(local_gpu, &grid, n_species, caps, B2M_MODE_STRICT, &ctx));
  check(b2m_world_init(ctx, id, rank, world));
  for (int s = 0; s < n_species; ++s)
    check(b2m_species_upload(ctx, s, slab_arrays[s], slab_counts[s]));
  if (rank == 0) check(b2m_field_upload(ctx, E, B, n_nodes));
  check(b2m_world_broadcast_field(ctx, 0));      // runtime.cpp:143
  uint64_t total = 0;
  check(b2m_world_set_total(ctx, &total));       // runtime.cpp:150
  for (int cycle = 0; cycle < cycles; ++cycle) {
    uint64_t sent = 0, n = 0;
    check(b2m_world_step(ctx, params, &sent, &n));  // runtime.cpp:227-269
  }
  b2m_ctx_destroy(ctx);
}
