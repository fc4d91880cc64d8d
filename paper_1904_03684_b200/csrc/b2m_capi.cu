// b2m_capi.cu — the C ABI (include/b2m.h): contexts, transfers, launches,
// fault surfacing and the y-slab migration steps (the native slab world that
// drives them is b2m_world.cu; the context itself is b2m_ctx.hpp).
//
// Context = the B200 replacement of one offload engine's DeviceArena +
// CommandQueue (device_arena.cpp:17-111, command_queue.cpp:9-95): device
// memory is carved up front, work goes to one CUDA stream, faults poison the
// context.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <vector>

#include "b2m_ctx.hpp"

namespace b2m {

namespace {
thread_local std::string g_last_error;
std::atomic<unsigned long long> g_launches{0};
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }

b2m_status fail(b2m_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

void note_launch(int n) { g_launches.fetch_add(static_cast<unsigned long long>(n)); }

// Thresholds of the exact floor(v/l) window (see WrapAxis in b2m_mover.cuh):
// RN(v/l) is monotone in v, so walk from a candidate with nextafter and
// confirm each side with the host's IEEE division.
static double last_below(double l, double k, double start) {
  double v = start;
  // move up while still below k, then down until below k
  for (int it = 0; it < 64 && v / l < k; ++it) {
    const double nv = std::nextafter(v, std::numeric_limits<double>::infinity());
    if (!(nv / l < k)) break;
    v = nv;
  }
  for (int it = 0; it < 64 && !(v / l < k); ++it) v = std::nextafter(v, -std::numeric_limits<double>::infinity());
  return v;
}

static double first_at_least(double l, double k, double start) {
  double v = start;
  for (int it = 0; it < 64 && v / l >= k; ++it) {
    const double nv = std::nextafter(v, -std::numeric_limits<double>::infinity());
    if (!(nv / l >= k)) break;
    v = nv;
  }
  for (int it = 0; it < 64 && !(v / l >= k); ++it) v = std::nextafter(v, std::numeric_limits<double>::infinity());
  return v;
}

WrapAxis make_wrap_axis(double l) {
  WrapAxis a;
  a.l = l;
  a.hi0 = last_below(l, 1.0, l);
  a.hi1 = last_below(l, 2.0, 2.0 * l);
  a.lom1 = first_at_least(l, -1.0, -l);
  return a;
}

DevGrid to_dev(const b2m_grid& g) {
  DevGrid d;
  d.nx = g.nx; d.ny = g.ny; d.nz = g.nz;
  d.lx = g.lx; d.ly = g.ly; d.lz = g.lz;
  d.dx = g.dx; d.dy = g.dy; d.dz = g.dz;
  d.rdx = 1.0 / g.dx; d.rdy = 1.0 / g.dy; d.rdz = 1.0 / g.dz;
  return d;
}

FastGrid to_fast(const b2m_grid& g) {
  FastGrid f;
  f.nx = g.nx; f.ny = g.ny; f.nz = g.nz;
  f.nxd = g.nx; f.nyd = g.ny; f.nzd = g.nz;
  f.rnx = 1.0 / g.nx; f.rny = 1.0 / g.ny; f.rnz = 1.0 / g.nz;
  f.rdx = 1.0 / g.dx; f.rdy = 1.0 / g.dy; f.rdz = 1.0 / g.dz;
  f.lx = g.lx; f.ly = g.ly; f.lz = g.lz;
  f.ax = make_wrap_axis(g.lx);
  f.ay = make_wrap_axis(g.ly);
  f.az = make_wrap_axis(g.lz);
  return f;
}

}  // namespace b2m

using namespace b2m;


namespace b2m {

b2m_status cuda_fail(b2m_ctx* ctx, cudaError_t e, const char* what) {
  std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
  cudaGetLastError();  // reported here: a non-sticky error must not resurface at a later check
  if (ctx) {
    ctx->poisoned = true;
    ctx->poison_msg = msg;
  }
  return fail(B2M_CUDA_ERROR, msg);
}


b2m_status check_ctx(b2m_ctx* ctx) {
  if (!ctx) return fail(B2M_INVALID_ARGUMENT, "null context");
  if (ctx->poisoned)
    return fail(B2M_ENGINE_FAULT, "device state is invalid after an earlier fault: " + ctx->poison_msg);
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  // every entry point checks cudaGetLastError() after its launches: drop a
  // non-sticky error some earlier, unrelated call of this host thread left
  // behind (a device fault is sticky and still reported)
  cudaGetLastError();
  return B2M_OK;
}

b2m_status check_species(b2m_ctx* ctx, int s) {
  if (s < 0 || s >= static_cast<int>(ctx->sp.size()))
    return fail(B2M_INVALID_ARGUMENT, "species id " + std::to_string(s) + " out of range");
  return B2M_OK;
}


SpeciesLaunch make_launch(b2m_ctx* ctx, int s, const b2m_mover_params& mp, uint64_t offset,
                          uint64_t n) {
  SpeciesLaunch L{};
  Species& S = ctx->sp[static_cast<size_t>(s)];
  if (ctx->mode == B2M_MODE_FAST) L.cells = S.cells;  // built by ensure_tables
  L.x = S.a[0] + offset; L.y = S.a[1] + offset; L.z = S.a[2] + offset;
  L.u = S.a[3] + offset; L.v = S.a[4] + offset; L.w = S.a[5] + offset;
  L.n = n;
  L.base = offset;
  L.dt = mp.dt;
  L.dto2 = 0.5 * mp.dt;
  L.beta = mp.beta;
  L.dto2_cell[0] = L.dto2 / ctx->grid.dx;
  L.dto2_cell[1] = L.dto2 / ctx->grid.dy;
  L.dto2_cell[2] = L.dto2 / ctx->grid.dz;
  L.rounds = mp.pc_iterations;
  L.species = s;
  L.col0 = offset;
  L.stride = S.stride;
  return L;
}

// STRICT: the per-cell corner node table of the current field (built on first
// use after every field change).
double* strict_nodes(b2m_ctx* ctx) {
  if (ctx->strict_gen != ctx->field_gen) {  // allocated at context creation
    launch_strict_nodes(ctx->grid.nx, ctx->grid.ny, ctx->grid.nz, ctx->dE, ctx->dB,
                        ctx->strict_nodes, ctx->stream);
    // the z-invariance flag of this field (the STRICT column kernel's test)
    if (ctx->zvar)
      launch_zinv_check(ctx->grid.nx, ctx->grid.ny, ctx->grid.nz, ctx->dE, ctx->dB, ctx->zvar,
                        ctx->stream);
    ctx->strict_gen = ctx->field_gen;
  }
  return ctx->strict_nodes;
}

// FAST: (re)build, in one launch, the beta-scaled cell tables of the given
// species whose field or beta changed since their last build.
void ensure_tables(b2m_ctx* ctx, const int* species, const b2m_mover_params* mp, int n) {
  if (ctx->mode != B2M_MODE_FAST) return;
  std::vector<double2*> tables;
  std::vector<double> scale;
  for (int m = 0; m < n; ++m) {
    Species& S = ctx->sp[static_cast<size_t>(species[m])];
    if (S.cells_gen == ctx->field_gen &&
        std::memcmp(&S.cells_beta, &mp[m].beta, sizeof(double)) == 0)
      continue;
    tables.push_back(S.cells);
    scale.push_back(mp[m].beta);
    S.cells_gen = ctx->field_gen;
    S.cells_beta = mp[m].beta;
  }
  if (!tables.empty())
    launch_field_to_cells(ctx->grid.nx, ctx->grid.ny, ctx->grid.nz, ctx->dE, ctx->dB,
                          scale.data(), tables.data(), static_cast<int>(tables.size()),
                          ctx->stream, ctx->zvar);
}

b2m_status check_params(const b2m_mover_params* mp) {
  if (!mp) return fail(B2M_INVALID_ARGUMENT, "null mover params");
  if (mp->pc_iterations < 1) return fail(B2M_CONFIG_ERROR, "pc_iterations: must be >= 1");
  return B2M_OK;
}

b2m_status reserve_sort(b2m_ctx* ctx);

b2m_status ensure_sort_scratch(b2m_ctx* ctx, uint64_t n) {
  if (n <= ctx->sort_cap) return B2M_OK;
  for (void* p : {static_cast<void*>(ctx->keys[0]), static_cast<void*>(ctx->keys[1]),
                  static_cast<void*>(ctx->vals[0]), static_cast<void*>(ctx->vals[1]),
                  static_cast<void*>(ctx->scratch), ctx->sort_temp}) {
    if (!p) continue;
    cudaFree(p);
    ctx->allocations.erase(std::remove(ctx->allocations.begin(), ctx->allocations.end(), p),
                           ctx->allocations.end());
  }
  ctx->sort_cap = 0;
  b2m_status st;
  for (int i = 0; i < 2; ++i) {
    if ((st = dalloc(ctx, &ctx->keys[i], n, "sort keys")) != B2M_OK) return st;
    if ((st = dalloc(ctx, &ctx->vals[i], n, "sort values")) != B2M_OK) return st;
  }
  if ((st = dalloc(ctx, &ctx->scratch, n, "sort scratch")) != B2M_OK) return st;
  ctx->sort_temp_bytes = sort_temp_bytes(n, 32);
  char* tmp = nullptr;
  if ((st = dalloc(ctx, &tmp, ctx->sort_temp_bytes, "sort temp")) != B2M_OK) return st;
  ctx->sort_temp = tmp;
  ctx->sort_cap = n;
  return B2M_OK;
}

// Everything the cell sort (b2m_sort_species) needs, allocated with the
// context so that no AllocError can appear mid-run (device_arena.cpp:20-55):
// per species a ping-pong set of the six arrays plus the counting sort's
// keys / bins / scan temp, or -- when the ping-pong sets do not fit (or
// B2M_SORT_FALLBACK=1) -- the radix-sort fallback's keys, values and one
// scratch array of the largest species.
b2m_status reserve_sort(b2m_ctx* ctx) {
  uint64_t cap = 0;
  for (const Species& S : ctx->sp) cap = std::max(cap, S.capacity);
  if (cap < 2) return B2M_OK;
  const uint64_t ncell = static_cast<uint64_t>(ctx->grid.nx) * ctx->grid.ny * ctx->grid.nz;
  b2m_status st;
  const char* fb = std::getenv("B2M_SORT_FALLBACK");
  bool pingpong = !(fb && fb[0] == '1');
  for (Species& S : ctx->sp) {
    if (!pingpong || S.capacity == 0) continue;
    double* blk = nullptr;
    if (cudaMalloc(reinterpret_cast<void**>(&blk), 6 * S.stride * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      pingpong = false;
      break;
    }
    ctx->allocations.push_back(blk);
    for (int a = 0; a < 6; ++a) S.alt[a] = blk + a * S.stride;
  }
  if (!pingpong) {  // release any partial ping-pong sets: the fallback serves every species
    for (Species& S : ctx->sp) {
      if (!S.alt[0]) continue;
      cudaFree(S.alt[0]);
      ctx->allocations.erase(
          std::remove(ctx->allocations.begin(), ctx->allocations.end(), S.alt[0]),
          ctx->allocations.end());
      for (auto& a : S.alt) a = nullptr;
    }
    return ensure_sort_scratch(ctx, cap);
  }
  if ((st = dalloc(ctx, &ctx->bin_keys, cap, "sort keys")) != B2M_OK) return st;
  ctx->bin_keys_cap = cap;
  if ((st = dalloc(ctx, &ctx->bin_count, ncell + 1, "sort bins")) != B2M_OK) return st;
  if ((st = dalloc(ctx, &ctx->bin_offs, ncell + 1, "sort bins")) != B2M_OK) return st;
  ctx->bin_temp_bytes = bin_scan_temp_bytes(ncell + 1);
  char* tmp = nullptr;
  if ((st = dalloc(ctx, &tmp, ctx->bin_temp_bytes, "sort scan temp")) != B2M_OK) return st;
  ctx->bin_temp = tmp;
  return B2M_OK;
}

}  // namespace b2m

extern "C" {

int b2m_abi_version(void) { return B2M_ABI_VERSION; }

const char* b2m_status_name(b2m_status s) {
  switch (s) {
    case B2M_OK: return "ok";
    case B2M_CONFIG_ERROR: return "ConfigError";
    case B2M_DOMAIN_ERROR: return "DomainError";
    case B2M_ALLOC_ERROR: return "AllocError";
    case B2M_NUMERICAL_FAULT: return "NumericalFault";
    case B2M_CFL_VIOLATION: return "CflViolation";
    case B2M_ENGINE_FAULT: return "EngineFault";
    case B2M_METRIC_ERROR: return "MetricError";
    case B2M_CUDA_ERROR: return "CudaError";
    case B2M_INVALID_ARGUMENT: return "InvalidArgument";
  }
  return "unknown";
}

const char* b2m_last_error(void) { return g_last_error.c_str(); }

int b2m_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

uint64_t b2m_launch_count(void) { return g_launches.load(); }

b2m_status b2m_grid_make(int nx, int ny, int nz, double lx, double ly, double lz,
                         b2m_grid* out) {
  if (!out) return fail(B2M_INVALID_ARGUMENT, "null grid");
  // grid.hpp:20-29
  if (nx < 2 || ny < 2 || nz < 2) return fail(B2M_CONFIG_ERROR, "grid: nx,ny,nz must each be >= 2");
  if (!(lx > 0.0) || !(ly > 0.0) || !(lz > 0.0))
    return fail(B2M_CONFIG_ERROR, "grid: lx,ly,lz must be positive");
  std::memset(out, 0, sizeof(*out));
  out->nx = nx; out->ny = ny; out->nz = nz;
  out->lx = lx; out->ly = ly; out->lz = lz;
  out->dx = lx / nx; out->dy = ly / ny; out->dz = lz / nz;
  return B2M_OK;
}

b2m_status b2m_mover_params_make(double dt, double qom, int pc_iterations,
                                 b2m_mover_params* out) {
  if (!out) return fail(B2M_INVALID_ARGUMENT, "null params");
  std::memset(out, 0, sizeof(*out));
  out->dt = dt;
  out->qom = qom;
  out->pc_iterations = pc_iterations;
  out->beta = qom * dt * 0.5;  // kernels.hpp:36-38
  return B2M_OK;
}

b2m_status b2m_set_device(int device) {
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaSetDevice");
  return B2M_OK;
}

b2m_status b2m_ctx_create(int device, const b2m_grid* g, int n_species, const uint64_t* capacity,
                          int mode, b2m_ctx** out) {
  if (!out || !g || (n_species > 0 && !capacity))
    return fail(B2M_INVALID_ARGUMENT, "null argument to b2m_ctx_create");
  *out = nullptr;
  if (n_species < 0 || n_species > 64) return fail(B2M_CONFIG_ERROR, "n_species out of range");
  if (mode != B2M_MODE_STRICT && mode != B2M_MODE_FAST)
    return fail(B2M_CONFIG_ERROR, "mode: unknown mover mode");
  if (g->nx < 2 || g->ny < 2 || g->nz < 2 || !(g->dx > 0) || !(g->dy > 0) || !(g->dz > 0))
    return fail(B2M_CONFIG_ERROR, "grid: invalid (use b2m_grid_make)");
  auto* ctx = new b2m_ctx();
  ctx->device = device;
  ctx->grid = *g;
  ctx->mode = mode;
  auto bail = [&](b2m_status st) {
    const std::string msg = g_last_error;
    b2m_ctx_destroy(ctx);
    g_last_error = msg;
    return st;
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete ctx;
    return fail(B2M_CUDA_ERROR, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  }
  if ((e = cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking)) != cudaSuccess) {
    cudaGetLastError();
    delete ctx;
    return fail(B2M_CUDA_ERROR, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
  }
  ctx->stream = ctx->own;
  for (auto& ev : ctx->ev) cudaEventCreate(&ev);
  const uint64_t nodes = static_cast<uint64_t>(g->nx + 1) * (g->ny + 1) * (g->nz + 1);
  const uint64_t ncell = static_cast<uint64_t>(g->nx) * g->ny * g->nz;
  ctx->n_nodes = nodes;
  b2m_status st;
  if ((st = dalloc(ctx, &ctx->dE, 3 * nodes, "field E")) != B2M_OK) return bail(st);
  if ((st = dalloc(ctx, &ctx->dB, 3 * nodes, "field B")) != B2M_OK) return bail(st);
  if ((st = dalloc(ctx, &ctx->strict_nodes, 48 * ncell, "strict node table")) != B2M_OK)
    return bail(st);
  if ((st = dalloc(ctx, &ctx->fault, 1, "fault word")) != B2M_OK) return bail(st);
  {
    const char* e3 = std::getenv("B2M_FAST_3D");  // diagnostics: general kernel only
    if (!(e3 && e3[0] == '1') && (st = dalloc(ctx, &ctx->zvar, 1, "z flag")) != B2M_OK)
      return bail(st);
  }
  if (cudaMallocHost(&ctx->fault_h, sizeof(FaultWord)) != cudaSuccess) {
    cudaGetLastError();
    return bail(fail(B2M_ALLOC_ERROR, "pinned fault word"));
  }
  ctx->sp.resize(static_cast<size_t>(n_species));
  for (int s = 0; s < n_species; ++s) {
    Species& S = ctx->sp[static_cast<size_t>(s)];
    S.capacity = capacity[s];
    S.stride = (S.capacity + 31) / 32 * 32;
    double* blk = nullptr;
    if ((st = dalloc(ctx, &blk, 6 * S.stride, "species arrays")) != B2M_OK) return bail(st);
    for (int a = 0; a < 6; ++a) S.a[a] = blk + a * S.stride;
    if ((st = dalloc(ctx, &S.cells, ncell * (kCellDoubles / 2), "field cells")) != B2M_OK)
      return bail(st);
  }
  if ((st = reserve_sort(ctx)) != B2M_OK) return bail(st);
  launch_fault_reset(ctx->fault, ctx->stream);
  if ((e = cudaStreamSynchronize(ctx->stream)) != cudaSuccess) {
    cuda_fail(ctx, e, "context init");
    return bail(B2M_CUDA_ERROR);
  }
  *out = ctx;
  return B2M_OK;
}

b2m_status b2m_ctx_destroy(b2m_ctx* ctx) {
  if (!ctx) return B2M_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (auto& c : ctx->stub)
    if (c.exec) cudaGraphExecDestroy(c.exec);
  for (void* p : ctx->allocations) cudaFree(p);
  if (ctx->mig_totals_h) cudaFreeHost(ctx->mig_totals_h);
  if (ctx->w.cnt_h) cudaFreeHost(ctx->w.cnt_h);
  if (ctx->w.red_h) cudaFreeHost(ctx->w.red_h);
  if (ctx->w.vin_h) cudaFreeHost(ctx->w.vin_h);
  if (ctx->w.bflag_h) cudaFreeHost(ctx->w.bflag_h);
  if (ctx->w.comm) nccl().CommDestroy(ctx->w.comm);
  if (ctx->fault_h) cudaFreeHost(ctx->fault_h);
  for (auto& ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : ctx->pipe_ev) cudaEventDestroy(ev);
  for (auto& ev : ctx->kt_ev) cudaEventDestroy(ev);
  if (ctx->up) cudaStreamDestroy(ctx->up);
  if (ctx->down) cudaStreamDestroy(ctx->down);
  if (ctx->own) cudaStreamDestroy(ctx->own);
  cudaGetLastError();
  delete ctx;
  return B2M_OK;
}

b2m_status b2m_ctx_set_stream(b2m_ctx* ctx, void* cuda_stream) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  ctx->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : ctx->own;
  return B2M_OK;
}

b2m_status b2m_ctx_set_mode(b2m_ctx* ctx, int mode) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (mode != B2M_MODE_STRICT && mode != B2M_MODE_FAST)
    return fail(B2M_CONFIG_ERROR, "mode: unknown mover mode");
  ctx->mode = mode;
  return B2M_OK;
}

b2m_status b2m_host_register(void* ptr, size_t bytes) {
  cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterDefault);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaHostRegister");
  return B2M_OK;
}

b2m_status b2m_host_unregister(void* ptr) {
  cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaHostUnregister");
  return B2M_OK;
}

b2m_status b2m_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(B2M_INVALID_ARGUMENT, "null out");
  cudaError_t e = cudaHostAlloc(out, bytes, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(B2M_ALLOC_ERROR, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
  }
  return B2M_OK;
}

b2m_status b2m_host_free(void* ptr) {
  cudaError_t e = cudaFreeHost(ptr);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaFreeHost");
  return B2M_OK;
}

// A new field: the FAST per-species tables are rebuilt on their next move.
static b2m_status relayout(b2m_ctx* ctx) {
  ++ctx->field_gen;
  ctx->field_ready = true;
  return B2M_OK;
}

b2m_status b2m_field_upload(b2m_ctx* ctx, const double* E, const double* B, uint64_t n_nodes) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (!E || !B) return fail(B2M_INVALID_ARGUMENT, "null field pointer");
  if (n_nodes != ctx->n_nodes)
    return fail(B2M_CONFIG_ERROR, "field: node count " + std::to_string(n_nodes) +
                                      " does not match the grid (" +
                                      std::to_string(ctx->n_nodes) + ")");
  const size_t bytes = 3 * n_nodes * sizeof(double);
  B2M_CUDA(ctx, cudaMemcpyAsync(ctx->dE, E, bytes, cudaMemcpyHostToDevice, ctx->stream));
  B2M_CUDA(ctx, cudaMemcpyAsync(ctx->dB, B, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return relayout(ctx);
}

b2m_status b2m_field_upload_device(b2m_ctx* ctx, const double* dE, const double* dB,
                                   uint64_t n_nodes) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (!dE || !dB) return fail(B2M_INVALID_ARGUMENT, "null field pointer");
  if (n_nodes != ctx->n_nodes) return fail(B2M_CONFIG_ERROR, "field: node count mismatch");
  const size_t bytes = 3 * n_nodes * sizeof(double);
  if (dE != ctx->dE)
    B2M_CUDA(ctx, cudaMemcpyAsync(ctx->dE, dE, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  if (dB != ctx->dB)
    B2M_CUDA(ctx, cudaMemcpyAsync(ctx->dB, dB, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  return relayout(ctx);
}

b2m_status b2m_field_device_ptrs(b2m_ctx* ctx, double** dE, double** dB) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (!dE || !dB) return fail(B2M_INVALID_ARGUMENT, "null output pointer");
  *dE = ctx->dE;
  *dB = ctx->dB;
  return B2M_OK;
}

b2m_status b2m_field_download(b2m_ctx* ctx, double* E, double* B) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (!E || !B) return fail(B2M_INVALID_ARGUMENT, "null field pointer");
  const size_t bytes = 3 * ctx->n_nodes * sizeof(double);
  B2M_CUDA(ctx, cudaMemcpyAsync(E, ctx->dE, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  B2M_CUDA(ctx, cudaMemcpyAsync(B, ctx->dB, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return b2m_sync(ctx, nullptr, nullptr);
}

b2m_status b2m_field_phase_stub(b2m_ctx* ctx, int passes) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (!ctx->field_ready) return fail(B2M_CONFIG_ERROR, "field stub: no field uploaded");
  if (passes <= 0) return B2M_OK;
  if (!ctx->dE_alt && (st = dalloc(ctx, &ctx->dE_alt, 3 * ctx->n_nodes, "field stub")) != B2M_OK)
    return st;
  // `passes` dependent launches of a ~µs kernel are launch-bound: capture them
  // once into a CUDA graph and replay it (re-captured when the pass count,
  // the ping-pong state or the stream changes)
  b2m_ctx::StubGraph* sg = nullptr;
  for (auto& c : ctx->stub)
    if (c.exec && c.passes == passes && c.in == ctx->dE && c.stream == ctx->stream) sg = &c;
  if (!sg) {
    sg = &ctx->stub[ctx->stub[0].exec && ctx->stub[0].in != ctx->dE ? 1 : 0];
    if (sg->exec) {
      cudaGraphExecDestroy(sg->exec);
      sg->exec = nullptr;
    }
    B2M_CUDA(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    double* out = launch_field_stub(ctx->grid.nx, ctx->grid.ny, ctx->grid.nz, ctx->dE, ctx->dB,
                                    ctx->dE_alt, passes, ctx->stream);
    note_launch(-(passes + 1));  // counted when the graph runs
    cudaGraph_t graph = nullptr;
    B2M_CUDA(ctx, cudaStreamEndCapture(ctx->stream, &graph));
    const cudaError_t e = cudaGraphInstantiate(&sg->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      sg->exec = nullptr;
      return cuda_fail(ctx, e, "cudaGraphInstantiate (field stub)");
    }
    sg->passes = passes;
    sg->in = ctx->dE;
    sg->stream = ctx->stream;
    sg->out = out;
  }
  B2M_CUDA(ctx, cudaGraphLaunch(sg->exec, ctx->stream));
  note_launch(passes + 1);
  if (sg->out != ctx->dE) std::swap(ctx->dE, ctx->dE_alt);
  B2M_CUDA(ctx, cudaGetLastError());
  return relayout(ctx);  // a new field: FAST tables rebuild on the next move
}

b2m_status b2m_field_phase_stub_host(const b2m_grid* g, double* E, double* B, int passes) {
  if (!g || !E || !B) return fail(B2M_INVALID_ARGUMENT, "null argument");
  if (passes <= 0) return B2M_OK;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaGetDevice");
  b2m_ctx* ctx = nullptr;
  b2m_status st = b2m_ctx_create(dev, g, 0, nullptr, B2M_MODE_STRICT, &ctx);
  if (st != B2M_OK) return st;
  const uint64_t nodes = static_cast<uint64_t>(g->nx + 1) * (g->ny + 1) * (g->nz + 1);
  if ((st = b2m_field_upload(ctx, E, B, nodes)) == B2M_OK &&
      (st = b2m_field_phase_stub(ctx, passes)) == B2M_OK)
    st = b2m_field_download(ctx, E, B);
  const std::string msg = g_last_error;
  b2m_ctx_destroy(ctx);
  g_last_error = msg;
  return st;
}

b2m_status b2m_species_upload_range(b2m_ctx* ctx, int s, const double* const* host6,
                                    uint64_t offset, uint64_t n) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if ((st = check_species(ctx, s)) != B2M_OK) return st;
  Species& S = ctx->sp[static_cast<size_t>(s)];
  if (offset + n > S.capacity)
    return fail(B2M_ALLOC_ERROR, "species " + std::to_string(s) + ": " +
                                     std::to_string(offset + n) + " particles exceed capacity " +
                                     std::to_string(S.capacity));
  if (n == 0) return B2M_OK;
  if (!host6) return fail(B2M_INVALID_ARGUMENT, "null host arrays");
  for (int a = 0; a < 6; ++a)
    B2M_CUDA(ctx, cudaMemcpyAsync(S.a[a] + offset, host6[a], n * sizeof(double),
                                  cudaMemcpyHostToDevice, ctx->stream));
  return B2M_OK;
}

b2m_status b2m_species_upload(b2m_ctx* ctx, int s, const double* const* host6, uint64_t n) {
  b2m_status st = b2m_species_upload_range(ctx, s, host6, 0, n);
  if (st == B2M_OK) ctx->sp[static_cast<size_t>(s)].count = n;
  return st;
}

b2m_status b2m_species_download_range(b2m_ctx* ctx, int s, double* const* host6, uint64_t offset,
                                      uint64_t n) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if ((st = check_species(ctx, s)) != B2M_OK) return st;
  Species& S = ctx->sp[static_cast<size_t>(s)];
  if (offset + n > S.capacity) return fail(B2M_INVALID_ARGUMENT, "download range beyond capacity");
  if (n == 0) return B2M_OK;
  if (!host6) return fail(B2M_INVALID_ARGUMENT, "null host arrays");
  for (int a = 0; a < 6; ++a)
    B2M_CUDA(ctx, cudaMemcpyAsync(host6[a], S.a[a] + offset, n * sizeof(double),
                                  cudaMemcpyDeviceToHost, ctx->stream));
  return B2M_OK;
}

b2m_status b2m_species_download(b2m_ctx* ctx, int s, double* const* host6, uint64_t max_n,
                                uint64_t* n_out) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if ((st = check_species(ctx, s)) != B2M_OK) return st;
  const uint64_t n = ctx->sp[static_cast<size_t>(s)].count;
  if (n_out) *n_out = n;
  if (n > max_n)
    return fail(B2M_ALLOC_ERROR, "download: host arrays hold " + std::to_string(max_n) +
                                     " particles, species has " + std::to_string(n));
  return b2m_species_download_range(ctx, s, host6, 0, n);
}

b2m_status b2m_species_set_count(b2m_ctx* ctx, int s, uint64_t n) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if ((st = check_species(ctx, s)) != B2M_OK) return st;
  Species& S = ctx->sp[static_cast<size_t>(s)];
  if (n > S.capacity) return fail(B2M_ALLOC_ERROR, "particle batch count > capacity");
  S.count = n;
  return B2M_OK;
}

b2m_status b2m_species_count(b2m_ctx* ctx, int s, uint64_t* n) {
  if (!ctx || !n) return fail(B2M_INVALID_ARGUMENT, "null argument");
  b2m_status st = check_species(ctx, s);
  if (st != B2M_OK) return st;
  *n = ctx->sp[static_cast<size_t>(s)].count;
  return B2M_OK;
}

b2m_status b2m_species_capacity(b2m_ctx* ctx, int s, uint64_t* cap) {
  if (!ctx || !cap) return fail(B2M_INVALID_ARGUMENT, "null argument");
  b2m_status st = check_species(ctx, s);
  if (st != B2M_OK) return st;
  *cap = ctx->sp[static_cast<size_t>(s)].capacity;
  return B2M_OK;
}

b2m_status b2m_species_device_ptrs(b2m_ctx* ctx, int s, double** out6) {
  if (!ctx || !out6) return fail(B2M_INVALID_ARGUMENT, "null argument");
  b2m_status st = check_species(ctx, s);
  if (st != B2M_OK) return st;
  for (int a = 0; a < 6; ++a) out6[a] = ctx->sp[static_cast<size_t>(s)].a[a];
  return B2M_OK;
}

b2m_status b2m_move_range(b2m_ctx* ctx, int s, const b2m_mover_params* mp, uint64_t offset,
                          uint64_t n) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if ((st = check_species(ctx, s)) != B2M_OK) return st;
  if ((st = check_params(mp)) != B2M_OK) return st;
  if (!ctx->field_ready) return fail(B2M_CONFIG_ERROR, "move: no field uploaded");
  Species& S = ctx->sp[static_cast<size_t>(s)];
  if (offset + n > S.count) return fail(B2M_INVALID_ARGUMENT, "move range beyond species count");
  ensure_tables(ctx, &s, mp, 1);
  const SpeciesLaunch L = make_launch(ctx, s, *mp, offset, n);
  if (ctx->mode == B2M_MODE_STRICT) {
    if (!launch_move_strict_tiles(to_dev(ctx->grid), to_fast(ctx->grid), strict_nodes(ctx), &L, 1, ctx->fault,
                                  ctx->stream, nullptr, nullptr, nullptr, ctx->zvar))
      return fail(B2M_CUDA_ERROR, "TMA tensor map setup failed (cuTensorMapEncodeTiled)");
  } else if (!launch_move_fast(to_fast(ctx->grid), &L, 1, ctx->fault, ctx->stream, nullptr,
                                      nullptr, nullptr, ctx->zvar)) {
    return fail(B2M_CUDA_ERROR, "TMA tensor map setup failed (cuTensorMapEncodeTiled)");
  }
  B2M_CUDA(ctx, cudaGetLastError());
  return B2M_OK;
}

b2m_status b2m_move(b2m_ctx* ctx, int s, const b2m_mover_params* mp) {
  if (!ctx) return fail(B2M_INVALID_ARGUMENT, "null context");
  b2m_status st = check_species(ctx, s);
  if (st != B2M_OK) return st;
  return b2m_move_range(ctx, s, mp, 0, ctx->sp[static_cast<size_t>(s)].count);
}

// b2m_move_all / b2m_move_deposit_all: qpp non-null = fused FAST deposit
static b2m_status move_all_impl(b2m_ctx* ctx, const b2m_mover_params* mp, const double* qpp) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (!mp) return fail(B2M_INVALID_ARGUMENT, "null mover params");
  if (!ctx->field_ready) return fail(B2M_CONFIG_ERROR, "move: no field uploaded");
  const int ns = static_cast<int>(ctx->sp.size());
  std::vector<SpeciesLaunch> L;
  std::vector<int> all(static_cast<size_t>(ns));
  for (int s = 0; s < ns; ++s) {
    if ((st = check_params(&mp[s])) != B2M_OK) return st;
    all[static_cast<size_t>(s)] = s;
  }
  ensure_tables(ctx, all.data(), mp, ns);
  // kernels.cpp:148,162: qv = q_per_particle * (1 / cell_volume)
  const double rvol = 1.0 / ((ctx->grid.dx * ctx->grid.dy) * ctx->grid.dz);
  for (int s = 0; s < ns; ++s) {
    L.push_back(make_launch(ctx, s, mp[s], 0, ctx->sp[static_cast<size_t>(s)].count));
    if (qpp) L.back().qv = qpp[s] * rvol;
  }
  const double* nodes = ctx->mode == B2M_MODE_STRICT ? strict_nodes(ctx) : nullptr;
  // slots 11 / 12 (and the kernel-timing log) bracket the mover launch(es)
  // alone, after any table rebuild
  B2M_CUDA(ctx, cudaEventRecord(ctx->ev[11], ctx->stream));
  const int kt = ctx->kt_n < ctx->kt_cap ? ctx->kt_n++ : -1;
  if (kt >= 0) B2M_CUDA(ctx, cudaEventRecord(ctx->kt_ev[2 * kt], ctx->stream));
  if (ctx->mode == B2M_MODE_STRICT) {
    if (!launch_move_strict_tiles(to_dev(ctx->grid), to_fast(ctx->grid), nodes, L.data(), ns,
                                  ctx->fault, ctx->stream, nullptr, nullptr, nullptr, ctx->zvar))
      return fail(B2M_CUDA_ERROR, "TMA tensor map setup failed (cuTensorMapEncodeTiled)");
  } else if (!launch_move_fast(to_fast(ctx->grid), L.data(), ns, ctx->fault, ctx->stream,
                               nullptr, nullptr, nullptr, ctx->zvar,
                               qpp ? ctx->mom : nullptr))
    return fail(B2M_CUDA_ERROR, "TMA tensor map setup failed (cuTensorMapEncodeTiled)");
  B2M_CUDA(ctx, cudaEventRecord(ctx->ev[12], ctx->stream));
  if (kt >= 0) B2M_CUDA(ctx, cudaEventRecord(ctx->kt_ev[2 * kt + 1], ctx->stream));
  B2M_CUDA(ctx, cudaGetLastError());
  return B2M_OK;
}

b2m_status b2m_move_all(b2m_ctx* ctx, const b2m_mover_params* mp) {
  return move_all_impl(ctx, mp, nullptr);
}

b2m_status b2m_move_deposit_all(b2m_ctx* ctx, const b2m_mover_params* mp,
                                const double* q_per_particle) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (!q_per_particle) return fail(B2M_INVALID_ARGUMENT, "null q_per_particle");
  if (!ctx->mom[0]) return fail(B2M_CONFIG_ERROR, "deposit: call b2m_moments_zero first");
  if (ctx->mode == B2M_MODE_FAST && !ctx->mom_pressure)
    return move_all_impl(ctx, mp, q_per_particle);
  // STRICT terms or the pressure tensor: the mover, then the deposit kernels
  if ((st = move_all_impl(ctx, mp, nullptr)) != B2M_OK) return st;
  for (int s = 0; s < static_cast<int>(ctx->sp.size()); ++s)
    if ((st = b2m_deposit(ctx, s, q_per_particle[s])) != B2M_OK) return st;
  return B2M_OK;
}

b2m_status b2m_kernel_timing_begin(b2m_ctx* ctx, int capacity) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (capacity < 0 || capacity > (1 << 20)) return fail(B2M_INVALID_ARGUMENT, "capacity");
  while (static_cast<int>(ctx->kt_ev.size()) < 2 * capacity) {
    cudaEvent_t e = nullptr;
    B2M_CUDA(ctx, cudaEventCreate(&e));
    ctx->kt_ev.push_back(e);
  }
  ctx->kt_cap = capacity;
  ctx->kt_n = 0;
  return B2M_OK;
}

b2m_status b2m_kernel_timing_read(b2m_ctx* ctx, float* ms, int max_n, int* n) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (!n || (max_n > 0 && !ms)) return fail(B2M_INVALID_ARGUMENT, "null argument");
  const int k = std::min(ctx->kt_n, max_n);
  for (int i = 0; i < k; ++i) {
    B2M_CUDA(ctx, cudaEventSynchronize(ctx->kt_ev[2 * i + 1]));
    B2M_CUDA(ctx, cudaEventElapsedTime(&ms[i], ctx->kt_ev[2 * i], ctx->kt_ev[2 * i + 1]));
  }
  *n = k;
  ctx->kt_cap = 0;
  ctx->kt_n = 0;
  return B2M_OK;
}

b2m_status b2m_run_mover_host(b2m_ctx* ctx, int n_species, double* const* host6_all,
                              const uint64_t* counts, const b2m_mover_params* mp, uint64_t chunk) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (!host6_all || !counts || !mp) return fail(B2M_INVALID_ARGUMENT, "null argument");
  if (n_species != static_cast<int>(ctx->sp.size()))
    return fail(B2M_CONFIG_ERROR, "run_mover: species count does not match the context");
  if (!ctx->field_ready) return fail(B2M_CONFIG_ERROR, "move: no field uploaded");
  if (chunk == 0) chunk = 1u << 21;
  for (int s = 0; s < n_species; ++s) {
    if ((st = check_params(&mp[s])) != B2M_OK) return st;
    if (counts[s] > ctx->sp[static_cast<size_t>(s)].capacity)
      return fail(B2M_ALLOC_ERROR, "species " + std::to_string(s) + ": " +
                                       std::to_string(counts[s]) + " particles exceed capacity");
  }
  if (!ctx->up) {
    B2M_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->up, cudaStreamNonBlocking));
    B2M_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->down, cudaStreamNonBlocking));
  }
  size_t n_chunks = 0;
  for (int s = 0; s < n_species; ++s) n_chunks += (counts[s] + chunk - 1) / chunk;
  while (ctx->pipe_ev.size() < 2 * n_chunks + 1) {
    cudaEvent_t e;
    B2M_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->pipe_ev.push_back(e);
  }
  // uploads start after everything already on the compute stream (field)
  cudaEvent_t* ev = ctx->pipe_ev.data();
  B2M_CUDA(ctx, cudaEventRecord(ev[2 * n_chunks], ctx->stream));
  B2M_CUDA(ctx, cudaStreamWaitEvent(ctx->up, ev[2 * n_chunks], 0));
  std::vector<int> all(static_cast<size_t>(n_species));
  for (int s = 0; s < n_species; ++s) all[static_cast<size_t>(s)] = s;
  ensure_tables(ctx, all.data(), mp, n_species);
  size_t c = 0;
  for (int s = 0; s < n_species; ++s) {
    Species& S = ctx->sp[static_cast<size_t>(s)];
    S.count = counts[s];
    double* const* h = host6_all + 6 * s;
    for (uint64_t off = 0; off < counts[s]; off += chunk, ++c) {
      const uint64_t n = std::min<uint64_t>(chunk, counts[s] - off);
      for (int a = 0; a < 6; ++a)
        B2M_CUDA(ctx, cudaMemcpyAsync(S.a[a] + off, h[a] + off, n * sizeof(double),
                                      cudaMemcpyHostToDevice, ctx->up));
      B2M_CUDA(ctx, cudaEventRecord(ev[2 * c], ctx->up));
      B2M_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ev[2 * c], 0));
      const SpeciesLaunch L = make_launch(ctx, s, mp[s], off, n);
      if (ctx->mode == B2M_MODE_STRICT) {
        if (!launch_move_strict_tiles(to_dev(ctx->grid), to_fast(ctx->grid), strict_nodes(ctx), &L, 1, ctx->fault,
                                      ctx->stream, nullptr, nullptr, nullptr, ctx->zvar))
          return fail(B2M_CUDA_ERROR, "TMA tensor map setup failed (cuTensorMapEncodeTiled)");
      } else if (!launch_move_fast(to_fast(ctx->grid), &L, 1, ctx->fault, ctx->stream, nullptr,
                                      nullptr, nullptr, ctx->zvar))
        return fail(B2M_CUDA_ERROR, "TMA tensor map setup failed (cuTensorMapEncodeTiled)");
      B2M_CUDA(ctx, cudaEventRecord(ev[2 * c + 1], ctx->stream));
      B2M_CUDA(ctx, cudaStreamWaitEvent(ctx->down, ev[2 * c + 1], 0));
      for (int a = 0; a < 6; ++a)
        B2M_CUDA(ctx, cudaMemcpyAsync(h[a] + off, S.a[a] + off, n * sizeof(double),
                                      cudaMemcpyDeviceToHost, ctx->down));
    }
  }
  B2M_CUDA(ctx, cudaGetLastError());
  B2M_CUDA(ctx, cudaStreamSynchronize(ctx->down));
  return b2m_sync(ctx, nullptr, nullptr);
}

b2m_status b2m_sort_species(b2m_ctx* ctx, int s) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if ((st = check_species(ctx, s)) != B2M_OK) return st;
  Species& S = ctx->sp[static_cast<size_t>(s)];
  const uint64_t n = S.count;
  if (n < 2) return B2M_OK;
  if (n > 0xffffffffull) return fail(B2M_CONFIG_ERROR, "sort: species larger than 2^32");
  const uint64_t ncell = static_cast<uint64_t>(ctx->grid.nx) * ctx->grid.ny * ctx->grid.nz;
  // every buffer below was reserved at b2m_ctx_create (reserve_sort): a
  // ping-pong set per species, or the radix-sort fallback's scratch
  if (S.alt[0]) {
    // counting sort straight into the ping-pong set, then swap
    launch_bin_sort(to_fast(ctx->grid), S.a, S.alt, n, ctx->bin_keys, ctx->bin_count,
                    ctx->bin_offs, ctx->bin_temp, ctx->bin_temp_bytes, ctx->stream);
    for (int a = 0; a < 6; ++a) std::swap(S.a[a], S.alt[a]);
    B2M_CUDA(ctx, cudaGetLastError());
    return B2M_OK;
  }
  // no memory for a second set: radix-sort (key, index) and gather array by
  // array through one scratch array
  if (n > ctx->sort_cap) return fail(B2M_ALLOC_ERROR, "sort: no scratch reserved");  // unreachable
  int bits = 1;
  while ((1ull << bits) <= ncell) ++bits;
  launch_cell_keys(to_fast(ctx->grid), S.a[0], S.a[1], S.a[2], n, ctx->keys[0], ctx->vals[0],
                   ctx->stream);
  launch_sort_pairs(ctx->sort_temp, ctx->sort_temp_bytes, ctx->keys[0], ctx->keys[1],
                    ctx->vals[0], ctx->vals[1], n, bits, ctx->stream);
  for (int a = 0; a < 6; ++a) {
    launch_gather(S.a[a], ctx->vals[1], n, ctx->scratch, ctx->stream);
    B2M_CUDA(ctx, cudaMemcpyAsync(S.a[a], ctx->scratch, n * sizeof(double),
                                  cudaMemcpyDeviceToDevice, ctx->stream));
  }
  B2M_CUDA(ctx, cudaGetLastError());
  return B2M_OK;
}

b2m_status b2m_sync(b2m_ctx* ctx, int* bad_species, int64_t* first_bad) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (bad_species) *bad_species = -1;
  if (first_bad) *first_bad = -1;
  B2M_CUDA(ctx, cudaMemcpyAsync(ctx->fault_h, ctx->fault, sizeof(FaultWord),
                                cudaMemcpyDeviceToHost, ctx->stream));
  B2M_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  const FaultWord f = *ctx->fault_h;
  if (f.numerical != ~0ull) {
    const int s = static_cast<int>(f.numerical >> 48);
    const int64_t i = static_cast<int64_t>(f.numerical & ((1ull << 48) - 1));
    if (bad_species) *bad_species = s;
    if (first_bad) *first_bad = i;
    ctx->poisoned = true;
    // kernels.cpp:71-72 / :98-99 message text
    ctx->poison_msg = "mover produced non-finite state at particle index " + std::to_string(i);
    return fail(B2M_NUMERICAL_FAULT, ctx->poison_msg);
  }
  if (f.domain != ~0ull) {
    const int s = static_cast<int>(f.domain >> 48);
    const int64_t i = static_cast<int64_t>(f.domain & ((1ull << 48) - 1));
    if (bad_species) *bad_species = s;
    if (first_bad) *first_bad = i;
    ctx->poisoned = true;
    // grid.hpp:67 message text
    ctx->poison_msg = "grid_cell_of: position outside domain (wrap first)";
    return fail(B2M_DOMAIN_ERROR, ctx->poison_msg);
  }
  if (f.cfl != ~0ull) {
    const int s = static_cast<int>(f.cfl >> 48);
    const int64_t i = static_cast<int64_t>(f.cfl & ((1ull << 48) - 1));
    if (bad_species) *bad_species = s;
    if (first_bad) *first_bad = i;
    double y = 0.0;
    cudaMemcpy(&y, ctx->sp[static_cast<size_t>(s)].a[1] + i, sizeof(double),
               cudaMemcpyDeviceToHost);
    const int dest = b2m_owner_of(&ctx->grid, ctx->sl.world, y);
    ctx->poisoned = true;
    // runtime.cpp:55-59 message text
    ctx->poison_msg = "particle " + std::to_string(i) + " of species " + std::to_string(s) +
                      " moved from slab " + std::to_string(ctx->sl.rank) +
                      " to non-neighbor slab " + std::to_string(dest) + " in one step";
    return fail(B2M_CFL_VIOLATION, ctx->poison_msg);
  }
  return B2M_OK;
}

b2m_status b2m_event_record(b2m_ctx* ctx, int slot) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (slot < 0 || slot >= kEventSlots) return fail(B2M_INVALID_ARGUMENT, "event slot");
  B2M_CUDA(ctx, cudaEventRecord(ctx->ev[slot], ctx->stream));
  return B2M_OK;
}

b2m_status b2m_event_elapsed_ms(b2m_ctx* ctx, int a, int b, float* ms) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (a < 0 || a >= kEventSlots || b < 0 || b >= kEventSlots || !ms)
    return fail(B2M_INVALID_ARGUMENT, "event slot");
  B2M_CUDA(ctx, cudaEventSynchronize(ctx->ev[b]));
  B2M_CUDA(ctx, cudaEventElapsedTime(ms, ctx->ev[a], ctx->ev[b]));
  return B2M_OK;
}

// ---- kernel-level one-shot ---------------------------------------------------

b2m_status b2m_move_batch_host(const b2m_grid* g, const b2m_mover_params* mp, const double* E,
                               const double* B, double* x, double* y, double* z, double* u,
                               double* v, double* w, uint64_t n, int mode, int64_t* first_bad) {
  if (first_bad) *first_bad = -1;
  if (!g || !mp || !E || !B) return fail(B2M_INVALID_ARGUMENT, "null argument");
  b2m_status st = check_params(mp);
  if (st != B2M_OK) return st;
  if (n == 0) return B2M_OK;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaGetDevice");
  // One cached context per host thread, reused while the grid, mode and
  // device match and the capacity suffices: a kernel-level caller moves every
  // species every cycle, and creating a context per call would dominate.
  struct Cache {
    b2m_ctx* ctx = nullptr;
    b2m_grid grid{};
    int mode = -1, dev = -1;
    uint64_t cap = 0;
    ~Cache() {
      if (ctx) b2m_ctx_destroy(ctx);
    }
  };
  thread_local Cache cache;
  if (cache.ctx && (cache.dev != dev || cache.mode != mode || cache.cap < n ||
                    std::memcmp(&cache.grid, g, sizeof(b2m_grid)) != 0)) {
    b2m_ctx_destroy(cache.ctx);
    cache.ctx = nullptr;
  }
  if (!cache.ctx) {
    const uint64_t cap = n;
    if ((st = b2m_ctx_create(dev, g, 1, &cap, mode, &cache.ctx)) != B2M_OK) {
      cache.ctx = nullptr;
      return st;
    }
    cache.grid = *g;
    cache.mode = mode;
    cache.dev = dev;
    cache.cap = cap;
  }
  b2m_ctx* ctx = cache.ctx;
  // a previous call's fault must not leak into this one
  ctx->poisoned = false;
  launch_fault_reset(ctx->fault, ctx->stream);
  const uint64_t nodes = static_cast<uint64_t>(g->nx + 1) * (g->ny + 1) * (g->nz + 1);
  const double* src[6] = {x, y, z, u, v, w};
  double* dst[6] = {x, y, z, u, v, w};
  int bad_s = -1;
  int64_t bad = -1;
  if ((st = b2m_field_upload(ctx, E, B, nodes)) == B2M_OK &&
      (st = b2m_species_upload(ctx, 0, src, n)) == B2M_OK &&
      (st = b2m_move(ctx, 0, mp)) == B2M_OK) {
    st = b2m_sync(ctx, &bad_s, &bad);
    if (st == B2M_OK || st == B2M_NUMERICAL_FAULT) {
      const std::string msg = g_last_error;
      // reference semantics: [0, bad) updated, [bad, n) untouched
      const uint64_t keep = st == B2M_OK ? n : static_cast<uint64_t>(bad);
      ctx->poisoned = false;
      b2m_status st2 = b2m_species_download_range(ctx, 0, dst, 0, keep);
      if (st2 == B2M_OK) {
        B2M_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
      }
      if (st == B2M_OK) st = st2;
      else g_last_error = msg;
      if (first_bad) *first_bad = bad;
    }
  }
  if (st != B2M_OK && st != B2M_NUMERICAL_FAULT) {  // unknown state: start afresh next time
    const std::string msg = g_last_error;
    b2m_ctx_destroy(cache.ctx);
    cache.ctx = nullptr;
    g_last_error = msg;
  }
  return st;
}

// ---- moments ------------------------------------------------------------------

b2m_status b2m_moments_zero(b2m_ctx* ctx, int with_pressure) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  const int na = with_pressure ? 10 : 4;
  const uint64_t nodes = static_cast<uint64_t>(ctx->grid.nx) * ctx->grid.ny * ctx->grid.nz;
  if (ctx->mom_arrays < na) {
    double* blk = nullptr;
    if ((st = dalloc(ctx, &blk, na * nodes, "moment mesh")) != B2M_OK) return st;
    for (int a = 0; a < 10; ++a) ctx->mom[a] = a < na ? blk + a * nodes : nullptr;
    ctx->mom_arrays = na;
    if ((st = world_reserve_moments(ctx, na * nodes)) != B2M_OK) return st;
  }
  for (int a = 0; a < na; ++a)
    B2M_CUDA(ctx, cudaMemsetAsync(ctx->mom[a], 0, nodes * sizeof(double), ctx->stream));
  ctx->mom_pressure = with_pressure != 0;
  return B2M_OK;
}

b2m_status b2m_deposit(b2m_ctx* ctx, int s, double q_per_particle) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if ((st = check_species(ctx, s)) != B2M_OK) return st;
  if (!ctx->mom[0]) return fail(B2M_CONFIG_ERROR, "deposit: call b2m_moments_zero first");
  Species& S = ctx->sp[static_cast<size_t>(s)];
  SpeciesLaunch L{};
  L.x = S.a[0]; L.y = S.a[1]; L.z = S.a[2];
  L.u = S.a[3]; L.v = S.a[4]; L.w = S.a[5];
  L.n = S.count;
  L.species = s;
  // kernels.cpp:148,162: qv = q_per_particle * (1 / cell_volume)
  const double qv = q_per_particle * (1.0 / ((ctx->grid.dx * ctx->grid.dy) * ctx->grid.dz));
  launch_deposit(to_dev(ctx->grid), L, qv, ctx->mom, ctx->mom_pressure,
                 ctx->mode == B2M_MODE_STRICT, ctx->fault, ctx->stream);
  B2M_CUDA(ctx, cudaGetLastError());
  return B2M_OK;
}

b2m_status b2m_moments_download(b2m_ctx* ctx, double* const* out, int n_arrays) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (!out || n_arrays < 1 || n_arrays > (ctx->mom_pressure ? 10 : 4) || !ctx->mom[0])
    return fail(B2M_INVALID_ARGUMENT, "moments_download: bad array count or no mesh");
  const uint64_t nodes = static_cast<uint64_t>(ctx->grid.nx) * ctx->grid.ny * ctx->grid.nz;
  for (int a = 0; a < n_arrays; ++a)
    B2M_CUDA(ctx, cudaMemcpyAsync(out[a], ctx->mom[a], nodes * sizeof(double),
                                  cudaMemcpyDeviceToHost, ctx->stream));
  return b2m_sync(ctx, nullptr, nullptr);
}

b2m_status b2m_moments_device_ptr(b2m_ctx* ctx, double** d_mesh, uint64_t* n_doubles) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (!d_mesh || !n_doubles) return fail(B2M_INVALID_ARGUMENT, "null argument");
  if (!ctx->mom[0]) return fail(B2M_CONFIG_ERROR, "moments: call b2m_moments_zero first");
  const uint64_t nodes = static_cast<uint64_t>(ctx->grid.nx) * ctx->grid.ny * ctx->grid.nz;
  *d_mesh = ctx->mom[0];
  *n_doubles = static_cast<uint64_t>(ctx->mom_pressure ? 10 : 4) * nodes;
  return B2M_OK;
}

b2m_status b2m_deposit_moments_host(const b2m_grid* g, const double* x, const double* y,
                                    const double* z, const double* u, const double* v,
                                    const double* w, uint64_t n, double q_per_particle,
                                    int with_pressure, double* const* out) {
  if (!g || !out) return fail(B2M_INVALID_ARGUMENT, "null argument");
  if (n == 0) return B2M_OK;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaGetDevice");
  b2m_ctx* ctx = nullptr;
  const uint64_t cap = n;
  b2m_status st = b2m_ctx_create(dev, g, 1, &cap, B2M_MODE_STRICT, &ctx);
  if (st != B2M_OK) return st;
  const double* src[6] = {x, y, z, u, v, w};
  const int na = with_pressure ? 10 : 4;
  const uint64_t nodes = static_cast<uint64_t>(g->nx) * g->ny * g->nz;
  std::vector<double> host(static_cast<size_t>(na) * nodes);
  std::vector<double*> dst(static_cast<size_t>(na));
  for (int a = 0; a < na; ++a) dst[static_cast<size_t>(a)] = host.data() + a * nodes;
  if ((st = b2m_species_upload(ctx, 0, src, n)) == B2M_OK &&
      (st = b2m_moments_zero(ctx, with_pressure)) == B2M_OK &&
      (st = b2m_deposit(ctx, 0, q_per_particle)) == B2M_OK &&
      (st = b2m_moments_download(ctx, dst.data(), na)) == B2M_OK) {
    // MomentMesh& out accumulates (kernels.cpp:169-180)
    for (int a = 0; a < na; ++a)
      for (uint64_t i = 0; i < nodes; ++i) out[a][i] += dst[static_cast<size_t>(a)][i];
  }
  const std::string msg = g_last_error;
  b2m_ctx_destroy(ctx);
  g_last_error = msg;
  return st;
}

// ---- partition layer ----------------------------------------------------------

int b2m_owner_of(const b2m_grid* g, int world, double y) {
  // runtime.cpp:39-44
  int j = static_cast<int>(y / g->dy);
  if (j >= g->ny) j = g->ny - 1;
  if (j < 0) j = 0;
  return j / (g->ny / world);
}

b2m_status b2m_slab_config(b2m_ctx* ctx, int rank, int world) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  // runtime.cpp:22-37 decompose
  if (world < 1) return fail(B2M_CONFIG_ERROR, "workers: must be >= 1");
  if (ctx->grid.ny % world != 0)
    return fail(B2M_CONFIG_ERROR, "workers: " + std::to_string(world) +
                                      " does not divide ny=" + std::to_string(ctx->grid.ny));
  const int slab = ctx->grid.ny / world;
  if (slab < 2)
    return fail(B2M_CONFIG_ERROR, "workers: slab would be " + std::to_string(slab) +
                                      " cells; each slab needs at least 2");
  if (rank < 0 || rank >= world) return fail(B2M_CONFIG_ERROR, "rank out of range");
  ctx->sl.rank = rank;
  ctx->sl.world = world;
  ctx->sl.prev = (rank + world - 1) % world;
  ctx->sl.next = (rank + 1) % world;
  ctx->sl.slab = slab;
  ctx->sl.dy = ctx->grid.dy;
  ctx->sl.ny = ctx->grid.ny;
  // y-range of slab r under owner_of (runtime.cpp:39-44): trunc(RN(y/dy))
  // reaches m exactly from the smallest y with RN(y/dy) >= m on (RN(y/dy) is
  // monotone in y); the last slab also takes the clamped j >= ny
  auto first_y = [&](int m) {
    if (m <= 0) return 0.0;
    uint64_t lo = 0, hi = 0;
    const double top = 2.0 * ctx->grid.ly;
    std::memcpy(&hi, &top, sizeof(double));
    while (lo < hi) {  // smallest bit pattern with (y / dy) >= m
      const uint64_t mid = lo + (hi - lo) / 2;
      double y;
      std::memcpy(&y, &mid, sizeof(double));
      if (y / ctx->grid.dy >= static_cast<double>(m))
        hi = mid;
      else
        lo = mid + 1;
    }
    double y;
    std::memcpy(&y, &lo, sizeof(double));
    return y;
  };
  auto range = [&](int r, double& a, double& b) {
    a = first_y(r * slab);
    b = r == world - 1 ? std::numeric_limits<double>::infinity() : first_y((r + 1) * slab);
  };
  range(rank, ctx->sl.own_lo, ctx->sl.own_hi);
  range(ctx->sl.prev, ctx->sl.prev_lo, ctx->sl.prev_hi);
  range(ctx->sl.next, ctx->sl.next_lo, ctx->sl.next_hi);
  ctx->slab_on = true;
  // migration scratch (once per context)
  if (ctx->mig_tcnt) return B2M_OK;
  const size_t ns = ctx->sp.size();
  if (ns > static_cast<size_t>(kMaxCompactSpecies))
    return fail(B2M_CONFIG_ERROR, "migration: at most " + std::to_string(kMaxCompactSpecies) +
                                      " species");
  ctx->mig_tile0.assign(ns, 0);
  uint64_t tiles = 0;
  for (size_t s = 0; s < ns; ++s) {
    ctx->mig_tile0[s] = tiles;
    tiles += std::max<uint64_t>(1, migrate_tiles(ctx->sp[s].capacity));
  }
  if ((st = dalloc(ctx, &ctx->mig_tcnt, tiles, "tile counts")) != B2M_OK) return st;
  if ((st = dalloc(ctx, &ctx->mig_toff, tiles, "tile offsets")) != B2M_OK) return st;
  if ((st = dalloc(ctx, &ctx->mig_totals, 3 * ns, "migration totals")) != B2M_OK) return st;
  B2M_CUDA(ctx, cudaMemsetAsync(ctx->mig_tcnt, 0, tiles * sizeof(unsigned long long),
                                ctx->stream));  // ordered with the movers on ctx->stream
  if (cudaMallocHost(&ctx->mig_totals_h, 3 * ns * sizeof(unsigned long long)) != cudaSuccess) {
    cudaGetLastError();
    return fail(B2M_ALLOC_ERROR, "pinned migration totals");
  }
  std::memset(ctx->mig_totals_h, 0, 3 * ns * sizeof(unsigned long long));
  for (size_t s = 0; s < ns; ++s) {
    Species& S = ctx->sp[s];
    const uint64_t cap = S.capacity;
    // outboxes of half the capacity: a slab boundary can cut through the
    // whole Harris sheet (world 2), and a heated state (the benchmark's
    // gem_like_field E accelerates electrons every cycle) migrates far more
    // than the physical ~0.2 % per cycle
    S.cap_out = std::max<uint64_t>(std::min<uint64_t>(cap, 1u << 16), cap / 2);
    // the movers and the compaction only test S.flags for null (owner scan
    // on); leavers are re-derived from y, so no per-particle byte is stored
    if ((st = dalloc(ctx, &S.flags, 1, "migration marker")) != B2M_OK) return st;
    if ((st = dalloc(ctx, &S.out[0], 6 * S.cap_out, "outbox prev")) != B2M_OK) return st;
    if ((st = dalloc(ctx, &S.out[1], 6 * S.cap_out, "outbox next")) != B2M_OK) return st;
    if ((st = dalloc(ctx, &S.holes, cap, "hole list")) != B2M_OK) return st;
    S.tcnt = ctx->mig_tcnt + ctx->mig_tile0[s];
    S.toff = ctx->mig_toff + ctx->mig_tile0[s];
    S.totals = ctx->mig_totals + 3 * s;
    S.totals_h = ctx->mig_totals_h + 3 * s;
  }
  const size_t need = scan_temp_bytes(tiles);
  if (need > ctx->scan_temp_bytes) {
    char* tmp = nullptr;
    if ((st = dalloc(ctx, &tmp, need, "scan temp")) != B2M_OK) return st;
    ctx->scan_temp = tmp;
    ctx->scan_temp_bytes = need;
  }
  return B2M_OK;
}

// Migration bookkeeping after the mover wrote the flags and tile counts of
// the given species: one scan over their (side by side) tile counts, every
// species' totals, the outbox + hole scatter, and one copy of all totals back.
static b2m_status migrate_compact(b2m_ctx* ctx, const int* species, const SpeciesLaunch* L,
                                  int n) {
  CompactSet C{};
  C.n = n;
  for (int m = 0; m < n; ++m) {
    const int s = species[m];
    Species& S = ctx->sp[static_cast<size_t>(s)];
    CompactSpecies& c = C.s[m];
    c.sp = L[m];
    c.flags = S.flags;
    c.out_prev = S.out[0];
    c.out_next = S.out[1];
    c.cap_out = S.cap_out;
    c.holes = S.holes;
    c.totals = S.totals;
    c.tile0 = ctx->mig_tile0[static_cast<size_t>(s)];
    c.n_tiles = migrate_tiles(S.count);  // 0 for an empty species: zero totals
  }
  C.sl = ctx->sl;
  launch_compact(C, ctx->scan_temp, ctx->scan_temp_bytes, ctx->mig_tcnt, ctx->mig_toff,
                 ctx->stream);
  B2M_CUDA(ctx, cudaMemcpyAsync(ctx->mig_totals_h, ctx->mig_totals,
                                3 * ctx->sp.size() * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, ctx->stream));
  return B2M_OK;
}

}  // extern "C"


// The mover over `n` species in ONE launch, fused with the owner scan (each
// particle gets its destination flag), then each species' compaction.
b2m_status b2m::move_migrate_species(b2m_ctx* ctx, const int* species,
                                      const b2m_mover_params* mp, int n) {
  b2m_status st;
  if (!ctx->slab_on) return fail(B2M_CONFIG_ERROR, "move_migrate: call b2m_slab_config first");
  if (!ctx->field_ready) return fail(B2M_CONFIG_ERROR, "move: no field uploaded");
  ensure_tables(ctx, species, mp, n);
  std::vector<SpeciesLaunch> L, all;
  std::vector<uint8_t*> fl;
  std::vector<unsigned long long*> tc;
  for (int m = 0; m < n; ++m) {
    const int s = species[m];
    Species& S = ctx->sp[static_cast<size_t>(s)];
    S.pre_count = S.count;
    S.migrate_pending = true;
    all.push_back(make_launch(ctx, s, mp[m], 0, S.count));
    if (S.count == 0) continue;  // no mover work; its totals come back zero
    L.push_back(all.back());
    fl.push_back(S.flags);
    tc.push_back(S.tcnt);
  }
  if (L.empty()) {
    for (int m = 0; m < n; ++m)
      std::memset(ctx->sp[static_cast<size_t>(species[m])].totals_h, 0,
                  3 * sizeof(unsigned long long));
    return B2M_OK;
  }
  const int nl = static_cast<int>(L.size());
  const bool ok =
      ctx->mode == B2M_MODE_STRICT
          ? launch_move_strict_tiles(to_dev(ctx->grid), to_fast(ctx->grid), strict_nodes(ctx),
                                     L.data(), nl, ctx->fault, ctx->stream, &ctx->sl, fl.data(),
                                     tc.data(), ctx->zvar)
          : launch_move_fast(to_fast(ctx->grid), L.data(), nl, ctx->fault, ctx->stream, &ctx->sl,
                             fl.data(), tc.data(), ctx->zvar);
  if (!ok) return fail(B2M_CUDA_ERROR, "TMA tensor map setup failed (cuTensorMapEncodeTiled)");
  if ((st = migrate_compact(ctx, species, all.data(), n)) != B2M_OK) return st;
  B2M_CUDA(ctx, cudaGetLastError());
  return B2M_OK;
}

extern "C" {

b2m_status b2m_move_migrate(b2m_ctx* ctx, int s, const b2m_mover_params* mp) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if ((st = check_species(ctx, s)) != B2M_OK) return st;
  if ((st = check_params(mp)) != B2M_OK) return st;
  return move_migrate_species(ctx, &s, mp, 1);
}

b2m_status b2m_move_migrate_all(b2m_ctx* ctx, const b2m_mover_params* mp) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if (!mp) return fail(B2M_INVALID_ARGUMENT, "null mover params");
  const int ns = static_cast<int>(ctx->sp.size());
  std::vector<int> all(static_cast<size_t>(ns));
  for (int s = 0; s < ns; ++s) {
    if ((st = check_params(&mp[s])) != B2M_OK) return st;
    all[static_cast<size_t>(s)] = s;
  }
  return move_migrate_species(ctx, all.data(), mp, ns);
}

b2m_status b2m_outbox(b2m_ctx* ctx, int s, int dir, double** d_recs, uint64_t* count) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if ((st = check_species(ctx, s)) != B2M_OK) return st;
  if (dir != 0 && dir != 1) return fail(B2M_INVALID_ARGUMENT, "dir must be 0 (prev) or 1 (next)");
  Species& S = ctx->sp[static_cast<size_t>(s)];
  if (!S.migrate_pending) return fail(B2M_CONFIG_ERROR, "outbox: no migration step pending");
  const uint64_t n = S.totals_h[dir];
  if (n > S.cap_out) {
    ctx->poisoned = true;
    ctx->poison_msg = "outbox capacity exceeded (" + std::to_string(n) + " > " +
                      std::to_string(S.cap_out) + ")";
    return fail(B2M_ALLOC_ERROR, ctx->poison_msg);
  }
  if (d_recs) *d_recs = S.out[dir];
  if (count) *count = n;
  return B2M_OK;
}

b2m_status b2m_inbox_append(b2m_ctx* ctx, int s, const double* d_recs, uint64_t n) {
  b2m_status st = check_ctx(ctx);
  if (st != B2M_OK) return st;
  if ((st = check_species(ctx, s)) != B2M_OK) return st;
  Species& S = ctx->sp[static_cast<size_t>(s)];
  if (n > 0 && !d_recs) return fail(B2M_INVALID_ARGUMENT, "null inbox");
  uint64_t holes = 0;
  uint64_t old_n = S.count;
  if (S.migrate_pending) {
    holes = S.totals_h[2];
    old_n = S.pre_count;
  }
  const uint64_t new_n = old_n - holes + n;
  if (new_n > S.capacity)
    return fail(B2M_ALLOC_ERROR, "particle batch capacity exceeded (fixed at allocation)");
  SpeciesLaunch L{};
  L.x = S.a[0]; L.y = S.a[1]; L.z = S.a[2];
  L.u = S.a[3]; L.v = S.a[4]; L.w = S.a[5];
  L.stride = S.stride;
  L.n = old_n;
  L.species = s;
  if (S.migrate_pending) {
    launch_fill(L, S.holes, holes, d_recs, n, ctx->sl, ctx->stream);
  } else if (n > 0) {
    // plain append: no holes
    launch_fill(L, S.holes, 0, d_recs, n, ctx->sl, ctx->stream);
  }
  B2M_CUDA(ctx, cudaGetLastError());
  S.count = new_n;
  S.migrate_pending = false;
  return B2M_OK;
}


}  // extern "C"
