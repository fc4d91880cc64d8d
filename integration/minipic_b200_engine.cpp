// minipic_b200_engine.cpp — the reference-side plug-in a maintainer adds to
// minipic (/root/reference/proj) to run its mover on B200s.
//
// It implements the reference's pic::Engine interface (engines.hpp:20-48) on
// top of the libb2m C ABI (include/b2m.h) and replaces the factory
// pic::make_engine (engines.cpp:204-212) with a dispatcher:
//
//   * B2M_ENGINE unset/0  -> the reference's own engines (ref_make_engine,
//                            i.e. engines.cpp compiled with
//                            -Dmake_engine=ref_make_engine, unmodified)
//   * B2M_ENGINE=1        -> every offload kind (naive/pinned/prefetch) runs
//                            on a B200; kind cpu stays the reference CPU mover
//
// B2M_MODE=strict (default here) makes the engine bit-identical to the
// reference CPU engine -- the contract of engines.hpp:18-19 -- and
// B2M_MODE=fast selects the FMA kernel (1e-12 contract).
//
// make_engine receives no worker id, so engines are mapped to GPUs in
// creation order modulo the device count (Simulation::distribute creates them
// in worker order, runtime.cpp:168-171).  Every libb2m call binds the
// context's device, so the reference's per-cycle worker threads
// (runtime.cpp:199-202) may drive the engine from any thread.
//
// Nothing in /root/reference is modified; the build recipe is
// integration/Makefile.
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "b2m.h"
#include "minipic/engines.hpp"
#include "minipic/errors.hpp"

namespace pic {

// engines.cpp compiled with -Dmake_engine=ref_make_engine
std::unique_ptr<Engine> ref_make_engine(EngineKind kind, const SimConfig& cfg);

namespace {

std::atomic<int> g_engine_counter{0};

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

class B200Engine final : public Engine {
 public:
  B200Engine(EngineKind kind, const SimConfig& cfg) : kind_(kind), grid_(cfg.grid) {
    const int ndev = b2m_device_count();
    if (ndev < 1) throw EngineFault("B200 engine: no CUDA device visible");
    device_ = g_engine_counter.fetch_add(1) % ndev;
    const char* m = std::getenv("B2M_MODE");
    mode_ = (m && std::strcmp(m, "fast") == 0) ? B2M_MODE_FAST : B2M_MODE_STRICT;
    static_assert(sizeof(b2m_grid) == sizeof(Grid), "b2m_grid mirrors pic::Grid");
    static_assert(sizeof(b2m_mover_params) == sizeof(MoverParams),
                  "b2m_mover_params mirrors pic::MoverParams");
  }

  ~B200Engine() override {
    for (void* p : pinned_) b2m_host_unregister(p);
    if (ctx_) b2m_ctx_destroy(ctx_);
  }

  EngineKind kind() const override { return kind_; }

  // DeviceArena::configure equivalent: all device memory carved up front
  // (AllocError now, never mid-run), grid constants uploaded.
  void prime(const FieldMesh& field, std::vector<ParticleBatch>& batches) override {
    std::vector<uint64_t> caps;
    for (const ParticleBatch& b : batches) caps.push_back(b.capacity());
    b2m_grid g;
    std::memcpy(&g, &grid_, sizeof(g));
    check(b2m_ctx_create(device_, &g, static_cast<int>(caps.size()), caps.data(), mode_, &ctx_),
          "prime");
    // pinned / prefetch kinds: page-lock the batches' own arrays in place
    // (their capacity is fixed at allocation, particle_batch.hpp:29-34), so
    // the per-cycle copies run at full PCIe speed straight from / into them;
    // the naive kind keeps pageable copies, as NaiveEngine does
    if (kind_ != EngineKind::naive) {
      for (ParticleBatch& b : batches) {
        double* a[6] = {b.xs(), b.ys(), b.zs(), b.us(), b.vs(), b.ws()};
        for (double* p : a)
          if (p && b.capacity() &&
              b2m_host_register(p, b.capacity() * sizeof(double)) == B2M_OK)
            pinned_.push_back(p);  // best effort: pageable copies still work
      }
    }
    stage_next(field, batches);
  }

  // PrefetchEngine::stage_next analogue (engines.cpp:169-173): the next
  // cycle's field is uploaded while the host runs moments/field work.
  void stage_next(const FieldMesh& field, const std::vector<ParticleBatch>&) override {
    const double t = log_.now();
    check(b2m_field_upload(ctx_, reinterpret_cast<const double*>(field.E.data()),
                           reinterpret_cast<const double*>(field.B.data()), field.node_count()),
          "field upload");
    log_.append({log_.next_seq(), CommandKind::copy_to_device, -1,
                 2 * field.node_count() * sizeof(Vec3), t, t, log_.now()});
    staged_ = true;
  }

  // Blocking: on return every batch holds its moved particles
  // (engines.hpp:35-37).  Species flow through the chunked
  // H2D -> kernel -> D2H pipeline of b2m_run_mover_host.
  void run_mover(const FieldMesh& field, std::vector<ParticleBatch>& batches,
                 const std::vector<MoverParams>& mp) override {
    if (!ctx_) prime(field, batches);
    if (!staged_) stage_next(field, batches);
    staged_ = false;
    const int ns = static_cast<int>(batches.size());
    std::vector<double*> ptrs(6 * static_cast<size_t>(ns));
    std::vector<uint64_t> counts(static_cast<size_t>(ns));
    std::vector<b2m_mover_params> params(static_cast<size_t>(ns));
    for (int s = 0; s < ns; ++s) {
      ParticleBatch& b = batches[static_cast<size_t>(s)];
      double* a[6] = {b.xs(), b.ys(), b.zs(), b.us(), b.vs(), b.ws()};
      for (int k = 0; k < 6; ++k) ptrs[6 * static_cast<size_t>(s) + k] = a[k];
      counts[static_cast<size_t>(s)] = b.count();
      std::memcpy(&params[static_cast<size_t>(s)], &mp[static_cast<size_t>(s)],
                  sizeof(b2m_mover_params));
    }
    const double t = log_.now();
    check(b2m_run_mover_host(ctx_, ns, ptrs.data(), counts.data(), params.data(), 0),
          "run_mover");
    for (int s = 0; s < ns; ++s)
      log_.append({log_.next_seq(), CommandKind::run_mover, s,
                   2 * batches[static_cast<size_t>(s)].bytes(), t, t, log_.now()});
  }

 private:
  // Offload faults surface as EngineFault and poison the engine, like the
  // reference's queue (command_queue.cpp:45-49, test_offload.cpp:464-481);
  // capacity problems stay AllocError, configuration problems ConfigError.
  void check(b2m_status st, const char* what) {
    if (st == B2M_OK) return;
    const std::string msg = std::string("B200 engine ") + what + ": " + b2m_last_error();
    if (st == B2M_ALLOC_ERROR) throw AllocError(msg);
    if (st == B2M_CONFIG_ERROR) throw ConfigError(msg);
    throw EngineFault(msg);
  }

  EngineKind kind_;
  Grid grid_;
  int device_ = 0;
  int mode_ = B2M_MODE_STRICT;
  b2m_ctx* ctx_ = nullptr;
  bool staged_ = false;
  std::vector<void*> pinned_;
};

}  // namespace

std::unique_ptr<Engine> make_engine(EngineKind kind, const SimConfig& cfg) {
  if (env_int("B2M_ENGINE", 0) != 0 && kind != EngineKind::cpu)
    return std::make_unique<B200Engine>(kind, cfg);
  return ref_make_engine(kind, cfg);
}

}  // namespace pic
