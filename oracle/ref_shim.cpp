// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" shim over the UNMODIFIED reference library (minipic), compiled
// from /root/reference/proj/src/*.cpp by oracle/Makefile into
// oracle/_ref/libminipic_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load it, and only as the
// checker or the timed CPU baseline -- never as the product path.
//
// Every entry point forwards to the reference's own public API:
//   ref_move_batch      -> pic::move_batch            (kernels.cpp:52-104)
//   ref_move_batch_mt   -> pic::move_batch on T disjoint ParticleSpan slices
//                          (SURVEY §8d CPU baseline (ii); kernels.hpp:46-48
//                          says spans are independent and reentrant)
//   ref_init_gem        -> pic::init_gem              (init.cpp:62-102)
//   ref_wrap_len        -> pic::wrap_len              (grid.hpp:45-50)
//   ref_grid_cell_of    -> pic::grid_cell_of          (grid.hpp:64-82)
//   ref_sim_*           -> pic::Simulation            (runtime.cpp:125-289)
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "minipic/bench.hpp"
#include "minipic/errors.hpp"
#include "minipic/grid.hpp"
#include "minipic/init.hpp"
#include "minipic/kernels.hpp"
#include "minipic/runtime.hpp"
#include "minipic/sim_config.hpp"

using namespace pic;

namespace {

// Status codes shared with include/b2m.h (b2m_status).
enum {
  kOk = 0,
  kConfig = 1,
  kDomain = 2,
  kAlloc = 3,
  kNumerical = 4,
  kCfl = 5,
  kEngine = 6,
  kMetric = 7,
  kOther = 99,
};

void put(char* err, int errlen, const char* msg) {
  if (err && errlen > 0) {
    std::strncpy(err, msg, std::size_t(errlen) - 1);
    err[errlen - 1] = 0;
  }
}

int map_exception(std::exception_ptr ep, char* err, int errlen) {
  try {
    std::rethrow_exception(ep);
  } catch (const ConfigError& e) {
    put(err, errlen, e.what());
    return kConfig;
  } catch (const DomainError& e) {
    put(err, errlen, e.what());
    return kDomain;
  } catch (const AllocError& e) {
    put(err, errlen, e.what());
    return kAlloc;
  } catch (const NumericalFault& e) {
    put(err, errlen, e.what());
    return kNumerical;
  } catch (const CflViolation& e) {
    put(err, errlen, e.what());
    return kCfl;
  } catch (const EngineFault& e) {
    put(err, errlen, e.what());
    return kEngine;
  } catch (const MetricError& e) {
    put(err, errlen, e.what());
    return kMetric;
  } catch (const std::exception& e) {
    put(err, errlen, e.what());
    return kOther;
  }
}

#define SHIM_TRY try {
#define SHIM_CATCH                                     \
  }                                                    \
  catch (...) {                                        \
    return map_exception(std::current_exception(), err, errlen); \
  }                                                    \
  return kOk;

FieldView view_of(const double* E, const double* B) {
  return {reinterpret_cast<const Vec3*>(E), reinterpret_cast<const Vec3*>(B)};
}

}  // namespace

extern "C" {

int ref_abi_version() { return 1; }

int ref_move_batch(double* x, double* y, double* z, double* u, double* v, double* w,
                   std::uint64_t n, const double* E, const double* B, int nx, int ny, int nz,
                   double lx, double ly, double lz, double dt, double qom, int pc, char* err,
                   int errlen) {
  SHIM_TRY
  const Grid g = Grid::make(nx, ny, nz, lx, ly, lz);
  const MoverParams mp = MoverParams::make(dt, qom, pc);
  move_batch(ParticleSpan{x, y, z, u, v, w, std::size_t(n)}, view_of(E, B), g, mp);
  SHIM_CATCH
}

// T threads, each running the reference mover on one contiguous slice.
int ref_move_batch_mt(double* x, double* y, double* z, double* u, double* v, double* w,
                      std::uint64_t n, const double* E, const double* B, int nx, int ny, int nz,
                      double lx, double ly, double lz, double dt, double qom, int pc,
                      int threads, char* err, int errlen) {
  SHIM_TRY
  const Grid g = Grid::make(nx, ny, nz, lx, ly, lz);
  const MoverParams mp = MoverParams::make(dt, qom, pc);
  if (threads < 1) threads = 1;
  const FieldView f = view_of(E, B);
  std::vector<std::exception_ptr> errs(static_cast<std::size_t>(threads));
  std::vector<std::thread> pool;
  const std::uint64_t chunk = (n + std::uint64_t(threads) - 1) / std::uint64_t(threads);
  for (int t = 0; t < threads; ++t) {
    const std::uint64_t lo = std::min<std::uint64_t>(n, chunk * std::uint64_t(t));
    const std::uint64_t hi = std::min<std::uint64_t>(n, lo + chunk);
    pool.emplace_back([&, t, lo, hi] {
      try {
        move_batch(ParticleSpan{x + lo, y + lo, z + lo, u + lo, v + lo, w + lo,
                                std::size_t(hi - lo)},
                   f, g, mp);
      } catch (...) {
        errs[std::size_t(t)] = std::current_exception();
      }
    });
  }
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
  SHIM_CATCH
}

// pic::deposit_moments (kernels.cpp:147-183) on a ParticleBatch built from the
// six arrays; out[0..3] rho,jx,jy,jz (+ out[4..9] pressure) are ACCUMULATED.
int ref_deposit_moments(const double* x, const double* y, const double* z, const double* u,
                        const double* v, const double* w, std::uint64_t n, int nx, int ny,
                        int nz, double lx, double ly, double lz, double qp, int with_pressure,
                        double* const* out, char* err, int errlen) {
  SHIM_TRY
  const Grid g = Grid::make(nx, ny, nz, lx, ly, lz);
  ParticleBatch b(0, 1.0, qp, std::size_t(n));
  for (std::uint64_t i = 0; i < n; ++i) b.append(x[i], y[i], z[i], u[i], v[i], w[i]);
  MomentMesh m = MomentMesh::make(g, with_pressure != 0);
  deposit_moments(b, g, m);
  const std::vector<double>* arr[10] = {&m.rho, &m.jx, &m.jy, &m.jz, &m.pxx,
                                        &m.pxy, &m.pxz, &m.pyy, &m.pyz, &m.pzz};
  for (int a = 0; a < (with_pressure ? 10 : 4); ++a)
    for (std::size_t i = 0; i < arr[a]->size(); ++i) out[a][i] += (*arr[a])[i];
  SHIM_CATCH
}

// pic::field_phase_stub (kernels.cpp:185-215) on a FieldMesh built from node
// AoS E/B (in place).
int ref_field_phase_stub(int nx, int ny, int nz, double lx, double ly, double lz, double* E,
                         double* B, int passes, char* err, int errlen) {
  SHIM_TRY
  const Grid g = Grid::make(nx, ny, nz, lx, ly, lz);
  FieldMesh m = FieldMesh::make(g);
  const std::size_t nodes = m.E.size();
  std::memcpy(m.E.data(), E, nodes * sizeof(Vec3));
  std::memcpy(m.B.data(), B, nodes * sizeof(Vec3));
  const FieldMesh out = field_phase_stub(m, g, passes);
  std::memcpy(E, out.E.data(), nodes * sizeof(Vec3));
  std::memcpy(B, out.B.data(), nodes * sizeof(Vec3));
  SHIM_CATCH
}

int ref_wrap_len(double v, double l, double* out) {
  *out = wrap_len(v, l);
  return kOk;
}

int ref_grid_cell_of(double px, double py, double pz, int nx, int ny, int nz, double lx,
                     double ly, double lz, int* ijk, double* f, char* err, int errlen) {
  SHIM_TRY
  const Grid g = Grid::make(nx, ny, nz, lx, ly, lz);
  const CellRef c = grid_cell_of(Vec3{px, py, pz}, g);
  ijk[0] = c.i; ijk[1] = c.j; ijk[2] = c.k;
  f[0] = c.fx; f[1] = c.fy; f[2] = c.fz;
  SHIM_CATCH
}

int ref_trilinear_weights(double px, double py, double pz, int nx, int ny, int nz, double lx,
                          double ly, double lz, std::int64_t* idx, double* wts, char* err,
                          int errlen) {
  SHIM_TRY
  const Grid g = Grid::make(nx, ny, nz, lx, ly, lz);
  const NodeWeights nw = trilinear_weights(Vec3{px, py, pz}, g);
  for (int c = 0; c < 8; ++c) {
    idx[c] = nw.idx[c];
    wts[c] = nw.w[c];
  }
  SHIM_CATCH
}

int ref_implicit_velocity(const double* vn, const double* Ep, const double* Bp, double dt,
                          double qom, double* out) {
  const MoverParams mp = MoverParams::make(dt, qom, 1);
  const Vec3 r = implicit_velocity(Vec3{vn[0], vn[1], vn[2]}, Vec3{Ep[0], Ep[1], Ep[2]},
                                   Vec3{Bp[0], Bp[1], Bp[2]}, mp);
  out[0] = r.x; out[1] = r.y; out[2] = r.z;
  return kOk;
}

// SimConfig for the GEM setup on an arbitrary grid (defaults elsewhere).
static SimConfig gem_cfg(int nx, int ny, int nz, double lx, double ly, double lz, int ppc,
                         std::uint64_t seed, int workers) {
  SimConfig cfg;
  cfg.grid = Grid::make(nx, ny, nz, lx, ly, lz);
  cfg.ppc = ppc;
  cfg.seed = seed;
  cfg.workers = workers;
  cfg.transfer.throttle = false;
  cfg.finalize();
  return cfg;
}

// Species table of the GEM setup: qom[4], q_per_particle[4], and the
// particle counts init_gem will produce.
int ref_gem_species(int nx, int ny, int nz, double lx, double ly, double lz, int ppc,
                    double* qom, double* qpp, std::uint64_t* counts, char* err, int errlen) {
  SHIM_TRY
  SimConfig cfg = gem_cfg(nx, ny, nz, lx, ly, lz, ppc, kDefaultSeed, 1);
  const InitialState st = init_gem(cfg);
  for (int s = 0; s < 4; ++s) {
    qom[s] = cfg.species[std::size_t(s)].qom;
    qpp[s] = cfg.species[std::size_t(s)].q_per_particle;
    counts[s] = st.batches[std::size_t(s)].count();
  }
  SHIM_CATCH
}

// Full GEM initial state. bufs[6*s + a] receives array a (x,y,z,u,v,w) of
// species s and must hold counts[s] doubles; E/B receive the node field.
int ref_init_gem(int nx, int ny, int nz, double lx, double ly, double lz, int ppc,
                 std::uint64_t seed, double* const* bufs, double* E, double* B, char* err,
                 int errlen) {
  SHIM_TRY
  SimConfig cfg = gem_cfg(nx, ny, nz, lx, ly, lz, ppc, seed, 1);
  const InitialState st = init_gem(cfg);
  for (int s = 0; s < 4; ++s) {
    const ParticleBatch& b = st.batches[std::size_t(s)];
    const std::size_t bytes = b.count() * sizeof(double);
    std::memcpy(bufs[6 * s + 0], b.xs(), bytes);
    std::memcpy(bufs[6 * s + 1], b.ys(), bytes);
    std::memcpy(bufs[6 * s + 2], b.zs(), bytes);
    std::memcpy(bufs[6 * s + 3], b.us(), bytes);
    std::memcpy(bufs[6 * s + 4], b.vs(), bytes);
    std::memcpy(bufs[6 * s + 5], b.ws(), bytes);
  }
  std::memcpy(E, st.field.E.data(), st.field.E.size() * sizeof(Vec3));
  std::memcpy(B, st.field.B.data(), st.field.B.size() * sizeof(Vec3));
  SHIM_CATCH
}

// ---- reference Simulation (runtime.cpp) driven from Python ----------------

struct RefSim {
  std::unique_ptr<Simulation> sim;
};

// Build a Simulation on the GEM setup (init_gem) or, when inject != 0, on an
// injected state: the caller passes 4 species (bufs/counts like ref_init_gem)
// plus E/B. engine: 0 cpu, 1 naive, 2 pinned, 3 prefetch.
int ref_sim_create(int nx, int ny, int nz, double lx, double ly, double lz, int ppc,
                   std::uint64_t seed, int workers, int engine, int pc, double dt,
                   int field_passes, int inject, double* const* bufs,
                   const std::uint64_t* counts, const double* E, const double* B,
                   void** out, char* err, int errlen) {
  SHIM_TRY
  SimConfig cfg;
  cfg.grid = Grid::make(nx, ny, nz, lx, ly, lz);
  cfg.ppc = ppc;
  cfg.seed = seed;
  cfg.workers = workers;
  cfg.engine = static_cast<EngineKind>(engine);
  cfg.pc_iterations = pc;
  cfg.dt = dt;
  cfg.field_passes = field_passes;
  cfg.transfer.throttle = false;
  cfg.finalize();
  auto h = std::make_unique<RefSim>();
  if (inject) {
    InitialState st;
    st.field = FieldMesh::make(cfg.grid);
    std::memcpy(st.field.E.data(), E, st.field.E.size() * sizeof(Vec3));
    std::memcpy(st.field.B.data(), B, st.field.B.size() * sizeof(Vec3));
    for (int s = 0; s < int(cfg.species.size()); ++s) {
      const Species& sp = cfg.species[std::size_t(s)];
      ParticleBatch b(sp.id, sp.qom, sp.q_per_particle, std::max<std::uint64_t>(counts[s], 1));
      for (std::uint64_t i = 0; i < counts[s]; ++i)
        b.append(bufs[6 * s][i], bufs[6 * s + 1][i], bufs[6 * s + 2][i], bufs[6 * s + 3][i],
                 bufs[6 * s + 4][i], bufs[6 * s + 5][i]);
      st.batches.push_back(std::move(b));
    }
    h->sim = std::make_unique<Simulation>(cfg, std::move(st));
  } else {
    h->sim = std::make_unique<Simulation>(cfg);
  }
  *out = h.release();
  SHIM_CATCH
}

int ref_sim_run(void* handle, int cycles, char* err, int errlen) {
  SHIM_TRY
  static_cast<RefSim*>(handle)->sim->run(cycles);
  SHIM_CATCH
}

int ref_sim_species_count(void* handle, int s, std::uint64_t* n) {
  *n = static_cast<RefSim*>(handle)->sim->gather_species(s).count();
  return kOk;
}

int ref_sim_gather(void* handle, int s, double* const* out6, char* err, int errlen) {
  SHIM_TRY
  const ParticleBatch b = static_cast<RefSim*>(handle)->sim->gather_species(s);
  const std::size_t bytes = b.count() * sizeof(double);
  std::memcpy(out6[0], b.xs(), bytes);
  std::memcpy(out6[1], b.ys(), bytes);
  std::memcpy(out6[2], b.zs(), bytes);
  std::memcpy(out6[3], b.us(), bytes);
  std::memcpy(out6[4], b.vs(), bytes);
  std::memcpy(out6[5], b.ws(), bytes);
  SHIM_CATCH
}

// Mean over cycles of t_mover (max over workers per cycle): the quantity
// bench.cpp:78-81 turns into one MPA/s figure per repetition.
int ref_sim_mean_mover_s(void* handle, double* out) {
  const auto& t = static_cast<RefSim*>(handle)->sim->timings();
  double s = 0.0;
  for (const CycleTimings& c : t) s += c.t_mover;
  *out = t.empty() ? 0.0 : s / double(t.size());
  return kOk;
}

void ref_sim_destroy(void* handle) { delete static_cast<RefSim*>(handle); }

int ref_mpa(std::uint64_t total, double t, double* out, char* err, int errlen) {
  SHIM_TRY
  *out = mpa(total, t);
  SHIM_CATCH
}

int ref_aggregate_runs(const double* v, int n, int warmup, double* harmonic, double* stddev,
                       char* err, int errlen) {
  SHIM_TRY
  const auto r = aggregate_runs(std::vector<double>(v, v + n), warmup);
  *harmonic = r.first;
  *stddev = r.second;
  SHIM_CATCH
}

int ref_decompose(int nx, int ny, int nz, int workers, int* out5, char* err, int errlen) {
  SHIM_TRY
  const Grid g = Grid::make(nx, ny, nz, 1.0, 1.0, 1.0);
  const auto subs = decompose(g, workers);
  for (std::size_t w = 0; w < subs.size(); ++w) {
    out5[5 * w + 0] = subs[w].worker_id;
    out5[5 * w + 1] = subs[w].j_lo;
    out5[5 * w + 2] = subs[w].j_hi;
    out5[5 * w + 3] = subs[w].prev;
    out5[5 * w + 4] = subs[w].next;
  }
  SHIM_CATCH
}

int ref_owner_of(double y, int nx, int ny, int nz, double lx, double ly, double lz, int workers) {
  const Grid g = Grid::make(nx, ny, nz, lx, ly, lz);
  return owner_of(y, g, workers);
}

}  // extern "C"
