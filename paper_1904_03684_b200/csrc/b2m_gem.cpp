// b2m_gem.cpp — synthetic GEM input for the mover, bit-identical to the
// reference's pic::init_gem (init.cpp:62-102) with the default GemParams
// (sim_config.hpp:30-39) and species table (config_file.cpp:55-75).
//
// The reference draws every species from one sequential splitmix64 stream
// (rng.hpp:12-56).  Because the generator is counter-based, the background
// species (exactly ppc particles per cell, init.cpp:21-32) can be generated
// in parallel: particle m of a species starts at uniform number
//     off(m) = 3m + 2*ceil(3m/2)
// (3 position draws, then the Box-Muller normals with their cached spare:
// normal call c draws a fresh pair iff c is even), and an odd particle's first
// normal is the sine half of the pair its predecessor drew last.  Sheet
// species (rejection sampling, init.cpp:38-52) stay sequential per species.
//
// Compiled by the host compiler without FMA contraction so every value
// matches the reference build bit for bit (verified in tests/test_gem.py).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "b2m.h"

namespace b2m {
b2m_status fail(b2m_status s, const std::string& msg);  // b2m_capi.cu
}

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

// GemParams defaults (sim_config.hpp:30-39)
constexpr double kB0 = 1.0, kLambda = 0.5, kNbOverN0 = 0.2, kPsi0 = 0.1, kTiOverTe = 5.0,
                 kMassRatio = 25.0, kUthE = 0.045, kUthI = 0.0126;

b2m_status gem_fail(b2m_status s, const char* msg) { return b2m::fail(s, msg); }

uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Stream {
  uint64_t s0;  // state before the first draw
  Stream(uint64_t seed, uint64_t stream) : s0(mix(seed) ^ mix(kGolden + stream)) {}
  // k-th uniform of the stream (0-based)
  double uniform_at(uint64_t k) const {
    return static_cast<double>(mix(s0 + (k + 1) * kGolden) >> 11) * 0x1.0p-53;
  }
};

// Sequential view (sheet species).
struct SeqRng {
  uint64_t state;
  double spare = 0.0;
  bool have_spare = false;
  SeqRng(uint64_t seed, uint64_t stream) : state(mix(seed) ^ mix(kGolden + stream)) {}
  double uniform() {
    state += kGolden;
    return static_cast<double>(mix(state) >> 11) * 0x1.0p-53;
  }
  double normal() {
    if (have_spare) {
      have_spare = false;
      return spare;
    }
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = kTwoPi * u2;
    spare = r * std::sin(a);
    have_spare = true;
    return r * std::cos(a);
  }
};

void box_muller(double u1_raw, double u2, double* c, double* s) {
  const double u1 = 1.0 - u1_raw;
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double a = kTwoPi * u2;
  *s = r * std::sin(a);
  *c = r * std::cos(a);
}

double wrap_len(double v, double l) {  // grid.hpp:45-50
  double w = v - l * std::floor(v / l);
  if (w >= l) w -= l;
  if (w < 0.0) w = 0.0;
  return w;
}

struct SpeciesDef {
  double qom, qpp;
  double uth[3];
  double u0[3];
  bool sheet;
};

SpeciesDef species_def(const b2m_grid& g, int ppc, int s) {
  // config_file.cpp:55-75
  const double v_cell = g.dx * g.dy * g.dz;
  const double drift = kB0 / kLambda;
  const double u_iz = -drift * kTiOverTe / (1.0 + kTiOverTe);
  const double u_ez = +drift * 1.0 / (1.0 + kTiOverTe);
  const double q_bg = kNbOverN0 * v_cell / double(ppc);
  const double q_sheet = v_cell / double(ppc);
  SpeciesDef d{};
  const bool electron = (s == 0 || s == 2);
  d.qom = electron ? -kMassRatio : +1.0;
  const double uth = electron ? kUthE : kUthI;
  d.uth[0] = d.uth[1] = d.uth[2] = uth;
  d.sheet = s >= 2;
  if (s == 0) d.qpp = -q_bg;
  if (s == 1) d.qpp = +q_bg;
  if (s == 2) { d.qpp = -q_sheet; d.u0[2] = u_ez; }
  if (s == 3) { d.qpp = +q_sheet; d.u0[2] = u_iz; }
  return d;
}

uint64_t sheet_count(const b2m_grid& g, int ppc) {  // init.cpp:54-58
  const double integral = 2.0 * kLambda * std::tanh(g.ly / (2.0 * kLambda));
  return static_cast<uint64_t>(
      std::llround(double(ppc) * double(int64_t(g.nx) * g.ny * g.nz) * integral / g.ly));
}

// Background species, particles [m0, m1) in (k,j,i,p) order, written at
// out[a][m - base].
void fill_background(const b2m_grid& g, int ppc, const SpeciesDef& d, const Stream& rs,
                     uint64_t m0, uint64_t m1, double* const* out, uint64_t base = 0) {
  for (uint64_t m = m0; m < m1; ++m) {
    uint64_t cell = m / uint64_t(ppc);
    const int i = int(cell % uint64_t(g.nx));
    cell /= uint64_t(g.nx);
    const int j = int(cell % uint64_t(g.ny));
    const int k = int(cell / uint64_t(g.ny));
    const uint64_t off = 3 * m + 2 * ((3 * m + 1) / 2);
    const double x = wrap_len((i + rs.uniform_at(off + 0)) * g.dx, g.lx);
    const double y = wrap_len((j + rs.uniform_at(off + 1)) * g.dy, g.ly);
    const double z = wrap_len((k + rs.uniform_at(off + 2)) * g.dz, g.lz);
    double nrm[3];
    uint64_t cur = off + 3;
    double spare = 0.0;
    bool have = false;
    if (m & 1) {
      // spare of the predecessor's last pair (drawn at its uniforms off(m-1)+5, +6)
      const uint64_t pm = m - 1;
      const uint64_t poff = 3 * pm + 2 * ((3 * pm + 1) / 2);
      double c, s;
      box_muller(rs.uniform_at(poff + 5), rs.uniform_at(poff + 6), &c, &s);
      spare = s;
      have = true;
    }
    for (int t = 0; t < 3; ++t) {
      if (have) {
        nrm[t] = spare;
        have = false;
      } else {
        double c, s;
        box_muller(rs.uniform_at(cur), rs.uniform_at(cur + 1), &c, &s);
        cur += 2;
        nrm[t] = c;
        spare = s;
        have = true;
      }
    }
    const uint64_t o = m - base;
    out[0][o] = x;
    out[1][o] = y;
    out[2][o] = z;
    out[3][o] = d.u0[0] + d.uth[0] * nrm[0];
    out[4][o] = d.u0[1] + d.uth[1] * nrm[1];
    out[5][o] = d.u0[2] + d.uth[2] * nrm[2];
  }
}

void fill_sheet(const b2m_grid& g, const SpeciesDef& d, uint64_t seed, int s, uint64_t n,
                double* const* out) {
  SeqRng r(seed, uint64_t(s));
  const double ymid = 0.5 * g.ly;
  for (uint64_t m = 0; m < n; ++m) {
    double y;
    for (;;) {
      y = r.uniform() * g.ly;
      const double c = std::cosh((y - ymid) / kLambda);
      if (r.uniform() <= 1.0 / (c * c)) break;
    }
    const double x = r.uniform() * g.lx;
    const double z = r.uniform() * g.lz;
    const double a = r.normal();
    const double b = r.normal();
    const double c = r.normal();
    out[0][m] = x;
    out[1][m] = wrap_len(y, g.ly);
    out[2][m] = wrap_len(z, g.lz);
    out[3][m] = d.u0[0] + d.uth[0] * a;
    out[4][m] = d.u0[1] + d.uth[1] * b;
    out[5][m] = d.u0[2] + d.uth[2] * c;
  }
}

int64_t node_index(const b2m_grid& g, int i, int j, int k) {
  return i + int64_t(g.nx + 1) * (j + int64_t(g.ny + 1) * k);
}

// field_mesh.hpp:46-59
void mirror_seams(const b2m_grid& g, double* F) {
  for (int k = 0; k <= g.nz; ++k)
    for (int j = 0; j <= g.ny; ++j) {
      const int ks = k == g.nz ? 0 : k, js = j == g.ny ? 0 : j;
      for (int i = 0; i <= g.nx; ++i) {
        const int is = i == g.nx ? 0 : i;
        if (is == i && js == j && ks == k) continue;
        const int64_t d = node_index(g, i, j, k), s = node_index(g, is, js, ks);
        F[3 * d] = F[3 * s];
        F[3 * d + 1] = F[3 * s + 1];
        F[3 * d + 2] = F[3 * s + 2];
      }
    }
}

bool valid(const b2m_grid* g, int ppc) {
  return g && g->nx >= 2 && g->ny >= 2 && g->nz >= 2 && ppc >= 1 && kLambda < g->ly / 2.0;
}

}  // namespace

extern "C" {

b2m_status b2m_gem_counts(const b2m_grid* g, int ppc, uint64_t* counts4) {
  if (!valid(g, ppc) || !counts4) return gem_fail(B2M_CONFIG_ERROR, "gem: invalid grid or ppc");
  const uint64_t bg = uint64_t(ppc) * uint64_t(g->nx) * g->ny * g->nz;
  const uint64_t sh = sheet_count(*g, ppc);
  counts4[0] = bg; counts4[1] = bg; counts4[2] = sh; counts4[3] = sh;
  return B2M_OK;
}

b2m_status b2m_gem_species_params(const b2m_grid* g, int ppc, double* qom4, double* qpp4) {
  if (!valid(g, ppc)) return gem_fail(B2M_CONFIG_ERROR, "gem: invalid grid or ppc");
  for (int s = 0; s < 4; ++s) {
    const SpeciesDef d = species_def(*g, ppc, s);
    if (qom4) qom4[s] = d.qom;
    if (qpp4) qpp4[s] = d.qpp;
  }
  return B2M_OK;
}

b2m_status b2m_gem_fill_species(const b2m_grid* g, int ppc, uint64_t seed, int s,
                                double* const* host6, int threads) {
  if (!valid(g, ppc) || !host6 || s < 0 || s > 3)
    return gem_fail(B2M_CONFIG_ERROR, "gem: invalid arguments");
  const SpeciesDef d = species_def(*g, ppc, s);
  if (d.sheet) {
    fill_sheet(*g, d, seed, s, sheet_count(*g, ppc), host6);
    return B2M_OK;
  }
  const uint64_t n = uint64_t(ppc) * uint64_t(g->nx) * g->ny * g->nz;
  const Stream rs(seed, uint64_t(s));
  if (threads <= 0) threads = int(std::max(1u, std::thread::hardware_concurrency()));
  threads = int(std::min<uint64_t>(uint64_t(threads), std::max<uint64_t>(1, n / 4096)));
  std::vector<std::thread> pool;
  const uint64_t chunk = (n + uint64_t(threads) - 1) / uint64_t(threads);
  for (int t = 0; t < threads; ++t) {
    const uint64_t lo = std::min(n, chunk * uint64_t(t)), hi = std::min(n, lo + chunk);
    pool.emplace_back([&, lo, hi] { fill_background(*g, ppc, d, rs, lo, hi, host6); });
  }
  for (auto& th : pool) th.join();
  return B2M_OK;
}

b2m_status b2m_gem_fill_species_range(const b2m_grid* g, int ppc, uint64_t seed, int s,
                                      uint64_t m0, uint64_t m1, double* const* host6,
                                      int threads) {
  if (!valid(g, ppc) || !host6 || s < 0 || s > 1 || m1 < m0)
    return gem_fail(B2M_CONFIG_ERROR, "gem: range fill needs a background species and m0 <= m1");
  const uint64_t n = uint64_t(ppc) * uint64_t(g->nx) * g->ny * g->nz;
  if (m1 > n) return gem_fail(B2M_CONFIG_ERROR, "gem: range beyond the species");
  const SpeciesDef d = species_def(*g, ppc, s);
  const Stream rs(seed, uint64_t(s));
  const uint64_t len = m1 - m0;
  if (threads <= 0) threads = int(std::max(1u, std::thread::hardware_concurrency()));
  threads = int(std::min<uint64_t>(uint64_t(threads), std::max<uint64_t>(1, len / 4096)));
  std::vector<std::thread> pool;
  const uint64_t chunk = (len + uint64_t(threads) - 1) / uint64_t(threads);
  for (int t = 0; t < threads; ++t) {
    const uint64_t lo = m0 + std::min(len, chunk * uint64_t(t));
    const uint64_t hi = std::min(m1, lo + chunk);
    if (lo >= hi) continue;
    pool.emplace_back([&, lo, hi] { fill_background(*g, ppc, d, rs, lo, hi, host6, m0); });
  }
  for (auto& th : pool) th.join();
  return B2M_OK;
}

b2m_status b2m_gem_field(const b2m_grid* g, double* E, double* B) {
  if (!valid(g, 1) || !E || !B) return gem_fail(B2M_CONFIG_ERROR, "gem: invalid arguments");
  const int64_t nodes = int64_t(g->nx + 1) * (g->ny + 1) * (g->nz + 1);
  std::memset(E, 0, size_t(3 * nodes) * sizeof(double));
  std::memset(B, 0, size_t(3 * nodes) * sizeof(double));
  const double ymid = 0.5 * g->ly;
  // init.cpp:72-86
  for (int k = 0; k < g->nz; ++k)
    for (int j = 0; j < g->ny; ++j)
      for (int i = 0; i < g->nx; ++i) {
        const double x = i * g->dx;
        const double y = j * g->dy;
        const double bx = kB0 * std::tanh((y - ymid) / kLambda) -
                          kPsi0 * (kPi / g->ly) * std::cos(2.0 * kPi * x / g->lx) *
                              std::sin(kPi * (y - ymid) / g->ly);
        const double by = kPsi0 * (2.0 * kPi / g->lx) * std::sin(2.0 * kPi * x / g->lx) *
                          std::cos(kPi * (y - ymid) / g->ly);
        const int64_t q = node_index(*g, i, j, k);
        B[3 * q] = bx;
        B[3 * q + 1] = by;
        B[3 * q + 2] = 0.0;
      }
  mirror_seams(*g, B);
  return B2M_OK;
}

b2m_status b2m_gem_like_field(const b2m_grid* g, double* E, double* B) {
  if (!g || !E || !B) return gem_fail(B2M_CONFIG_ERROR, "gem: invalid arguments");
  const int64_t nodes = int64_t(g->nx + 1) * (g->ny + 1) * (g->nz + 1);
  std::memset(E, 0, size_t(3 * nodes) * sizeof(double));
  std::memset(B, 0, size_t(3 * nodes) * sizeof(double));
  for (int k = 0; k < g->nz; ++k)
    for (int j = 0; j < g->ny; ++j)
      for (int i = 0; i < g->nx; ++i) {
        const double x = i * g->dx, y = j * g->dy;
        const int64_t q = node_index(*g, i, j, k);
        E[3 * q] = 0.01 * std::sin(y);
        E[3 * q + 1] = 0.0;
        E[3 * q + 2] = 0.02;
        B[3 * q] = std::tanh((y - g->ly / 2) / 0.5);
        B[3 * q + 1] = 0.05 * std::sin(x);
        B[3 * q + 2] = 0.0;
      }
  mirror_seams(*g, E);
  mirror_seams(*g, B);
  return B2M_OK;
}

}  // extern "C"
