/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Plain-C restatement of the reference particle mover ("minipic",
 * /root/reference/proj) used ONLY as the parity checker by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg.  The product path
 * (paper_1904_03684_b200/) never links or calls it.
 *
 * Parity is PINNED: tests/test_oracle.py checks this file bit-for-bit against
 * the unmodified reference library (oracle/_ref/libminipic_ref.so, built by
 * oracle/Makefile from the reference sources) and against the committed golden
 * vectors in tests/golden/ that the reference produced.
 *
 * Arithmetic is IEEE binary64 with no contraction (built with
 * -ffp-contract=off, no -march), matching the reference's FMA-free build
 * (SURVEY §0).  Every operation keeps the reference's evaluation order.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

typedef struct {
  int nx, ny, nz;
  double lx, ly, lz;
  double dx, dy, dz;
} or_grid;

/* grid.hpp:20-28 Grid::make -- cell sizes are l/n (IEEE division). */
void or_grid_make(or_grid* g, int nx, int ny, int nz, double lx, double ly, double lz) {
  g->nx = nx; g->ny = ny; g->nz = nz;
  g->lx = lx; g->ly = ly; g->lz = lz;
  g->dx = lx / nx; g->dy = ly / ny; g->dz = lz / nz;
}

/* grid.hpp:36-38 node-major index i + (nx+1)*(j + (ny+1)*k). */
static int64_t node_of(const or_grid* g, int i, int j, int k) {
  return (int64_t)i + (int64_t)(g->nx + 1) * ((int64_t)j + (int64_t)(g->ny + 1) * k);
}

/* grid.hpp:45-50 wrap_len: v - l*floor(v/l), then the two rounding fixups. */
double or_wrap_len(double v, double l) {
  double q = floor(v / l);
  double w = v - l * q;
  if (w >= l) w = w - l;
  if (w < 0.0) w = 0.0;
  return w;
}

/* grid.hpp:64-82 grid_cell_of.  Returns 0 on success, -1 when the position is
 * outside [0,l) in some axis (the reference throws DomainError; NaN fails
 * every comparison and lands here too). */
int or_grid_cell_of(const or_grid* g, double px, double py, double pz, int* ijk, double* f) {
  double s[3];
  int c[3];
  if (!(px >= 0.0 && px < g->lx && py >= 0.0 && py < g->ly && pz >= 0.0 && pz < g->lz))
    return -1;
  s[0] = px / g->dx; s[1] = py / g->dy; s[2] = pz / g->dz;
  c[0] = (int)s[0]; c[1] = (int)s[1]; c[2] = (int)s[2];     /* truncation */
  if (c[0] >= g->nx) c[0] = g->nx - 1;
  if (c[1] >= g->ny) c[1] = g->ny - 1;
  if (c[2] >= g->nz) c[2] = g->nz - 1;
  for (int a = 0; a < 3; ++a) {
    double fa = s[a] - (double)c[a];
    if (fa > 1.0) fa = 1.0;
    f[a] = fa;
    ijk[a] = c[a];
  }
  return 0;
}

/* kernels.cpp:10-22 trilinear_weights: corner c = di + 2dj + 4dk,
 * w = (wx[di]*wy[dj])*wz[dk]. */
int or_trilinear_weights(const or_grid* g, double px, double py, double pz, int64_t* idx,
                         double* wts) {
  int ijk[3];
  double f[3];
  if (or_grid_cell_of(g, px, py, pz, ijk, f) != 0) return -1;
  const double wx[2] = {1.0 - f[0], f[0]};
  const double wy[2] = {1.0 - f[1], f[1]};
  const double wz[2] = {1.0 - f[2], f[2]};
  for (int corner = 0; corner < 8; ++corner) {
    const int di = corner & 1, dj = (corner >> 1) & 1, dk = (corner >> 2) & 1;
    idx[corner] = node_of(g, ijk[0] + di, ijk[1] + dj, ijk[2] + dk);
    double wxy = wx[di] * wy[dj];
    wts[corner] = wxy * wz[dk];
  }
  return 0;
}

/* kernels.cpp:40-50 implicit_velocity (closed Cayley form, fixed op order). */
void or_implicit_velocity(const double* vn, const double* Ep, const double* Bp, double beta,
                          double* out) {
  const double vt0 = vn[0] + beta * Ep[0];
  const double vt1 = vn[1] + beta * Ep[1];
  const double vt2 = vn[2] + beta * Ep[2];
  const double o0 = beta * Bp[0], o1 = beta * Bp[1], o2 = beta * Bp[2];
  const double omsq = (o0 * o0 + o1 * o1) + o2 * o2;
  const double denom = 1.0 / (1.0 + omsq);
  const double vdot = (vt0 * o0 + vt1 * o1) + vt2 * o2;
  out[0] = ((vt0 + (vt1 * o2 - vt2 * o1)) + vdot * o0) * denom;
  out[1] = ((vt1 + (vt2 * o0 - vt0 * o2)) + vdot * o1) * denom;
  out[2] = ((vt2 + (vt0 * o1 - vt1 * o0)) + vdot * o2) * denom;
}

/* kernels.cpp:52-104 move_batch.  E and B are node arrays of 3 doubles per
 * node (FieldView layout, field_mesh.hpp:13-16).  beta = qom*dt*0.5 as
 * MoverParams::make computes it (kernels.hpp:36-38).  Returns -1 on success or
 * the index of the first particle whose state went non-finite; as in the
 * reference, particles before that index are updated and it and every later
 * particle are left untouched. */
int64_t or_move_batch(double* x, double* y, double* z, double* u, double* v, double* w,
                      uint64_t n, const double* E, const double* B, const or_grid* g, double dt,
                      double qom, int pc_iterations) {
  const double beta = qom * dt * 0.5;
  const double dto2 = 0.5 * dt;
  for (uint64_t i = 0; i < n; ++i) {
    const double x0[3] = {x[i], y[i], z[i]};
    const double v0[3] = {u[i], v[i], w[i]};
    double xt[3] = {x0[0], x0[1], x0[2]};
    double vb[3] = {v0[0], v0[1], v0[2]};
    for (int r = 0; r < pc_iterations; ++r) {
      int64_t idx[8];
      double wt[8];
      if (or_trilinear_weights(g, xt[0], xt[1], xt[2], idx, wt) != 0) return (int64_t)i;
      /* gather: accumulators start at +0.0 and add corners in order
       * (kernels.cpp:74-81) */
      double Ef[3] = {0.0, 0.0, 0.0}, Bf[3] = {0.0, 0.0, 0.0};
      for (int c = 0; c < 8; ++c) {
        const double* e = E + 3 * idx[c];
        const double* b = B + 3 * idx[c];
        for (int a = 0; a < 3; ++a) {
          Ef[a] += wt[c] * e[a];
          Bf[a] += wt[c] * b[a];
        }
      }
      or_implicit_velocity(v0, Ef, Bf, beta, vb);
      /* predictor (kernels.cpp:92) */
      xt[0] = or_wrap_len(x0[0] + vb[0] * dto2, g->lx);
      xt[1] = or_wrap_len(x0[1] + vb[1] * dto2, g->ly);
      xt[2] = or_wrap_len(x0[2] + vb[2] * dto2, g->lz);
    }
    /* final update (kernels.cpp:95-96) */
    const double x1[3] = {or_wrap_len(x0[0] + vb[0] * dt, g->lx),
                          or_wrap_len(x0[1] + vb[1] * dt, g->ly),
                          or_wrap_len(x0[2] + vb[2] * dt, g->lz)};
    const double v1[3] = {2.0 * vb[0] - v0[0], 2.0 * vb[1] - v0[1], 2.0 * vb[2] - v0[2]};
    for (int a = 0; a < 3; ++a)
      if (!isfinite(x1[a]) || !isfinite(v1[a])) return (int64_t)i; /* kernels.cpp:98-99 */
    x[i] = x1[0]; y[i] = x1[1]; z[i] = x1[2];
    u[i] = v1[0]; v[i] = v1[1]; w[i] = v1[2];
  }
  return -1;
}

/* Convenience wrapper with the grid given by value (ctypes-friendly). */
int64_t or_move_batch_g(double* x, double* y, double* z, double* u, double* v, double* w,
                        uint64_t n, const double* E, const double* B, int nx, int ny, int nz,
                        double lx, double ly, double lz, double dt, double qom, int pc) {
  or_grid g;
  or_grid_make(&g, nx, ny, nz, lx, ly, lz);
  return or_move_batch(x, y, z, u, v, w, n, E, B, &g, dt, qom, pc);
}

/* ---- GEM input generation (init.cpp, rng.hpp) ---------------------------- */

/* kernels.cpp:185-215 field_phase_stub: `passes` rounds of
 * e + (1/12) * sum_nb (E_nb - e) over the 6 periodic face neighbours of
 * every unique node (the six differences added left to right), ping-ponging
 * between two meshes; then mirror_seams (field_mesh.hpp:46-59) copies the
 * 0-planes of E and B onto the n-planes.  passes <= 0 returns the input
 * unchanged (no mirroring).  E, B: node AoS with seams, updated in place. */
void or_field_phase_stub_g(int nx, int ny, int nz, double* E, double* B, int passes,
                           double* scratch) {
  if (passes <= 0) return;
  const int64_t sx = nx + 1, sy = ny + 1;
  const int64_t nodes = sx * sy * (int64_t)(nz + 1);
  double* cur = E;
  double* nxt = scratch;
  for (int64_t q = 0; q < 3 * nodes; ++q) nxt[q] = E[q];
  for (int pass = 0; pass < passes; ++pass) {
    for (int k = 0; k < nz; ++k) {
      const int km = (k + nz - 1) % nz, kp = (k + 1) % nz;
      for (int j = 0; j < ny; ++j) {
        const int jm = (j + ny - 1) % ny, jp = (j + 1) % ny;
        for (int i = 0; i < nx; ++i) {
          const int im = (i + nx - 1) % nx, ip = (i + 1) % nx;
          const int64_t c = i + sx * (j + sy * k);
          const int64_t nb[6] = {im + sx * (j + sy * k), ip + sx * (j + sy * k),
                                 i + sx * (jm + sy * k), i + sx * (jp + sy * k),
                                 i + sx * (j + sy * km), i + sx * (j + sy * kp)};
          for (int a = 0; a < 3; ++a) {
            const double e = cur[3 * c + a];
            double sum = cur[3 * nb[0] + a] - e;
            for (int m = 1; m < 6; ++m) sum = sum + (cur[3 * nb[m] + a] - e);
            nxt[3 * c + a] = e + (1.0 / 12.0) * sum;
          }
        }
      }
    }
    double* t = cur; cur = nxt; nxt = t;
  }
  if (cur != E)
    for (int64_t q = 0; q < 3 * nodes; ++q) E[q] = cur[q];
  /* mirror_seams */
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j) {
      const int ks = k == nz ? 0 : k, js = j == ny ? 0 : j;
      for (int i = 0; i <= nx; ++i) {
        const int is = i == nx ? 0 : i;
        if (is == i && js == j && ks == k) continue;
        const int64_t d = i + sx * (j + sy * k), src = is + sx * (js + sy * ks);
        for (int a = 0; a < 3; ++a) {
          E[3 * d + a] = E[3 * src + a];
          B[3 * d + a] = B[3 * src + a];
        }
      }
    }
}

/* kernels.cpp:147-183 deposit_moments: every particle scatters
 * wq = ((q/V * wx) * wy) * wz onto the 8 corners of its cell, corner order
 * c = di + 2dj + 4dk, the upper corners wrapping onto node 0 (periodic, nodes
 * == cells, index i + nx*(j + ny*k), kernels.hpp:63-65); rho += wq,
 * j += wq*u, and (with_pressure) p_ab += (wq*u_a)*u_b, in particle order.
 * out[0..3] = rho, jx, jy, jz; out[4..9] = pxx, pxy, pxz, pyy, pyz, pzz.
 * Returns -1, or the index of the first particle outside the domain (the
 * reference's grid_cell_of throws DomainError there). */
int64_t or_deposit_moments_g(const double* x, const double* y, const double* z, const double* u,
                             const double* v, const double* w, uint64_t n, int nx, int ny,
                             int nz, double lx, double ly, double lz, double qp,
                             int with_pressure, double* const* out) {
  or_grid g;
  or_grid_make(&g, nx, ny, nz, lx, ly, lz);
  const double inv_vol = 1.0 / (g.dx * g.dy * g.dz);
  for (uint64_t p = 0; p < n; ++p) {
    int c[3];
    double f[3];
    if (or_grid_cell_of(&g, x[p], y[p], z[p], c, f) != 0) return (int64_t)p;
    const double wx[2] = {1.0 - f[0], f[0]};
    const double wy[2] = {1.0 - f[1], f[1]};
    const double wz[2] = {1.0 - f[2], f[2]};
    const int ii[2] = {c[0], c[0] + 1 == nx ? 0 : c[0] + 1};
    const int jj[2] = {c[1], c[1] + 1 == ny ? 0 : c[1] + 1};
    const int kk[2] = {c[2], c[2] + 1 == nz ? 0 : c[2] + 1};
    const double ux = u[p], uy = v[p], uz = w[p];
    const double qv = qp * inv_vol;
    for (int corner = 0; corner < 8; ++corner) {
      const int di = corner & 1, dj = (corner >> 1) & 1, dk = (corner >> 2) & 1;
      const double wq = qv * wx[di] * wy[dj] * wz[dk];
      const int64_t idx = (int64_t)ii[di] + (int64_t)nx * ((int64_t)jj[dj] + (int64_t)ny * kk[dk]);
      out[0][idx] += wq;
      out[1][idx] += wq * ux;
      out[2][idx] += wq * uy;
      out[3][idx] += wq * uz;
      if (with_pressure) {
        out[4][idx] += wq * ux * ux;
        out[5][idx] += wq * ux * uy;
        out[6][idx] += wq * ux * uz;
        out[7][idx] += wq * uy * uy;
        out[8][idx] += wq * uy * uz;
        out[9][idx] += wq * uz * uz;
      }
    }
  }
  return -1;
}

/* rng.hpp:12-56 CounterRng: splitmix64 stream keyed by (seed, stream). */
typedef struct {
  uint64_t state;
  double spare;
  int have_spare;
} or_rng;

static uint64_t or_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void or_rng_init(or_rng* r, uint64_t seed, uint64_t stream) {
  r->state = or_mix(seed) ^ or_mix(0x9E3779B97F4A7C15ull + stream);
  r->spare = 0.0;
  r->have_spare = 0;
}

double or_rng_uniform(or_rng* r) {
  r->state += 0x9E3779B97F4A7C15ull;
  return (double)(or_mix(r->state) >> 11) * 0x1.0p-53;
}

double or_rng_normal(or_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  const double u1 = 1.0 - or_rng_uniform(r);
  const double u2 = or_rng_uniform(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double ang = 6.283185307179586476925286766559 * u2;
  r->spare = rad * sin(ang);
  r->have_spare = 1;
  return rad * cos(ang);
}

/* init.cpp:54-58 sheet_count. */
uint64_t or_sheet_count(const or_grid* g, double lambda, int ppc) {
  const double integral = 2.0 * lambda * tanh(g->ly / (2.0 * lambda));
  const double cells = (double)((int64_t)g->nx * g->ny * g->nz);
  return (uint64_t)llround((double)ppc * cells * integral / g->ly);
}

/* One GEM species (init.cpp:21-52, species table config_file.cpp:55-75).
 * sheet=0: exactly ppc per cell in (k,j,i,p) order; sheet=1: sech^2 rejection
 * sampling in y.  uth and u0 are per-axis; writes n particles. */
void or_fill_species(const or_grid* g, int sheet, int ppc, uint64_t n, double lambda,
                     const double* uth, const double* u0, uint64_t seed, uint64_t stream,
                     double* x, double* y, double* z, double* u, double* v, double* w) {
  or_rng r;
  or_rng_init(&r, seed, stream);
  uint64_t m = 0;
  if (!sheet) {
    for (int k = 0; k < g->nz; ++k)
      for (int j = 0; j < g->ny; ++j)
        for (int i = 0; i < g->nx; ++i)
          for (int p = 0; p < ppc; ++p) {
            x[m] = or_wrap_len((i + or_rng_uniform(&r)) * g->dx, g->lx);
            y[m] = or_wrap_len((j + or_rng_uniform(&r)) * g->dy, g->ly);
            z[m] = or_wrap_len((k + or_rng_uniform(&r)) * g->dz, g->lz);
            const double a = or_rng_normal(&r), b = or_rng_normal(&r), c = or_rng_normal(&r);
            u[m] = u0[0] + uth[0] * a;
            v[m] = u0[1] + uth[1] * b;
            w[m] = u0[2] + uth[2] * c;
            ++m;
          }
    return;
  }
  const double ymid = 0.5 * g->ly;
  for (; m < n; ++m) {
    double yy;
    for (;;) {
      yy = or_rng_uniform(&r) * g->ly;
      const double ch = cosh((yy - ymid) / lambda);
      if (or_rng_uniform(&r) <= 1.0 / (ch * ch)) break;
    }
    const double xx = or_rng_uniform(&r) * g->lx;
    const double zz = or_rng_uniform(&r) * g->lz;
    const double a = or_rng_normal(&r), b = or_rng_normal(&r), c = or_rng_normal(&r);
    x[m] = xx;
    y[m] = or_wrap_len(yy, g->ly);
    z[m] = or_wrap_len(zz, g->lz);
    u[m] = u0[0] + uth[0] * a;
    v[m] = u0[1] + uth[1] * b;
    w[m] = u0[2] + uth[2] * c;
  }
}

/* test_offload.cpp:60-71 gem_like_field fixture: E=(0.01 sin y, 0, 0.02),
 * B=(tanh((y-ly/2)/0.5), 0.05 sin x, 0) on unique nodes, seams mirrored
 * (field_mesh.hpp:46-59). */
void or_gem_like_field(const or_grid* g, double* E, double* B) {
  const int nx1 = g->nx + 1, ny1 = g->ny + 1, nz1 = g->nz + 1;
  for (int64_t q = 0; q < (int64_t)nx1 * ny1 * nz1; ++q) {
    E[3 * q] = E[3 * q + 1] = E[3 * q + 2] = 0.0;
    B[3 * q] = B[3 * q + 1] = B[3 * q + 2] = 0.0;
  }
  for (int k = 0; k <= g->nz; ++k)
    for (int j = 0; j <= g->ny; ++j)
      for (int i = 0; i <= g->nx; ++i) {
        const int is = i == g->nx ? 0 : i, js = j == g->ny ? 0 : j, ks = k == g->nz ? 0 : k;
        const double xx = is * g->dx, yy = js * g->dy;
        const int64_t q = node_of(g, i, j, k);
        (void)ks;
        E[3 * q + 0] = 0.01 * sin(yy);
        E[3 * q + 1] = 0.0;
        E[3 * q + 2] = 0.02;
        B[3 * q + 0] = tanh((yy - g->ly / 2) / 0.5);
        B[3 * q + 1] = 0.05 * sin(xx);
        B[3 * q + 2] = 0.0;
      }
}

void or_gem_like_field_g(int nx, int ny, int nz, double lx, double ly, double lz, double* E,
                         double* B) {
  or_grid g;
  or_grid_make(&g, nx, ny, nz, lx, ly, lz);
  or_gem_like_field(&g, E, B);
}

void or_fill_species_g(int nx, int ny, int nz, double lx, double ly, double lz, int sheet,
                       int ppc, uint64_t n, double lambda, const double* uth, const double* u0,
                       uint64_t seed, uint64_t stream, double* x, double* y, double* z,
                       double* u, double* v, double* w) {
  or_grid g;
  or_grid_make(&g, nx, ny, nz, lx, ly, lz);
  or_fill_species(&g, sheet, ppc, n, lambda, uth, u0, seed, stream, x, y, z, u, v, w);
}

uint64_t or_sheet_count_g(int nx, int ny, int nz, double lx, double ly, double lz,
                          double lambda, int ppc) {
  or_grid g;
  or_grid_make(&g, nx, ny, nz, lx, ly, lz);
  return or_sheet_count(&g, lambda, ppc);
}
