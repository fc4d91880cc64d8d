"""Synthetic GEM input (the reference's ``init_gem``, init.cpp:62-102).

Native, multithreaded and bit-identical to the reference generator
(``b2m_gem_*`` in csrc/b2m_gem.cpp).  The mover never sees E != 0 in a stock
GEM run, so benchmarks and parity fixtures add the nonzero E of
the reference's own ``gem_like_field`` fixture (test_offload.cpp:60-71).
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _capi
from .mover import FieldMesh, Grid, MoverParams, ParticleBatch

DEFAULT_SEED = 12345  # sim_config.hpp:32


def gem_counts(grid: Grid, ppc: int):
    c = (C.c_uint64 * 4)()
    _capi.check(_capi.lib().b2m_gem_counts(C.byref(grid.to_c()), ppc, c))
    return [int(v) for v in c]


def gem_species_params(grid: Grid, ppc: int):
    qom = np.zeros(4)
    qpp = np.zeros(4)
    _capi.check(_capi.lib().b2m_gem_species_params(C.byref(grid.to_c()), ppc, _capi.dptr(qom),
                                                   _capi.dptr(qpp)))
    return qom, qpp


def init_gem_species(grid: Grid, ppc: int, seed: int = DEFAULT_SEED, pinned: bool = False,
                     threads: int = 0, species=(0, 1, 2, 3)):
    """The four GEM ParticleBatches (bg e-, bg i+, sheet e-, sheet i+).  The
    two sequential sheet species are generated concurrently with the
    parallel background ones."""
    counts = gem_counts(grid, ppc)
    qom, qpp = gem_species_params(grid, ppc)
    batches = {s: ParticleBatch(s, float(qom[s]), float(qpp[s]), counts[s], pinned=pinned)
               for s in species}
    g = grid.to_c()
    errs = []

    def fill(s):
        b = batches[s]
        st = _capi.lib().b2m_gem_fill_species(C.byref(g), ppc, seed, s, _capi.ptr6(b.arrays),
                                              threads)
        if st != 0:
            errs.append((st, _capi.last_error()))
        b.set_count(counts[s])

    sheet = [threading.Thread(target=fill, args=(s,)) for s in species if s >= 2]
    for t in sheet:
        t.start()
    for s in species:
        if s < 2:
            fill(s)
    for t in sheet:
        t.join()
    if errs:
        _capi.check(errs[0][0])
    return [batches[s] for s in species]


def init_gem_slab(grid: Grid, ppc: int, rank: int, world: int, seed: int = DEFAULT_SEED,
                  pinned: bool = True, threads: int = 0):
    """This rank's share of the reference GEM state: exactly the particles
    ``Simulation::distribute`` hands to worker ``rank`` (owner_of(y) == rank,
    runtime.cpp:150-166), in the reference's emission order.  Background
    species are generated only for the k-planes' j-rows around the slab (the
    counter RNG jumps ahead); the sheet species, whose count does not grow
    with the domain, are generated whole and filtered."""
    from .partition import decompose, owner_of
    sub = decompose(grid, world)[rank]
    counts = gem_counts(grid, ppc)
    qom, qpp = gem_species_params(grid, ppc)
    g = grid.to_c()
    row = grid.nx * ppc                       # particles per (k, j) row
    j0, j1 = max(sub.j_lo - 1, 0), min(sub.j_hi + 1, grid.ny)
    out = []
    for s in range(4):
        if s < 2:
            # rows that can hold this rank's particles: the slab +- 1 row, and
            # for rank 0 also the top row (y rounding up to ly wraps to 0)
            rows = [(j0, j1)]
            if rank == 0 and j1 < grid.ny:
                rows.append((grid.ny - 1, grid.ny))
            parts = []
            for k in range(grid.nz):
                for ja, jb in rows:
                    m0 = (k * grid.ny + ja) * row
                    m1 = (k * grid.ny + jb) * row
                    arrs = [np.empty(m1 - m0) for _ in range(6)]
                    _capi.check(_capi.lib().b2m_gem_fill_species_range(
                        C.byref(g), ppc, seed, s, m0, m1, _capi.ptr6(arrs), threads))
                    keep = owner_of(arrs[1], grid, world) == rank
                    parts.append([a[keep] for a in arrs])
            p6 = [np.concatenate([p[a] for p in parts]) for a in range(6)]
        else:
            full = init_gem_species(grid, ppc, seed, species=(s,))[0]
            keep = owner_of(full.span()[1], grid, world) == rank
            p6 = [a[keep] for a in full.span()]
        b = ParticleBatch(s, float(qom[s]), float(qpp[s]), len(p6[0]), pinned=pinned)
        b.assign(p6)
        out.append(b)
    return out


def gem_field(grid: Grid) -> FieldMesh:
    """Harris-sheet B with the psi perturbation, E = 0 (init.cpp:72-86)."""
    f = FieldMesh(grid)
    _capi.check(_capi.lib().b2m_gem_field(C.byref(grid.to_c()), _capi.dptr(f.E), _capi.dptr(f.B)))
    return f


def gem_like_field(grid: Grid) -> FieldMesh:
    """E=(0.01 sin y, 0, 0.02), B=(tanh((y-ly/2)/0.5), 0.05 sin x, 0)
    (test_offload.cpp:60-71)."""
    f = FieldMesh(grid)
    _capi.check(_capi.lib().b2m_gem_like_field(C.byref(grid.to_c()), _capi.dptr(f.E),
                                               _capi.dptr(f.B)))
    return f


def gem_bench_field(grid: Grid, z_varying: bool = False) -> FieldMesh:
    """Benchmark field: init_gem's B plus the gem_like_field E (nonzero, so
    the mover's E path is exercised).  Both are z-invariant (the
    GEM problem is 2-D in 3-D).  z_varying=True adds a small z-dependent Ez,
    1e-3 sin(2 pi z / lz), so the general 3-D gather is measured too."""
    f = gem_field(grid)
    E = gem_like_field(grid).E
    f.E[:] = E
    if z_varying:
        nz = grid.nz
        z = np.arange(nz + 1) * (grid.lz / nz)
        dz = 1e-3 * np.sin(2.0 * np.pi * z / grid.lz)
        dz[nz] = dz[0]  # the mirrored seam plane equals plane 0 bit for bit
        Ev = f.E.reshape(nz + 1, grid.ny + 1, grid.nx + 1, 3)
        Ev[..., 2] += dz[:, None, None]
    return f


def gem_mover_params(ppc_grid: Grid, ppc: int, dt: float = 0.1, pc: int = 3):
    qom, _ = gem_species_params(ppc_grid, ppc)
    return [MoverParams.make(dt, float(q), pc) for q in qom]
