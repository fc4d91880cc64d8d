"""Reference-facing mover API: the B200 drop-in for ``pic::move_batch``.

Mirrors the reference's core types and kernel call so code written against
minipic reads the same:

* ``Grid``          grid.hpp:15-41 (``Grid.make`` validates like ``Grid::make``)
* ``MoverParams``   kernels.hpp:30-39 (``beta = qom*dt*0.5``)
* ``ParticleBatch`` particle_batch.hpp:29-85 (SoA x,y,z,u,v,w; fixed capacity)
* ``FieldMesh``     field_mesh.hpp:23-60 (node-centred E,B with mirrored seams)
* ``move_batch``    kernels.hpp:49 / kernels.cpp:52-104

``move_batch`` runs the hand-written sm_100a kernel through the C ABI
(``b2m_move_batch_host``).  There is no CPU fallback: without libb2m.so or a
GPU the call raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from .errors import AllocError, NumericalFault

MODES = {"strict": 0, "fast": 1}


def _mode(mode) -> int:
    if isinstance(mode, int):
        return mode
    return MODES[mode]


@dataclass(frozen=True)
class Grid:
    nx: int
    ny: int
    nz: int
    lx: float
    ly: float
    lz: float
    dx: float
    dy: float
    dz: float

    @staticmethod
    def make(nx: int, ny: int, nz: int, lx: float, ly: float, lz: float) -> "Grid":
        g = _capi.b2m_grid()
        _capi.check(_capi.lib().b2m_grid_make(nx, ny, nz, lx, ly, lz, C.byref(g)))
        return Grid(g.nx, g.ny, g.nz, g.lx, g.ly, g.lz, g.dx, g.dy, g.dz)

    def cells(self) -> int:
        return self.nx * self.ny * self.nz

    def nodes(self) -> int:
        return (self.nx + 1) * (self.ny + 1) * (self.nz + 1)

    def node_index(self, i: int, j: int, k: int) -> int:
        return i + (self.nx + 1) * (j + (self.ny + 1) * k)

    def cell_volume(self) -> float:
        return self.dx * self.dy * self.dz

    def as_tuple(self):
        return (self.nx, self.ny, self.nz, self.lx, self.ly, self.lz)

    def to_c(self) -> _capi.b2m_grid:
        g = _capi.b2m_grid()
        g.nx, g.ny, g.nz = self.nx, self.ny, self.nz
        g.lx, g.ly, g.lz = self.lx, self.ly, self.lz
        g.dx, g.dy, g.dz = self.dx, self.dy, self.dz
        return g


@dataclass(frozen=True)
class MoverParams:
    dt: float = 0.0
    qom: float = 0.0
    pc_iterations: int = 1
    beta: float = 0.0

    @staticmethod
    def make(dt: float, qom: float, pc_iterations: int) -> "MoverParams":
        return MoverParams(dt, qom, pc_iterations, qom * dt * 0.5)

    def to_c(self) -> _capi.b2m_mover_params:
        p = _capi.b2m_mover_params()
        p.dt, p.qom, p.pc_iterations, p.beta = self.dt, self.qom, self.pc_iterations, self.beta
        return p


class FieldMesh:
    """Node-centred E and B, ``(nodes, 3)`` float64 each, node-major index
    i + j*(nx+1) + k*(nx+1)*(ny+1); seam planes duplicate the 0-planes."""

    def __init__(self, grid: Grid, E=None, B=None):
        n = grid.nodes()
        self.nx1, self.ny1, self.nz1 = grid.nx + 1, grid.ny + 1, grid.nz + 1
        self.E = np.zeros((n, 3)) if E is None else np.ascontiguousarray(E, dtype=np.float64).reshape(n, 3)
        self.B = np.zeros((n, 3)) if B is None else np.ascontiguousarray(B, dtype=np.float64).reshape(n, 3)

    @staticmethod
    def make(grid: Grid) -> "FieldMesh":
        return FieldMesh(grid)

    def node_count(self) -> int:
        return self.E.shape[0]

    def index(self, i: int, j: int, k: int) -> int:
        return i + self.nx1 * (j + self.ny1 * k)

    def mirror_seams(self) -> None:
        """field_mesh.hpp:46-59"""
        nx, ny, nz = self.nx1 - 1, self.ny1 - 1, self.nz1 - 1
        for F in (self.E, self.B):
            G = F.reshape(nz + 1, ny + 1, nx + 1, 3)
            G[:, :, nx] = G[:, :, 0]
            G[:, ny, :] = G[:, 0, :]
            G[nz, :, :] = G[0, :, :]


def field_phase_stub(mesh: FieldMesh, grid: Grid, passes: int) -> FieldMesh:
    """The field-phase stand-in on the GPU (kernels.cpp:185-215): a new mesh
    with ``passes`` rounds of 7-point averaging of E (B unchanged, seams
    mirrored), bit-identical to the reference."""
    out = FieldMesh(grid, mesh.E.copy(), mesh.B.copy())
    if passes > 0:
        g = grid.to_c()
        _capi.check(_capi.lib().b2m_field_phase_stub_host(C.byref(g), _capi.dptr(out.E),
                                                          _capi.dptr(out.B), int(passes)))
    return out


class ParticleBatch:
    """SoA store of one species with fixed capacity (particle_batch.hpp:29-85).

    ``pinned=True`` allocates page-locked host memory through libb2m so the
    engine's host<->device copies run asynchronously."""

    def __init__(self, species_id: int, qom: float, q_per_particle: float, capacity: int,
                 pinned: bool = False):
        self.species_id = species_id
        self.qom = qom
        self.q_per_particle = q_per_particle
        self._capacity = int(capacity)
        self._count = 0
        self._pinned_ptr = None
        if pinned and capacity > 0:
            p = C.c_void_p()
            _capi.check(_capi.lib().b2m_host_alloc(6 * 8 * capacity, C.byref(p)))
            self._pinned_ptr = p
            buf = (C.c_double * (6 * capacity)).from_address(p.value)
            flat = np.frombuffer(buf, dtype=np.float64)
        else:
            flat = np.zeros(6 * max(capacity, 1))
        self._flat = flat
        self.arrays = [flat[a * capacity:(a + 1) * capacity] for a in range(6)]

    def __del__(self):
        if getattr(self, "_pinned_ptr", None) is not None:
            try:
                self.arrays = None
                self._flat = None
                _capi.lib().b2m_host_free(self._pinned_ptr)
            except Exception:
                pass
            self._pinned_ptr = None

    x = property(lambda s: s.arrays[0][:s._count])
    y = property(lambda s: s.arrays[1][:s._count])
    z = property(lambda s: s.arrays[2][:s._count])
    u = property(lambda s: s.arrays[3][:s._count])
    v = property(lambda s: s.arrays[4][:s._count])
    w = property(lambda s: s.arrays[5][:s._count])

    def count(self) -> int:
        return self._count

    def capacity(self) -> int:
        return self._capacity

    def bytes(self) -> int:
        return 6 * 8 * self._count

    def span(self):
        """Six float64 views of the live particles (ParticleSpan)."""
        return [a[:self._count] for a in self.arrays]

    def append(self, x, y, z, u, v, w) -> None:
        if self._count == self._capacity:
            raise AllocError("particle batch capacity exceeded (fixed at allocation)")
        for a, val in zip(self.arrays, (x, y, z, u, v, w)):
            a[self._count] = val
        self._count += 1

    def assign(self, p6) -> None:
        n = len(p6[0])
        if n > self._capacity:
            raise AllocError("particle batch capacity exceeded (fixed at allocation)")
        for a, src in zip(self.arrays, p6):
            a[:n] = src
        self._count = n

    def set_count(self, n: int) -> None:
        if n > self._capacity:
            raise AllocError("particle batch count > capacity")
        self._count = int(n)


def _as_span(p):
    if isinstance(p, ParticleBatch):
        return p.span()
    return list(p)


def move_batch(p, field, grid: Grid, mp: MoverParams, mode="fast") -> None:
    """Advance every particle one step on the GPU (kernels.cpp:52-104).

    ``p`` is a ParticleBatch or six float64 arrays (ParticleSpan), updated in
    place; ``field`` a FieldMesh or an ``(E, B)`` pair in FieldView layout.
    Raises ``NumericalFault("mover produced non-finite state at particle index
    i")`` like the reference: particles before i are updated, i and later are
    untouched.  ``mode``: "fast" (FMA; 1e-12 contract) or "strict"
    (bit-identical to the reference)."""
    span = _as_span(p)
    for a in span:
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise TypeError("particle arrays must be contiguous float64")
    n = len(span[0])
    if isinstance(field, FieldMesh):
        E, B = field.E, field.B
    else:
        E, B = field
    E = np.ascontiguousarray(E, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    if E.size != 3 * grid.nodes() or B.size != 3 * grid.nodes():
        from .errors import ConfigError
        raise ConfigError("field: node count does not match the grid")
    g = grid.to_c()
    cmp = mp.to_c()
    bad = C.c_int64(-1)
    st = _capi.lib().b2m_move_batch_host(C.byref(g), C.byref(cmp), _capi.dptr(E), _capi.dptr(B),
                                         *[_capi.dptr(a) for a in span], n, _mode(mode),
                                         C.byref(bad))
    if st == 4:
        raise NumericalFault(_capi.last_error(), index=bad.value)
    _capi.check(st)


class MomentMesh:
    """Charge, current and (optionally) pressure on the nx*ny*nz periodic
    nodes (MomentMesh, kernels.hpp:54-69; index i + nx*(j + ny*k))."""

    NAMES = ("rho", "jx", "jy", "jz", "pxx", "pxy", "pxz", "pyy", "pyz", "pzz")

    def __init__(self, nx: int, ny: int, nz: int, with_pressure: bool = False):
        self.nx, self.ny, self.nz = nx, ny, nz
        self.with_pressure = bool(with_pressure)
        n = nx * ny * nz
        self.arrays = [np.zeros(n) for _ in range(10 if with_pressure else 4)]
        for name, a in zip(self.NAMES, self.arrays):
            setattr(self, name, a)

    @staticmethod
    def make(grid: Grid, with_pressure: bool = False) -> "MomentMesh":
        return MomentMesh(grid.nx, grid.ny, grid.nz, with_pressure)

    def index(self, i: int, j: int, k: int) -> int:
        return i + self.nx * (j + self.ny * k)

    def zero(self) -> None:
        for a in self.arrays:
            a[:] = 0.0

    def add(self, other: "MomentMesh") -> None:
        n = 10 if (self.with_pressure and other.with_pressure) else 4
        for a, b in zip(self.arrays[:n], other.arrays[:n]):
            a += b

    def total_charge(self, grid: Grid) -> float:
        # MomentMesh::total_charge (kernels.cpp:141-145): sequential sum * volume
        return float(np.cumsum(self.rho)[-1]) * grid.cell_volume() if self.rho.size else 0.0


def deposit_moments(b, grid: Grid, out: MomentMesh, q_per_particle: float | None = None) -> None:
    """Scatter the particles' charge, current (and pressure) onto ``out`` on the
    GPU (deposit_moments, kernels.cpp:147-183); ``out`` accumulates.  ``b`` is
    a ParticleBatch (its q_per_particle) or six float64 arrays with
    ``q_per_particle`` given.  Raises DomainError for a particle outside the
    domain, like the reference's grid_cell_of."""
    span = _as_span(b)
    qp = b.q_per_particle if isinstance(b, ParticleBatch) else q_per_particle
    if qp is None:
        raise TypeError("q_per_particle required for raw arrays")
    span = [np.ascontiguousarray(a, dtype=np.float64) for a in span]
    g = grid.to_c()
    ptrs = (_capi._dp * len(out.arrays))(*[_capi.dptr(a) for a in out.arrays])
    _capi.check(_capi.lib().b2m_deposit_moments_host(C.byref(g), *[_capi.dptr(a) for a in span],
                                                     len(span[0]), float(qp),
                                                     int(out.with_pressure), ptrs))
