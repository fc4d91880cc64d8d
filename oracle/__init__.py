"""TEST INFRASTRUCTURE — the parity checkers.  NOT part of the product.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU baseline.  The product package ``paper_1904_03684_b200`` never
imports it.

Two checkers are exposed through ctypes:

* ``port``  -- ``liboracle_port.so`` built from ``mover_oracle.c``, a plain-C
  restatement of the reference mover (kernels.cpp:10-104, grid.hpp:45-82) and
  of the GEM input generator (init.cpp:21-58, rng.hpp:12-56).
* ``ref``   -- ``_ref/libminipic_ref.so``, the UNMODIFIED reference library
  compiled from its own sources by ``Makefile`` (only where /root/reference is
  present; the built .so travels to the GPU box with the repo snapshot).
* ``ref_b200`` -- ``_ref/libminipic_b200.so``: the same reference library
  with the B200 engine plug-in (integration/) linked in, so the reference's
  own Simulation can be checked against its own CPU engine.

Parity of ``port`` against ``ref`` is pinned by tests/test_oracle.py and by the
golden vectors under tests/golden/ that the reference generated.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle_port.so")
REF_SO = os.path.join(HERE, "_ref", "libminipic_ref.so")
# the reference library with the B200 engine plugged in (integration/Makefile)
B200_SO = os.path.join(HERE, "_ref", "libminipic_b200.so")
REF_SRC = "/root/reference/proj/src/kernels.cpp"

_dp = C.POINTER(C.c_double)
_u64 = C.c_uint64

STATUS_NAMES = {0: "ok", 1: "ConfigError", 2: "DomainError", 3: "AllocError",
                4: "NumericalFault", 5: "CflViolation", 6: "EngineFault",
                7: "MetricError", 99: "Error"}


def build(quiet: bool = True) -> None:
    """Compile the checkers (``make -C oracle``).  The reference library is
    built only when its sources are present (this container)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.msg = msg


# --------------------------------------------------------------------------
# plain-C port
# --------------------------------------------------------------------------
_port = None


def port() -> C.CDLL:
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build()
        lib = C.CDLL(PORT_SO)
        lib.or_wrap_len.restype = C.c_double
        lib.or_wrap_len.argtypes = [C.c_double, C.c_double]
        lib.or_move_batch_g.restype = C.c_int64
        lib.or_move_batch_g.argtypes = [_dp] * 6 + [_u64, _dp, _dp] + [C.c_int] * 3 + \
            [C.c_double] * 3 + [C.c_double, C.c_double, C.c_int]
        lib.or_gem_like_field_g.restype = None
        lib.or_gem_like_field_g.argtypes = [C.c_int] * 3 + [C.c_double] * 3 + [_dp, _dp]
        lib.or_fill_species_g.restype = None
        lib.or_fill_species_g.argtypes = [C.c_int] * 3 + [C.c_double] * 3 + \
            [C.c_int, C.c_int, _u64, C.c_double, _dp, _dp, _u64, _u64] + [_dp] * 6
        lib.or_field_phase_stub_g.restype = None
        lib.or_field_phase_stub_g.argtypes = [C.c_int] * 3 + [_dp, _dp, C.c_int, _dp]
        lib.or_deposit_moments_g.restype = C.c_int64
        lib.or_deposit_moments_g.argtypes = [_dp] * 6 + [_u64] + [C.c_int] * 3 + \
            [C.c_double] * 3 + [C.c_double, C.c_int, C.POINTER(_dp)]
        lib.or_sheet_count_g.restype = _u64
        lib.or_sheet_count_g.argtypes = [C.c_int] * 3 + [C.c_double] * 4 + [C.c_int]
        _port = lib
    return _port


def port_move_batch(p6, E, B, grid, dt, qom, pc) -> int:
    """Oracle mover in place on six float64 arrays.  Returns -1 or the first
    faulting particle index (kernels.cpp:98-99 semantics)."""
    nx, ny, nz, lx, ly, lz = grid
    n = len(p6[0])
    return int(port().or_move_batch_g(*[_ptr(a) for a in p6], n, _ptr(E), _ptr(B),
                                      nx, ny, nz, lx, ly, lz, dt, qom, pc))


def port_deposit_moments(p6, grid, qp: float, with_pressure: bool = False):
    """The C restatement of deposit_moments; returns [rho, jx, jy, jz (, p..)]
    or raises OracleError(DomainError) naming the first particle outside."""
    out = [np.zeros(grid[0] * grid[1] * grid[2]) for _ in range(10 if with_pressure else 4)]
    ptrs = (_dp * 10)(*[_ptr(a) for a in out] + [None] * (10 - len(out)))
    bad = port().or_deposit_moments_g(*[_ptr(np.ascontiguousarray(a)) for a in p6], len(p6[0]),
                                      *grid, qp, int(with_pressure), ptrs)
    if bad >= 0:
        raise OracleError(2, f"particle {bad} outside the domain")
    return out


def port_field_phase_stub(E, B, grid, passes: int):
    """The C restatement of field_phase_stub; returns new (E, B)."""
    E, B = np.array(E, dtype=np.float64), np.array(B, dtype=np.float64)
    scratch = np.empty_like(E)
    port().or_field_phase_stub_g(grid[0], grid[1], grid[2], _ptr(E), _ptr(B), passes,
                                 _ptr(scratch))
    return E, B


def port_wrap_len(v: float, l: float) -> float:
    return port().or_wrap_len(v, l)


def port_gem_like_field(grid):
    nx, ny, nz, lx, ly, lz = grid
    nodes = (nx + 1) * (ny + 1) * (nz + 1)
    E = np.zeros(3 * nodes)
    B = np.zeros(3 * nodes)
    port().or_gem_like_field_g(nx, ny, nz, lx, ly, lz, _ptr(E), _ptr(B))
    return E, B


# GEM species table (config_file.cpp:55-75 with sim_config.hpp:30-39 defaults)
GEM_LAMBDA = 0.5
GEM_UTH_E = 0.045
GEM_UTH_I = 0.0126
GEM_DRIFT = 1.0 / 0.5  # b0/lambda


def gem_species_table():
    """(qom, sheet, uth, u0) for the 4 GEM species in reference order."""
    u_iz = -GEM_DRIFT * 5.0 / (1.0 + 5.0)
    u_ez = +GEM_DRIFT * 1.0 / (1.0 + 5.0)
    ue = np.array([GEM_UTH_E] * 3)
    ui = np.array([GEM_UTH_I] * 3)
    z = np.zeros(3)
    return [(-25.0, 0, ue, z), (1.0, 0, ui, z),
            (-25.0, 1, ue, np.array([0.0, 0.0, u_ez])),
            (1.0, 1, ui, np.array([0.0, 0.0, u_iz]))]


def port_gem_species(grid, ppc: int, seed: int = 12345, species=(0, 1, 2, 3)):
    """GEM particles from the C port, one list of 6 arrays per species."""
    nx, ny, nz, lx, ly, lz = grid
    lib = port()
    out = []
    table = gem_species_table()
    for s in species:
        qom, sheet, uth, u0 = table[s]
        n = lib.or_sheet_count_g(nx, ny, nz, lx, ly, lz, GEM_LAMBDA, ppc) if sheet \
            else ppc * nx * ny * nz
        arrs = [np.empty(n) for _ in range(6)]
        lib.or_fill_species_g(nx, ny, nz, lx, ly, lz, sheet, ppc, n, GEM_LAMBDA,
                              _ptr(np.ascontiguousarray(uth)), _ptr(np.ascontiguousarray(u0)),
                              seed, s, *[_ptr(a) for a in arrs])
        out.append(arrs)
    return out


# --------------------------------------------------------------------------
# unmodified reference library
# --------------------------------------------------------------------------
_ref = None
_ref_b200 = None


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.exists(REF_SRC)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            if not os.path.exists(REF_SRC):
                raise FileNotFoundError("reference library not built and sources absent")
            build()
        _ref = _bind_ref(C.CDLL(REF_SO))
    return _ref


def b200_integration_available() -> bool:
    return os.path.exists(B200_SO)


def ref_b200() -> C.CDLL:
    """The unmodified reference Simulation with libb2m's pic::Engine plugged
    in (integration/minipic_b200_engine.cpp); B2M_ENGINE=1 selects it."""
    global _ref_b200
    if _ref_b200 is None:
        _ref_b200 = _bind_ref(C.CDLL(B200_SO))
    return _ref_b200


def _bind_ref(lib: C.CDLL) -> C.CDLL:
    eb = [C.c_char_p, C.c_int]
    g6 = [C.c_int] * 3 + [C.c_double] * 3
    lib.ref_move_batch.argtypes = [_dp] * 6 + [_u64, _dp, _dp] + g6 + \
        [C.c_double, C.c_double, C.c_int] + eb
    lib.ref_move_batch_mt.argtypes = [_dp] * 6 + [_u64, _dp, _dp] + g6 + \
        [C.c_double, C.c_double, C.c_int, C.c_int] + eb
    lib.ref_wrap_len.argtypes = [C.c_double, C.c_double, _dp]
    lib.ref_grid_cell_of.argtypes = [C.c_double] * 3 + g6 + [C.POINTER(C.c_int), _dp] + eb
    lib.ref_trilinear_weights.argtypes = [C.c_double] * 3 + g6 + \
        [C.POINTER(C.c_int64), _dp] + eb
    lib.ref_implicit_velocity.argtypes = [_dp, _dp, _dp, C.c_double, C.c_double, _dp]
    lib.ref_gem_species.argtypes = g6 + [C.c_int, _dp, _dp, C.POINTER(_u64)] + eb
    lib.ref_init_gem.argtypes = g6 + [C.c_int, _u64, C.POINTER(_dp), _dp, _dp] + eb
    lib.ref_sim_create.argtypes = g6 + [C.c_int, _u64, C.c_int, C.c_int, C.c_int,
                                        C.c_double, C.c_int, C.c_int, C.POINTER(_dp),
                                        C.POINTER(_u64), _dp, _dp,
                                        C.POINTER(C.c_void_p)] + eb
    lib.ref_sim_run.argtypes = [C.c_void_p, C.c_int] + eb
    lib.ref_sim_species_count.argtypes = [C.c_void_p, C.c_int, C.POINTER(_u64)]
    lib.ref_sim_gather.argtypes = [C.c_void_p, C.c_int, C.POINTER(_dp)] + eb
    lib.ref_sim_mean_mover_s.argtypes = [C.c_void_p, _dp]
    lib.ref_sim_destroy.argtypes = [C.c_void_p]
    lib.ref_sim_destroy.restype = None
    lib.ref_mpa.argtypes = [_u64, C.c_double, _dp] + eb
    lib.ref_aggregate_runs.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp] + eb
    lib.ref_decompose.argtypes = [C.c_int] * 4 + [C.POINTER(C.c_int)] + eb
    lib.ref_owner_of.argtypes = [C.c_double] + g6 + [C.c_int]
    lib.ref_field_phase_stub.argtypes = g6 + [_dp, _dp, C.c_int] + eb
    lib.ref_deposit_moments.argtypes = [_dp] * 6 + [_u64] + g6 + [C.c_double, C.c_int,
                                                                   C.POINTER(_dp)] + eb
    return lib


def _errbuf():
    return C.create_string_buffer(512)


def _check(st: int, buf) -> None:
    if st != 0:
        raise OracleError(st, buf.value.decode(errors="replace"))


def ref_move_batch(p6, E, B, grid, dt, qom, pc, threads: int = 0) -> None:
    """pic::move_batch on six float64 arrays (in place).  Raises OracleError
    with status 4 (NumericalFault) exactly when the reference throws."""
    buf = _errbuf()
    n = len(p6[0])
    if threads:
        st = ref().ref_move_batch_mt(*[_ptr(a) for a in p6], n, _ptr(E), _ptr(B), *grid,
                                     dt, qom, pc, threads, buf, 512)
    else:
        st = ref().ref_move_batch(*[_ptr(a) for a in p6], n, _ptr(E), _ptr(B), *grid,
                                  dt, qom, pc, buf, 512)
    _check(st, buf)


MOMENT_NAMES = ("rho", "jx", "jy", "jz", "pxx", "pxy", "pxz", "pyy", "pyz", "pzz")


def _moment_arrays(grid, with_pressure):
    nx, ny, nz = grid[:3]
    return [np.zeros(nx * ny * nz) for _ in range(10 if with_pressure else 4)]


def ref_deposit_moments(p6, grid, qp: float, with_pressure: bool = False):
    """pic::deposit_moments (kernels.cpp:147-183) of six float64 arrays onto
    a fresh MomentMesh; returns [rho, jx, jy, jz (, pxx .. pzz)]."""
    out = _moment_arrays(grid, with_pressure)
    ptrs = (_dp * 10)(*[_ptr(a) for a in out] + [None] * (10 - len(out)))
    buf = _errbuf()
    st = ref().ref_deposit_moments(*[_ptr(np.ascontiguousarray(a)) for a in p6], len(p6[0]),
                                   *grid, qp, int(with_pressure), ptrs, buf, 512)
    _check(st, buf)
    return out


def ref_field_phase_stub(E, B, grid, passes: int):
    """pic::field_phase_stub; returns new (E, B) node AoS arrays."""
    E, B = np.array(E, dtype=np.float64), np.array(B, dtype=np.float64)
    buf = _errbuf()
    _check(ref().ref_field_phase_stub(*grid, _ptr(E), _ptr(B), passes, buf, 512), buf)
    return E, B


def ref_wrap_len(v: float, l: float) -> float:
    out = C.c_double()
    ref().ref_wrap_len(v, l, C.byref(out))
    return out.value


def ref_grid_cell_of(pos, grid):
    buf = _errbuf()
    ijk = (C.c_int * 3)()
    f = np.zeros(3)
    st = ref().ref_grid_cell_of(*pos, *grid, ijk, _ptr(f), buf, 512)
    _check(st, buf)
    return tuple(ijk), f


def ref_trilinear_weights(pos, grid):
    buf = _errbuf()
    idx = (C.c_int64 * 8)()
    w = np.zeros(8)
    st = ref().ref_trilinear_weights(*pos, *grid, idx, _ptr(w), buf, 512)
    _check(st, buf)
    return np.array(idx[:], dtype=np.int64), w


def ref_implicit_velocity(vn, E, B, dt, qom):
    out = np.zeros(3)
    a = [np.ascontiguousarray(x, dtype=np.float64) for x in (vn, E, B)]
    ref().ref_implicit_velocity(_ptr(a[0]), _ptr(a[1]), _ptr(a[2]), dt, qom, _ptr(out))
    return out


def ref_gem_species(grid, ppc):
    buf = _errbuf()
    qom = np.zeros(4)
    qpp = np.zeros(4)
    counts = (_u64 * 4)()
    st = ref().ref_gem_species(*grid, ppc, _ptr(qom), _ptr(qpp), counts, buf, 512)
    _check(st, buf)
    return qom, qpp, [int(c) for c in counts]


def ref_init_gem(grid, ppc, seed=12345, counts=None):
    """pic::init_gem -> (list of 4 species x 6 arrays, E, B)."""
    nx, ny, nz = grid[:3]
    if counts is None:
        counts = ref_gem_species(grid, ppc)[2]
    parts = [[np.empty(n) for _ in range(6)] for n in counts]
    nodes = (nx + 1) * (ny + 1) * (nz + 1)
    E = np.empty(3 * nodes)
    B = np.empty(3 * nodes)
    ptrs = (_dp * 24)(*[_ptr(a) for sp in parts for a in sp])
    buf = _errbuf()
    st = ref().ref_init_gem(*grid, ppc, seed, ptrs, _ptr(E), _ptr(B), buf, 512)
    _check(st, buf)
    return parts, E, B


class RefSimulation:
    """pic::Simulation (runtime.cpp) with a given engine kind / worker count."""

    ENGINES = {"cpu": 0, "naive": 1, "pinned": 2, "prefetch": 3}

    def __init__(self, grid, ppc, workers=1, engine="cpu", pc=3, dt=0.1, field_passes=100,
                 seed=12345, inject=None, lib=None):
        lib = lib or ref()
        self.lib = lib
        buf = _errbuf()
        h = C.c_void_p()
        if inject is None:
            st = lib.ref_sim_create(*grid, ppc, seed, workers, self.ENGINES[engine], pc, dt,
                                    field_passes, 0, None, None, None, None, C.byref(h),
                                    buf, 512)
        else:
            parts, E, B = inject
            self._keep = (parts, E, B)
            ptrs = (_dp * 24)(*[_ptr(a) for sp in parts for a in sp])
            counts = (_u64 * 4)(*[len(sp[0]) for sp in parts])
            st = lib.ref_sim_create(*grid, ppc, seed, workers, self.ENGINES[engine], pc, dt,
                                    field_passes, 1, ptrs, counts, _ptr(E), _ptr(B),
                                    C.byref(h), buf, 512)
        _check(st, buf)
        self.h = h

    def run(self, cycles: int) -> None:
        buf = _errbuf()
        _check(self.lib.ref_sim_run(self.h, cycles, buf, 512), buf)

    def gather(self, s: int):
        n = _u64()
        self.lib.ref_sim_species_count(self.h, s, C.byref(n))
        out = [np.empty(n.value) for _ in range(6)]
        buf = _errbuf()
        _check(self.lib.ref_sim_gather(self.h, s, (_dp * 6)(*[_ptr(a) for a in out]), buf, 512),
               buf)
        return out

    def mean_mover_s(self) -> float:
        out = C.c_double()
        self.lib.ref_sim_mean_mover_s(self.h, C.byref(out))
        return out.value

    def __del__(self):
        if getattr(self, "h", None):
            try:
                self.lib.ref_sim_destroy(self.h)
            except Exception:
                pass
            self.h = None


def multiset(p6) -> np.ndarray:
    """Bitwise multiset of particles (test_runtime.cpp:31-45): rows of the six
    float64 bit patterns, sorted lexicographically."""
    bits = np.stack([np.ascontiguousarray(a).view(np.uint64) for a in p6], axis=1)
    order = np.lexsort(bits.T[::-1])
    return bits[order]
