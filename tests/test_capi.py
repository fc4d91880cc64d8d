"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/b2m.h declares, its value types are layout-identical to the
reference's, host-side validation matches the reference's
error taxonomy, and compute calls fail loudly when no GPU is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
from paper_1904_03684_b200 import _capi
from paper_1904_03684_b200.errors import ConfigError, MinipicError
from paper_1904_03684_b200.mover import Grid, MoverParams, move_batch

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "b2m.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(b2m_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(built):
    lib = C.CDLL(_capi.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding covers exactly the declared surface
    assert sorted(_capi.SIGNATURES) == syms


def test_value_type_layouts(built):
    assert C.sizeof(_capi.b2m_grid) == 64
    assert _capi.b2m_grid.lx.offset == 16 and _capi.b2m_grid.dz.offset == 56
    assert C.sizeof(_capi.b2m_mover_params) == 32
    assert _capi.b2m_mover_params.pc_iterations.offset == 16
    assert _capi.b2m_mover_params.beta.offset == 24


def test_grid_make_validates_like_reference(built):
    with pytest.raises(ConfigError, match="nx,ny,nz must each be >= 2"):
        Grid.make(1, 4, 4, 1, 1, 1)
    with pytest.raises(ConfigError, match="lx,ly,lz must be positive"):
        Grid.make(4, 4, 4, 0.0, 1, 1)
    with pytest.raises(ConfigError):
        Grid.make(4, 4, 4, 1, -2.0, 1)
    g = Grid.make(8, 4, 2, 4.0, 2.0, 1.0)
    assert (g.dx, g.dy, g.dz) == (0.5, 0.5, 0.5)
    assert g.cells() == 64 and g.nodes() == 9 * 5 * 3
    # the default grid has dx = 0.4, dy = dz = 0.2
    d = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
    assert (d.dx, d.dy, d.dz) == (25.6 / 64, 12.8 / 64, 6.4 / 32)


def test_mover_params_make(built):
    p = _capi.b2m_mover_params()
    assert _capi.lib().b2m_mover_params_make(0.1, -25.0, 3, C.byref(p)) == 0
    assert p.beta == -25.0 * 0.1 * 0.5 == MoverParams.make(0.1, -25.0, 3).beta
    assert p.pc_iterations == 3


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library unavailable")
def test_owner_of_matches_reference(built):
    g = Grid.make(8, 8, 8, 6.4, 6.4, 6.4)
    cg = g.to_c()
    r = np.random.default_rng(0)
    ys = list(r.random(2000) * 6.4) + [0.0, np.nextafter(6.4, 0), 1.6, np.nextafter(1.6, 0), 3.2]
    for world in (1, 2, 4):
        for y in ys:
            assert _capi.lib().b2m_owner_of(C.byref(cg), world, y) == \
                oracle.ref().ref_owner_of(y, *g.as_tuple(), world)


def test_status_names(built):
    names = [_capi.lib().b2m_status_name(s).decode() for s in range(10)]
    assert names[:8] == ["ok", "ConfigError", "DomainError", "AllocError", "NumericalFault",
                         "CflViolation", "EngineFault", "MetricError"]


def test_compute_without_gpu_fails_loudly(built):
    if _capi.lib().b2m_device_count() > 0:
        pytest.skip("GPU present: covered by the gpu tests")
    g = Grid.make(4, 4, 4, 4.0, 4.0, 4.0)
    n = g.nodes()
    E = np.zeros(3 * n)
    B = np.zeros(3 * n)
    p = [np.ones(4) for _ in range(6)]
    with pytest.raises(MinipicError):
        move_batch(p, (E, B), g, MoverParams.make(0.1, 1.0, 3))


def test_world_entry_points_validate_before_touching_a_gpu(built):
    """The native world's argument checks (no GPU needed): null id buffer,
    null / non-world contexts, bad loopback arguments."""
    lib = _capi.lib()
    INVALID = 9  # B2M_INVALID_ARGUMENT
    assert lib.b2m_world_id(None) == INVALID
    arr = (_capi.b2m_mover_params * 1)(MoverParams.make(0.1, 1.0, 3).to_c())
    assert lib.b2m_world_step(None, arr, None, None) == INVALID
    assert lib.b2m_world_init(None, None, 0, 1) == INVALID
    assert lib.b2m_world_set_total(None, None) == INVALID
    assert lib.b2m_world_broadcast_field(None, 0) == INVALID
    assert lib.b2m_world_reduce_moments(None) == INVALID
    assert lib.b2m_world_loopback_step(None, 2, arr, None) == INVALID
    assert "null" in _capi.last_error() or "bad arguments" in _capi.last_error()


def test_integration_world_example_compiles(built, tmp_path):
    """INTEGRATION.md's native-world cycle compiles against include/b2m.h and
    links against libb2m.so (compile only: running it needs GPUs)."""
    import shutil
    import subprocess
    gxx = shutil.which("g++")
    if not gxx:
        pytest.skip("no g++")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    so = tmp_path / "libexample.so"
    r = subprocess.run([gxx, "-std=c++17", "-fPIC", "-shared", "-I", os.path.join(root, "include"),
                        os.path.join(root, "integration", "world_example.cpp"), "-o", str(so),
                        "-L", os.path.dirname(_capi.LIB_PATH), "-lb2m"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
