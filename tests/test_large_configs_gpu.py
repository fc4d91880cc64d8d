"""Sampled parity at the large SURVEY §8(d) configurations, against the
UNMODIFIED reference mover (oracle/_ref, pic::move_batch built from the
reference's own sources; the C port when it is absent):

  * C4: 64x64x32 cells, 905 ppc -> 255,774,720 particles, pc 3
  * C5: 128x128x64 cells, L = (51.2, 25.6, 12.8), 460 ppc -> 1,002,373,120
        particles (48 GB of SoA), pc 4 and 5, and the general 3-D kernel
        (a z-varying field) at pc 3

The whole state is generated on the host in chunks by the bit-exact GEM
generator and kept resident on the device; one FAST cycle moves ALL of it.
The mover is per-particle independent (kernels.hpp:46-48), so sampled spans --
the head, the middle and the tail of every species, where tile and span
boundaries and 64-bit offsets sit -- are downloaded before and after the
cycle and the "before" copies are moved by the reference on the host.  The
whole state is also checked for size-independent properties: positions inside
the domain, everything finite, per-species counts unchanged.  Needs a B200."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle
from paper_1904_03684_b200 import _capi, gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import Grid, MoverParams
from tests._util import assert_within_contract, cells_of

pytestmark = pytest.mark.gpu

SPAN = 1 << 15
CHUNK = 1 << 24


def _grid(cfg):
    return (Grid.make(128, 128, 64, 51.2, 25.6, 12.8) if cfg == "c5"
            else Grid.make(64, 64, 32, 25.6, 12.8, 6.4))


def _load_state(grid, ppc, field):
    counts = gem.gem_counts(grid, ppc)
    qom, _ = gem.gem_species_params(grid, ppc)
    st = DeviceStore(grid, counts, "fast")
    st.upload_field(field)
    g = grid.to_c()
    for s in range(4):
        if s >= 2:  # the current-sheet species: generated whole (range fill is background-only)
            b = gem.init_gem_species(grid, ppc, species=(s,))[0]
            st.upload(s, b.span())
            continue
        for m0 in range(0, counts[s], CHUNK):
            m1 = min(counts[s], m0 + CHUNK)
            arrs = [np.empty(m1 - m0) for _ in range(6)]
            _capi.check(_capi.lib().b2m_gem_fill_species_range(
                C.byref(g), ppc, gem.DEFAULT_SEED, s, m0, m1, _capi.ptr6(arrs), 0))
            _capi.check(_capi.lib().b2m_species_upload_range(st.h, s, _capi.ptr6(arrs), m0,
                                                             m1 - m0))
        _capi.check(_capi.lib().b2m_species_set_count(st.h, s, counts[s]))
    st.sync()
    return st, counts, [float(q) for q in qom]


def _spans(n):
    starts = sorted({0, max(0, n // 2 - SPAN // 2), max(0, n - SPAN)})
    return [(a, min(SPAN, n - a)) for a in starts]


def _download(st, s, spans):
    out = []
    for a, k in spans:
        p6 = [np.empty(k) for _ in range(6)]
        st.download_range(s, p6, a, k)
        out.append(p6)
    st.sync()
    return out


def _ref_move(p6, field, grid, qom, pc):
    out = [a.copy() for a in p6]
    E, B = field.E.ravel(), field.B.ravel()
    if os.path.exists(oracle.REF_SO):
        oracle.ref_move_batch(out, E, B, grid.as_tuple(), 0.1, qom, pc, threads=8)
    else:
        assert oracle.port_move_batch(out, E, B, grid.as_tuple(), 0.1, qom, pc) == -1
    return out


def _whole_state_properties(st, grid, counts):
    import torch
    from paper_1904_03684_b200.partition import _CudaArray
    L = grid.as_tuple()[3:]
    for s in range(4):
        assert st.count(s) == counts[s]
        ptrs = st.device_ptrs(s)
        cols = [torch.as_tensor(_CudaArray(p, (counts[s],)), device="cuda") for p in ptrs]
        for a in range(3):
            assert bool(((cols[a] >= 0) & (cols[a] < L[a])).all()), (s, a)
        for c in cols:
            assert bool(torch.isfinite(c).all()), s


def _check_cycle(cfg, ppc, pcs, z_varying=False):
    grid = _grid(cfg)
    field = gem.gem_bench_field(grid, z_varying=z_varying)
    st, counts, qom = _load_state(grid, ppc, field)
    try:
        for pc in pcs:
            spans = [_spans(counts[s]) for s in range(4)]
            before = [_download(st, s, spans[s]) for s in range(4)]
            st.move_all([MoverParams.make(0.1, qom[s], pc) for s in range(4)])
            st.sync()
            after = [_download(st, s, spans[s]) for s in range(4)]
            for s in range(4):
                for (a, k), p0, got in zip(spans[s], before[s], after[s]):
                    want = _ref_move(p0, field, grid, qom[s], pc)
                    what = f"{cfg} pc {pc} species {s} [{a}, {a + k})"
                    assert_within_contract(got, want, grid.as_tuple(), what=what)
                    np.testing.assert_array_equal(cells_of(got, grid.as_tuple()),
                                                  cells_of(want, grid.as_tuple()), err_msg=what)
            _whole_state_properties(st, grid, counts)
    finally:
        st.close()


def test_c4_sampled_vs_reference(gpu):
    """SURVEY C4 (the strong-scaling workload), 255,774,720 particles, pc 3."""
    assert sum(gem.gem_counts(_grid("c4"), 905)) == 255774720
    _check_cycle("c4", 905, (3,))


def test_c5_sampled_vs_reference(gpu):
    """SURVEY C5, 1,002,373,120 particles (48 GB SoA) on one B200, pc 4 then
    pc 5 (two consecutive cycles, each checked)."""
    assert sum(gem.gem_counts(_grid("c5"), 460)) == 1002373120
    _check_cycle("c5", 460, (4, 5))


def test_c5_general_3d_kernel_sampled_vs_reference(gpu):
    """C5 with a z-varying field: the general trilinear FAST kernel at 1.0e9
    particles, pc 3."""
    _check_cycle("c5", 460, (3,), z_varying=True)
