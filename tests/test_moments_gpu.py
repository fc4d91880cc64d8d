"""GPU parity of moment deposition (deposit_moments, kernels.cpp:147-183)
against the pinned C oracle.

Per-particle terms are computed exactly as the reference (same divisions,
same products), so single-particle meshes are bit-identical; sums over many
particles are added in another order (per-lane cell runs + FP64 atomics), so
they agree to rounding: |gpu - ref| <= 1e-12 * max|ref| per array (the
reference's own tests use 1e-12 relative on totals, test_kernels.cpp:274).
Mirrors test_kernels.cpp:232-295 and test_init.cpp:131-143.
"""
import numpy as np
import pytest

import oracle
from paper_1904_03684_b200 import DomainError, Grid, MomentMesh, deposit_moments
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import MoverParams
from tests._util import random_particles

pytestmark = pytest.mark.gpu

TOL = 1e-12


def assert_moments_close(got, want, tol=TOL, what=""):
    assert len(got) == len(want)
    for name, g, w in zip(MomentMesh.NAMES, got, want):
        scale = float(np.max(np.abs(w))) if w.size else 0.0
        err = float(np.max(np.abs(g - w))) if w.size else 0.0
        if scale == 0.0:
            assert err == 0.0, f"{what} {name}: expected zeros, max |got| {err}"
        else:
            assert err <= tol * scale, f"{what} {name}: max err {err:.3e} vs scale {scale:.3e}"


def gpu_deposit(p6, grid, qp, pressure=False):
    g = Grid.make(*grid)
    m = MomentMesh.make(g, pressure)
    deposit_moments([np.ascontiguousarray(a) for a in p6], g, m, q_per_particle=qp)
    return m


def test_single_particle_corners_and_seam_bitwise(gpu):
    """test_kernels.cpp:232-256: one term per node -> bit-identical."""
    grid = (4, 4, 4, 4.0, 4.0, 4.0)
    for x, u in ((0.5, 2.0), (3.5, 0.0)):
        p = [np.array([x]), np.array([x]), np.array([x]), np.array([u]), np.zeros(1),
             np.zeros(1)]
        m = gpu_deposit(p, grid, 0.75, pressure=True)
        want = oracle.port_deposit_moments(p, grid, 0.75, True)
        for a, b in zip(m.arrays, want):
            np.testing.assert_array_equal(a, b)
        assert m.total_charge(Grid.make(*grid)) == pytest.approx(0.75, rel=1e-15)


def test_random_batch_conserves_charge_and_current(gpu):
    """test_kernels.cpp:258-280: 5000 particles; total charge and current."""
    grid = (6, 5, 7, 3.0, 2.5, 3.5)
    p = random_particles(grid, 5000, 31, vscale=1.0)
    q = -0.0125
    m = gpu_deposit(p, grid, q, pressure=True)
    assert_moments_close(m.arrays, oracle.port_deposit_moments(p, grid, q, True), what="random")
    g = Grid.make(*grid)
    assert abs(m.total_charge(g) - q * 5000) <= 1e-12 * abs(q * 5000)
    assert float(np.sum(m.jx)) * g.cell_volume() == pytest.approx(q * float(np.sum(p[3])),
                                                                    rel=1e-11)


def test_gem_c1_all_species_with_pressure(gpu, golden):
    """The reference C1 GEM state (oracle-pinned, golden.json c1_moments):
    every species' moments incl. the pressure tensor."""
    gd = golden["c1_init"]
    grid = tuple(gd["grid"])
    parts = oracle.port_gem_species(grid, gd["ppc"], gd["seed"])
    qpp = [float.fromhex(h) for h in golden["c1_moments"]["qpp"]]
    for s, p in enumerate(parts):
        m = gpu_deposit(p, grid, qpp[s], pressure=True)
        assert_moments_close(m.arrays, oracle.port_deposit_moments(p, grid, qpp[s], True),
                             what=f"species {s}")


def test_quasi_neutral_gem_total_charge(gpu):
    """test_init.cpp:131-143: the GEM state is neutral to 1e-12 of |q|."""
    g = Grid.make(16, 16, 8, 12.8, 6.4, 3.2)
    batches = gem.init_gem_species(g, 8)
    m = MomentMesh.make(g)
    abs_q = 0.0
    for b in batches:
        deposit_moments(b, g, m)
        abs_q += abs(b.q_per_particle) * b.count()
    assert abs(m.total_charge(g)) <= 1e-12 * abs_q


def test_domain_error_names_reference_message(gpu):
    grid = (4, 4, 4, 4.0, 4.0, 4.0)
    p = [np.array([1.0, 4.0]), np.array([1.0, 1.0]), np.array([1.0, 1.0]), np.zeros(2),
         np.zeros(2), np.zeros(2)]
    with pytest.raises(DomainError, match="outside domain"):
        gpu_deposit(p, grid, 1.0)


def test_device_store_deposit_after_move_and_sort(gpu):
    """Engine-level: resident particles are moved, cell-sorted, then
    deposited on the device; equals the oracle deposit of the same particles
    (cell order does not change the moments beyond rounding)."""
    g = Grid.make(16, 16, 8, 6.4, 6.4, 3.2)
    grid = g.as_tuple()
    batches = gem.init_gem_species(g, 8)
    field = gem.gem_like_field(g)
    mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
    st = DeviceStore(g, [b.count() for b in batches], "fast")
    st.upload_field(field)
    for s, b in enumerate(batches):
        st.upload(s, b.span())
    st.move_all(mps)
    for s in range(len(batches)):
        st.sort(s)
    st.moments_zero(with_pressure=True)
    for s, b in enumerate(batches):
        st.deposit(s, b.q_per_particle)
    mine = MomentMesh.make(g, True)
    st.moments_download(mine)
    want = [np.zeros(g.cells()) for _ in range(10)]
    for s, b in enumerate(batches):
        p = [np.empty(b.count()) for _ in range(6)]
        st.download(s, p)
        st.sync()
        for a, w in zip(oracle.port_deposit_moments(p, grid, b.q_per_particle, True), want):
            w += a
    assert_moments_close(mine.arrays, want, what="device store")


def test_unsorted_large_batch(gpu):
    """Random order (every particle its own cell run): the flush-per-particle
    path, 200k particles."""
    grid = (32, 16, 16, 12.8, 6.4, 6.4)
    p = random_particles(grid, 200_000, 7)
    m = gpu_deposit(p, grid, 0.01, pressure=False)
    assert_moments_close(m.arrays, oracle.port_deposit_moments(p, grid, 0.01, False),
                         what="unsorted")


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
def test_against_the_reference_library_itself(gpu):
    """The UNMODIFIED reference deposit_moments on the same particles."""
    grid = (6, 5, 7, 3.0, 2.5, 3.5)
    p = random_particles(grid, 20000, 33, vscale=1.0)
    m = gpu_deposit(p, grid, -0.0125, pressure=True)
    assert_moments_close(m.arrays, oracle.ref_deposit_moments(p, grid, -0.0125, True),
                         what="vs reference")


@pytest.mark.parametrize("order", ["random", "sorted", "sorted_jittered"])
def test_cell_groups_runs_and_strays(gpu, order):
    """The warp-group deposit's paths: many particles per cell within 32
    (shared-memory group sums), runs of one cell across groups (the carried
    cell), strays alone in their cell (direct atomics), a ragged tail."""
    grid = (4, 4, 4, 4.0, 4.0, 4.0)
    n = 100_003
    p = random_particles(grid, n, 41, vscale=1.0)
    cell = (np.floor(p[0]).astype(np.int64) + 4 * (np.floor(p[1]).astype(np.int64)
            + 4 * np.floor(p[2]).astype(np.int64)))
    if order != "random":
        perm = np.argsort(cell, kind="stable")
        if order == "sorted_jittered":
            rng = np.random.default_rng(5)
            sw = rng.integers(0, n, size=(n // 10, 2))
            for a, b in sw:
                perm[a], perm[b] = perm[b], perm[a]
        p = [np.ascontiguousarray(a[perm]) for a in p]
    m = gpu_deposit(p, grid, 0.003, pressure=True)
    assert_moments_close(m.arrays, oracle.port_deposit_moments(p, grid, 0.003, True),
                         what=order)


@pytest.mark.parametrize("mode", ["fast", "strict"])
def test_deposit_on_drifted_state(gpu, mode):
    """The realistic cycle state: cell-sorted, then several mover steps of
    drift (runs broken, strays in neighbouring cells) before the deposit."""
    g = Grid.make(16, 16, 8, 6.4, 6.4, 3.2)
    grid = g.as_tuple()
    batches = gem.init_gem_species(g, 16)
    field = gem.gem_like_field(g)
    mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
    st = DeviceStore(g, [b.count() for b in batches], mode)
    st.upload_field(field)
    for s, b in enumerate(batches):
        st.upload(s, b.span())
        st.sort(s)
    for _ in range(6):
        st.move_all(mps)
    st.moments_zero(with_pressure=True)
    for s, b in enumerate(batches):
        st.deposit(s, b.q_per_particle)
    mine = MomentMesh.make(g, True)
    st.moments_download(mine)
    want = [np.zeros(g.cells()) for _ in range(10)]
    for s, b in enumerate(batches):
        p = [np.empty(b.count()) for _ in range(6)]
        st.download(s, p)
        st.sync()
        for a, w in zip(oracle.port_deposit_moments(p, grid, b.q_per_particle, True), want):
            w += a
    assert_moments_close(mine.arrays, want, what=f"drifted {mode}")


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
def test_full_c2_moments_vs_reference(gpu):
    """All 61,046,784 C2 particles, cell-sorted then moved once (drifted):
    rho, J and the pressure tensor from the device deposit agree with the
    UNMODIFIED reference deposit_moments over the same particles."""
    g = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
    grid = g.as_tuple()
    batches = gem.init_gem_species(g, 216, pinned=True)
    st = DeviceStore(g, [b.count() for b in batches], "strict")
    st.upload_field(gem.gem_bench_field(g))
    for s, b in enumerate(batches):
        st.upload(s, b.span())
        st.sort(s)
    st.move_all([MoverParams.make(0.1, b.qom, 3) for b in batches])
    st.moments_zero(with_pressure=True)
    for s, b in enumerate(batches):
        st.deposit(s, b.q_per_particle)
    mine = MomentMesh.make(g, True)
    st.moments_download(mine)
    want = [np.zeros(g.cells()) for _ in range(10)]
    for s, b in enumerate(batches):
        p = [np.empty(b.count()) for _ in range(6)]
        st.download(s, p)
        st.sync()
        for a, w in zip(oracle.ref_deposit_moments(p, grid, b.q_per_particle, True), want):
            w += a
    assert_moments_close(mine.arrays, want, what="C2 vs reference")


def test_empty_species_and_batches(gpu):
    """An empty batch deposits nothing; a store whose species are empty
    moves, sorts and deposits without touching the mesh."""
    grid = (4, 4, 4, 4.0, 4.0, 4.0)
    p = [np.empty(0) for _ in range(6)]
    m = gpu_deposit(p, grid, 1.0, pressure=True)
    assert all(not np.any(a) for a in m.arrays)
    g = Grid.make(*grid)
    st = DeviceStore(g, [0, 16], "strict")
    st.upload_field(gem.gem_field(g))
    q = random_particles(grid, 16, 3)
    st.upload(1, q)
    mps = [MoverParams.make(0.1, -25.0, 3), MoverParams.make(0.1, 1.0, 3)]
    st.move_all(mps)
    st.sort(0)
    st.sort(1)
    st.moments_zero(with_pressure=False)
    st.deposit(0, 1.0)
    mine = MomentMesh.make(g, False)
    st.moments_download(mine)
    assert all(not np.any(a) for a in mine.arrays)
    assert st.count(0) == 0 and st.count(1) == 16
    st.close()


# ---- the fused mover + deposit (b2m_move_deposit_all, b2m_fused.cuh) -------

def _two_stores(g, batches, field, mode, sort=True, steps=0, mps=None):
    """Two identical device stores of `batches` (optionally sorted, then
    `steps` plain mover cycles of drift)."""
    out = []
    for _ in range(2):
        st = DeviceStore(g, [b.count() for b in batches], mode)
        st.upload_field(field)
        for s, b in enumerate(batches):
            st.upload(s, b.span())
            if sort:
                st.sort(s)
        for _ in range(steps):
            st.move_all(mps)
        out.append(st)
    return out


def _fused_vs_separate(g, batches, field, mode="fast", sort=True, steps=0, pressure=False):
    mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
    qs = [b.q_per_particle for b in batches]
    a, b_ = _two_stores(g, batches, field, mode, sort, steps, mps)
    a.moments_zero(pressure)
    a.move_all(mps)
    for s, q in enumerate(qs):
        a.deposit(s, q)
    b_.moments_zero(pressure)
    b_.move_deposit_all(mps, qs)
    ma, mb = MomentMesh.make(g, pressure), MomentMesh.make(g, pressure)
    a.moments_download(ma)
    b_.moments_download(mb)
    # the mover arithmetic is the same code: particles bit-identical (as a
    # multiset -- the counting sort's order within a cell is not deterministic)
    for s, bt in enumerate(batches):
        pa = [np.empty(bt.count()) for _ in range(6)]
        pb = [np.empty(bt.count()) for _ in range(6)]
        a.download(s, pa)
        b_.download(s, pb)
        a.sync()
        b_.sync()
        ra = np.stack([x.view(np.uint64) for x in pa], 1)
        rb = np.stack([x.view(np.uint64) for x in pb], 1)
        ra = ra[np.lexsort(ra.T[::-1])]
        rb = rb[np.lexsort(rb.T[::-1])]
        np.testing.assert_array_equal(ra, rb)
    # and the moments of the moved state: the oracle's deposit of it
    want = [np.zeros(g.cells()) for _ in range(10 if pressure else 4)]
    for s, bt in enumerate(batches):
        p = [np.empty(bt.count()) for _ in range(6)]
        b_.download(s, p)
        b_.sync()
        for x, w in zip(oracle.port_deposit_moments(p, g.as_tuple(), bt.q_per_particle,
                                                    pressure), want):
            w += x
    a.close()
    b_.close()
    return ma, mb, want


@pytest.mark.parametrize("zvar", [False, True])
@pytest.mark.parametrize("sort,steps", [(True, 0), (True, 6), (False, 0)])
def test_fused_move_deposit_vs_separate_and_oracle(gpu, zvar, sort, steps):
    """One fused launch (FAST, rho + J through FP64 DMMA in the mover's tile
    loop) against b2m_move_all + b2m_deposit and against the oracle deposit of
    the moved state: the column kernel (z-invariant field) and the general
    3-D kernel (z-varying), right after a sort, after drift, and unsorted
    (GEM init order: every row mixes cells)."""
    g = Grid.make(16, 16, 8, 6.4, 6.4, 3.2)
    batches = gem.init_gem_species(g, 24)
    field = gem.gem_bench_field(g, z_varying=zvar)
    ma, mb, want = _fused_vs_separate(g, batches, field, sort=sort, steps=steps)
    assert_moments_close(mb.arrays, want, what="fused vs oracle")
    assert_moments_close(mb.arrays, ma.arrays, what="fused vs separate")


@pytest.mark.parametrize("mode,pressure", [("strict", False), ("fast", True)])
def test_move_deposit_all_unfused_paths(gpu, mode, pressure):
    """STRICT (bit-identical terms) and the pressure tensor take the
    mover-then-deposit path of b2m_move_deposit_all: same results."""
    g = Grid.make(8, 8, 8, 6.4, 6.4, 6.4)
    batches = gem.init_gem_species(g, 16)
    ma, mb, want = _fused_vs_separate(g, batches, gem.gem_bench_field(g), mode=mode,
                                      pressure=pressure)
    assert_moments_close(mb.arrays, ma.arrays, what=f"{mode} pressure={pressure} vs separate")
    assert_moments_close(mb.arrays, want, what=f"{mode} pressure={pressure}")


def test_fused_deposit_skips_faulted_particles(gpu):
    """A particle that faults in the mover (NaN velocity) is not deposited
    and does not poison the accumulator: the mesh equals the deposit of the
    other particles; the fault is reported by sync."""
    g = Grid.make(8, 8, 8, 6.4, 6.4, 6.4)
    grid = g.as_tuple()
    p = random_particles(grid, 4099, 77, vscale=0.05)
    p[3][1000] = np.nan
    st = DeviceStore(g, [4099], "fast")
    st.upload_field(gem.gem_bench_field(g))
    st.upload(0, p)
    st.moments_zero(False)
    ptr, n = st.moments_device()
    st.move_deposit_all([MoverParams.make(0.1, -25.0, 3)], [0.5])
    import torch
    from paper_1904_03684_b200.partition import _CudaArray
    torch.cuda.synchronize()
    mesh = torch.as_tensor(_CudaArray(ptr, (n,)), device="cuda").cpu().numpy().copy()
    from paper_1904_03684_b200.errors import NumericalFault as NF
    with pytest.raises(NF):
        st.sync()
    st.close()
    # the expected mesh: every particle but the faulted one, moved by the oracle
    q = [np.delete(a, 1000) for a in p]
    E, B = gem.gem_bench_field(g).E.ravel(), gem.gem_bench_field(g).B.ravel()
    assert oracle.port_move_batch(q, E, B, grid, 0.1, -25.0, 3) == -1
    want = oracle.port_deposit_moments(q, grid, 0.5, False)
    assert np.all(np.isfinite(mesh))
    assert_moments_close(list(mesh.reshape(4, -1)), want, what="faulted particle skipped")


def test_fused_full_c2_vs_separate(gpu):
    """All 61,046,784 C2 particles (gem+E, z-invariant: the column kernel),
    cell-sorted: fused rho + J equal the separate deposit to rounding and the
    moved particles are bit-identical (every array as a sorted multiset)."""
    g = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
    batches = gem.init_gem_species(g, 216, pinned=True)
    mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
    qs = [b.q_per_particle for b in batches]
    a, b_ = _two_stores(g, batches, gem.gem_bench_field(g), "fast", True, 0, mps)
    a.moments_zero(False)
    a.move_all(mps)
    for s, q in enumerate(qs):
        a.deposit(s, q)
    b_.moments_zero(False)
    b_.move_deposit_all(mps, qs)
    ma, mb = MomentMesh.make(g, False), MomentMesh.make(g, False)
    a.moments_download(ma)
    b_.moments_download(mb)
    assert_moments_close(mb.arrays, ma.arrays, what="C2 fused vs separate")
    import torch
    from paper_1904_03684_b200.partition import _CudaArray
    for s, bt in enumerate(batches):
        # multiset equality of the moved particles (the sort's order within a
        # cell is not deterministic): sorted columns of every array
        for c, (pa, pb) in enumerate(zip(a.device_ptrs(s), b_.device_ptrs(s))):
            ta = torch.as_tensor(_CudaArray(pa, (bt.count(),)), device="cuda")
            tb = torch.as_tensor(_CudaArray(pb, (bt.count(),)), device="cuda")
            assert bool((torch.sort(ta)[0].view(torch.int64) ==
                         torch.sort(tb)[0].view(torch.int64)).all()), (s, c)
    a.close()
    b_.close()


def _fast_store_deposit(p, grid, q, pressure=False):
    g = Grid.make(*grid)
    st = DeviceStore(g, [len(p[0])], "fast")
    st.upload_field(gem.gem_field(g))
    st.upload(0, p)
    st.moments_zero(pressure)
    st.deposit(0, q)
    m = MomentMesh.make(g, pressure)
    st.moments_download(m)
    st.close()
    return m


@pytest.mark.parametrize("pressure", [False, True])
@pytest.mark.parametrize("order", ["random", "sorted", "sorted_jittered", "one_cell"])
def test_fast_dmma_deposit_paths_vs_oracle(gpu, order, pressure):
    """The FAST rho + J kernel (deposit_dmma_kernel) on every path: rows in
    one cell (the carried cell across rows), runs across rows, groups taken
    by the extra DMMA passes, strays by direct atomics (random order), one
    cell holding everything; a ragged tail."""
    grid = (4, 4, 4, 4.0, 4.0, 4.0)
    n = 100_003
    p = random_particles(grid, n, 43, vscale=1.0)
    if order == "one_cell":
        p[0] = 1.0 + 0.999 * (p[0] / 4.0)
        p[1] = 2.0 + 0.999 * (p[1] / 4.0)
        p[2] = 3.0 + 0.999 * (p[2] / 4.0)
    cell = (np.floor(p[0]).astype(np.int64) + 4 * (np.floor(p[1]).astype(np.int64)
            + 4 * np.floor(p[2]).astype(np.int64)))
    if order in ("sorted", "sorted_jittered"):
        perm = np.argsort(cell, kind="stable")
        if order == "sorted_jittered":
            rng = np.random.default_rng(9)
            for a, b in rng.integers(0, n, size=(n // 10, 2)):
                perm[a], perm[b] = perm[b], perm[a]
        p = [np.ascontiguousarray(a[perm]) for a in p]
    m = _fast_store_deposit(p, grid, 0.003, pressure)
    assert_moments_close(m.arrays, oracle.port_deposit_moments(p, grid, 0.003, pressure),
                         what=f"fast {order} pressure={pressure}")


def test_fast_dmma_deposit_domain_error(gpu):
    """A particle outside the domain: DomainError from the FAST kernel too
    (grid.hpp:65-67)."""
    grid = (4, 4, 4, 4.0, 4.0, 4.0)
    p = random_particles(grid, 1000, 5)
    p[0][777] = 4.0
    g = Grid.make(*grid)
    st = DeviceStore(g, [1000], "fast")
    st.upload_field(gem.gem_field(g))
    st.upload(0, p)
    st.moments_zero(False)
    st.deposit(0, 1.0)
    with pytest.raises(DomainError, match="outside domain"):
        st.sync()
    st.close()
