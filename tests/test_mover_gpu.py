"""Parity of the sm_100a mover (through the C ABI) with the oracle and the
reference's golden vectors.  Needs a B200: ``pytest -m gpu``.

STRICT mode must be bit-identical to the reference; FAST mode must meet the
north-star contract (1e-12, count and cell indices exact; tests/_util.py)."""
import numpy as np
import pytest

import oracle
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import B200Engine, DeviceStore
from paper_1904_03684_b200.errors import EngineFault, NumericalFault
from paper_1904_03684_b200.mover import FieldMesh, Grid, MoverParams, move_batch
from tests._util import (assert_bitwise, assert_within_contract, cells_of, cramer_vbar, digest,
                         from_hex, random_field, random_particles, sort_keys_of, uniform_field)

pytestmark = pytest.mark.gpu

MODES = ["strict", "fast"]


def port_move(p6, E, B, grid, dt, qom, pc):
    out = [np.ascontiguousarray(a, dtype=np.float64).copy() for a in p6]
    assert oracle.port_move_batch(out, E, B, grid, dt, qom, pc) == -1
    return out


def gpu_move(p6, E, B, grid, dt, qom, pc, mode):
    out = [np.ascontiguousarray(a, dtype=np.float64).copy() for a in p6]
    move_batch(out, (E, B), Grid.make(*grid), MoverParams.make(dt, qom, pc), mode=mode)
    return out


def check(got, want, grid, mode, what=""):
    if mode == "strict":
        assert_bitwise(got, want, what)
    else:
        assert_within_contract(got, want, grid, what=what)
        np.testing.assert_array_equal(cells_of(got, grid), cells_of(want, grid))


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("case,field", [("c1_move", "like"), ("c1_move_gemfield_pc5", "gem"),
                                        ("c1_move_pc1", "like"), ("desk_move", "like+gemB")])
def test_golden_cases(gpu, golden, mode, case, field):
    gd = golden[case]
    grid = tuple(gd["grid"])
    init = golden["desk_init" if case.startswith("desk") else "c1_init"]
    g = Grid.make(*grid)
    batches = gem.init_gem_species(g, init["ppc"], init["seed"])
    if field == "gem":
        f = gem.gem_field(g)
    elif field == "like":
        f = gem.gem_like_field(g)
    else:
        f = gem.gem_bench_field(g)
    E, B = f.E.ravel(), f.B.ravel()
    assert digest([E, B]) == gd["field_sha"]
    for s, sp in enumerate(gd["species"]):
        p0 = batches[s].span()
        assert digest(p0) == sp["in_sha"]
        got = gpu_move(p0, E, B, grid, gd["dt"], sp["qom"], gd["pc"], mode)
        if mode == "strict":
            assert digest(got) == sp["out_sha"], f"species {s} not bit-identical to the reference"
        else:
            want = port_move(p0, E, B, grid, gd["dt"], sp["qom"], gd["pc"])
            assert digest(want) == sp["out_sha"]
            check(got, want, grid, mode, f"species {s}")


@pytest.mark.parametrize("mode", MODES)
def test_spec_kat(gpu, golden, mode):
    k = golden["kat"]
    grid = tuple(k["grid"])
    E, B = uniform_field(grid, [0, 0, 0], [0, 0, 1])
    p0 = [np.array([v]) for v in list(from_hex(k["x0"])) + list(from_hex(k["v0"]))]
    got = gpu_move(p0, E, B, grid, k["dt"], k["qom"], k["pc"], mode)
    want = [np.array([v]) for v in list(from_hex(k["x1"])) + list(from_hex(k["v1"]))]
    check(got, want, grid, mode, "KAT")


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("seed,qom,pc", [(1, -25.0, 3), (2, 1.0, 3), (3, -25.0, 5), (4, 1.0, 1),
                                         (5, -25.0, 2), (6, 1.0, 4)])
def test_random_fields_vs_oracle(gpu, mode, seed, qom, pc):
    grid = (6, 5, 4, 2.4, 2.0, 1.6)
    E, B = random_field(grid, seed, scale=0.7)
    p0 = random_particles(grid, 50000, seed)
    check(gpu_move(p0, E, B, grid, 0.1, qom, pc, mode), port_move(p0, E, B, grid, 0.1, qom, pc),
          grid, mode, "random fields")


@pytest.mark.parametrize("mode", MODES)
def test_edge_positions_vs_oracle(gpu, mode):
    grid = (4, 4, 4, 4.0, 4.0, 4.0)
    E, B = random_field(grid, 9, scale=0.5)
    L = 4.0
    edge = [0.0, -0.0, 1.0, 2.0, 3.0, np.nextafter(L, 0.0), np.nextafter(1.0, 0.0),
            np.nextafter(3.0, 4.0), 5e-324, 1e-17]
    xs = np.array(np.meshgrid(edge, edge, edge)).reshape(3, -1)
    n = xs.shape[1]
    r = np.random.default_rng(5)
    for vs in (0.3, 1e-18, 4.0):  # tiny velocities keep positions on the edges
        p0 = [xs[0].copy(), xs[1].copy(), xs[2].copy()] + [vs * r.standard_normal(n) for _ in range(3)]
        for qom in (-25.0, 1.0):
            check(gpu_move(p0, E, B, grid, 0.1, qom, 3, mode),
                  port_move(p0, E, B, grid, 0.1, qom, 3), grid, mode, f"edges vs={vs}")


@pytest.mark.parametrize("mode", MODES)
def test_seam_crossings_wrap_exactly(gpu, mode):
    """Particles crossing the periodic seam in the final update, with exactly
    representable x0 + v*dt (dt = 1/8, offsets in units of ulp(L)): every
    mode must then produce the reference's wrap_len bit for bit, including
    the rounding fix-ups of grid.hpp:45-50."""
    grid = (8, 8, 8, 6.4, 6.4, 6.4)
    E, B = uniform_field(grid, [0, 0, 0], [0, 0, 0])
    L = 6.4
    ulp = 2.0 ** -50  # spacing of doubles in [4, 8)
    r = np.random.default_rng(11)
    n = 8192
    k = r.integers(0, 64, n).astype(np.float64)
    m = r.integers(-64, 64, n).astype(np.float64)
    top = np.nextafter(L, 0.0) - k * ulp          # just below L
    bot = k * 2.0 ** -60                           # just above 0
    x = np.where(np.arange(n) % 2 == 0, top, bot)
    v = m * ulp * 8.0                              # v*dt = m*ulp exactly
    v = np.where(np.arange(n) % 2 == 0, np.abs(v), -np.abs(v) * 2.0 ** -10)
    p0 = [x.copy(), x.copy(), x.copy(), v.copy(), v.copy(), v.copy()]
    got = gpu_move(p0, E, B, grid, 0.125, 1.0, 3, mode)
    want = port_move(p0, E, B, grid, 0.125, 1.0, 3)
    assert_bitwise(got, want, "seam")
    for a in range(3):
        assert np.all((got[a] >= 0) & (got[a] < L))


@pytest.mark.parametrize("mode", MODES)
def test_nan_fault_semantics(gpu, golden, mode):
    gd = golden["nan_fault"]
    g = Grid.make(4, 4, 4, 4.0, 4.0, 4.0)
    E, B = uniform_field(g.as_tuple(), [0, 0, 0], [0, 0, 1])
    p = [np.array([1.0, 2.0, 3.0]), np.array([1.0, 2.0, 3.0]), np.array([1.0, 2.0, 3.0]),
         np.array([0.1, np.nan, 0.1]), np.zeros(3), np.zeros(3)]
    with pytest.raises(NumericalFault, match="particle index 1$") as ei:
        move_batch(p, (E, B), g, MoverParams.make(0.1, 1.0, 2), mode=mode)
    assert ei.value.index == 1
    for a in range(6):
        want = from_hex(gd["after"][a])
        if mode == "strict":
            np.testing.assert_array_equal(np.nan_to_num(p[a]), np.nan_to_num(want))
        else:
            np.testing.assert_allclose(np.nan_to_num(p[a]), np.nan_to_num(want), rtol=1e-12, atol=1e-14)
        # the faulting particle and every later one are untouched
        assert p[a][2] == [3.0, 3.0, 3.0, 0.1, 0.0, 0.0][a]
        if a != 3:
            assert p[a][1] == [2.0, 2.0, 2.0, 0.0, 0.0, 0.0][a]
    assert np.isnan(p[3][1])


@pytest.mark.parametrize("mode", MODES)
def test_out_of_domain_input_faults(gpu, mode):
    g = Grid.make(4, 4, 4, 4.0, 4.0, 4.0)
    E, B = uniform_field(g.as_tuple(), [0, 0, 0], [0, 0, 1])
    p = [np.array([1.0, 4.0, 2.0, -0.5]), np.ones(4), np.ones(4), np.zeros(4), np.zeros(4),
         np.zeros(4)]
    with pytest.raises(NumericalFault) as ei:
        move_batch(p, (E, B), g, MoverParams.make(0.1, 1.0, 3), mode=mode)
    assert ei.value.index == 1
    assert p[0][0] == 1.0 and p[0][1] == 4.0 and p[0][3] == -0.5


@pytest.mark.parametrize("mode", MODES)
def test_empty_batch_is_noop(gpu, mode):
    g = Grid.make(4, 4, 4, 4.0, 4.0, 4.0)
    E, B = uniform_field(g.as_tuple(), [0, 0, 0], [0, 0, 1])
    p = [np.zeros(0) for _ in range(6)]
    move_batch(p, (E, B), g, MoverParams.make(0.1, 1.0, 3), mode=mode)


@pytest.mark.parametrize("mode", MODES)
def test_uniform_field_pc_fixed_point(gpu, mode):
    """SPEC.md: with uniform fields the corrector is a fixed point, so pc 1
    and pc 3 agree -- up to the rounding of the gather's partition of unity,
    which the reference itself shows (it is NOT bitwise pc-invariant; the
    SPEC's "bitwise" claim does not hold for the reference either)."""
    grid = (8, 8, 8, 4.0, 4.0, 4.0)
    E, B = uniform_field(grid, [0.3, -0.2, 0.1], [0.5, 0.25, -0.75])
    p0 = random_particles(grid, 20000, 3)
    a = gpu_move(p0, E, B, grid, 0.1, -25.0, 1, mode)
    b = gpu_move(p0, E, B, grid, 0.1, -25.0, 3, mode)
    assert_within_contract(a, b, grid, tol=1e-13)
    check(a, port_move(p0, E, B, grid, 0.1, -25.0, 1), grid, mode, "pc1")
    check(b, port_move(p0, E, B, grid, 0.1, -25.0, 3), grid, mode, "pc3")


@pytest.mark.parametrize("mode", MODES)
def test_independent_cramer_oracle_uniform_fields(gpu, mode):
    """The device mover against an independent solve (test_kernels.cpp:183-214,
    test_acceptance.cpp:205-241): on uniform fields the implicit velocity is
    the Cramer-rule solution of (I - beta[x B]) vbar = vn + beta E, so
    x1 = wrap(x0 + vbar dt) and v1 = 2 vbar - v0 to 1e-14 absolute, the
    reference's own bar, for qom in {1, -25}."""
    grid = (8, 8, 8, 4.0, 4.0, 4.0)
    rng = np.random.default_rng(23)
    L = np.array(grid[3:])
    for trial, qom in enumerate([1.0, -25.0, 1.0]):
        E0, B0 = rng.standard_normal(3), rng.standard_normal(3)
        E, B = uniform_field(grid, E0, B0)
        p0 = random_particles(grid, 10000, 100 + trial)
        dt = 0.1
        got = gpu_move(p0, E, B, grid, dt, qom, 3, mode)
        v0, x0 = np.stack(p0[3:], axis=1), np.stack(p0[:3], axis=1)
        vbar = cramer_vbar(v0, np.broadcast_to(E0, v0.shape), np.broadcast_to(B0, v0.shape),
                           qom * dt * 0.5)
        x1 = x0 + vbar * dt
        x1 = x1 - L * np.floor(x1 / L)
        dx = np.abs(np.stack(got[:3], axis=1) - x1)
        assert np.max(np.minimum(dx, L - dx)) <= 1e-14, (mode, qom)
        assert np.max(np.abs(np.stack(got[3:], axis=1) - (2 * vbar - v0))) <= 1e-14, (mode, qom)


@pytest.mark.parametrize("mode", MODES)
def test_gyration_and_exb_drift(gpu, mode):
    """The reference's physics checks (test_kernels.cpp:365-403) through the
    device mover: in a uniform B the speed is kept to 1e-13 over 100 steps;
    in crossed E and B a particle from rest drifts at E/B to 1 % over one
    gyration period."""
    grid = (4, 4, 4, 8.0, 8.0, 8.0)
    N = 32
    dt = 2.0 * np.tan(np.pi / N)
    E, B = uniform_field(grid, [0, 0, 0], [0, 0, 1])
    p = [np.array([4.0]), np.array([4.0]), np.array([4.0]), np.array([0.2]), np.array([0.0]),
         np.array([0.1])]
    s0 = np.hypot(0.2, 0.1)
    for _ in range(100):
        p = gpu_move(p, E, B, grid, dt, 1.0, 3, mode)
        assert abs(np.sqrt(p[3][0] ** 2 + p[4][0] ** 2 + p[5][0] ** 2) - s0) <= 1e-13 * s0
    e, bz = 0.02, 1.0
    E, B = uniform_field(grid, [0, e, 0], [0, 0, bz])
    p = [np.array([4.0]), np.array([4.0]), np.array([4.0]), np.zeros(1), np.zeros(1), np.zeros(1)]
    xu, xp = 4.0, 4.0
    for _ in range(N):
        p = gpu_move(p, E, B, grid, dt, 1.0, 3, mode)
        d = p[0][0] - xp
        d = d + 8.0 if d < -4.0 else (d - 8.0 if d > 4.0 else d)
        xu += d
        xp = p[0][0]
    assert abs((xu - 4.0) / (N * dt) - e / bz) <= 0.01 * e / bz


@pytest.mark.parametrize("path", ["counting", "radix_fallback"])
@pytest.mark.parametrize("mode", MODES)
def test_device_store_sort_preserves_multiset(gpu, mode, path, monkeypatch):
    """Both cell sorts: the counting sort into the ping-pong set, and the
    low-memory radix sort + gather used when no second set fits."""
    if path == "radix_fallback":
        monkeypatch.setenv("B2M_SORT_FALLBACK", "1")
    g = Grid.make(16, 16, 8, 6.4, 6.4, 3.2)
    grid = g.as_tuple()
    p0 = random_particles(grid, 100000, 21)
    f = FieldMesh(g, *random_field(grid, 2, 0.3))
    st = DeviceStore(g, [len(p0[0])], mode)
    st.upload_field(f)
    st.upload(0, p0)
    st.sort(0)
    srt = [np.empty_like(a) for a in p0]
    assert st.download(0, srt) == len(p0[0])
    st.sync()
    np.testing.assert_array_equal(oracle.multiset(srt), oracle.multiset(p0))
    keys = sort_keys_of(srt, grid)
    assert np.all(np.diff(keys) >= 0)
    # moving the sorted batch == moving those particles with the oracle
    st.move(0, MoverParams.make(0.1, -25.0, 3))
    out = [np.empty_like(a) for a in p0]
    st.download(0, out)
    st.sync()
    want = port_move(srt, f.E.ravel(), f.B.ravel(), grid, 0.1, -25.0, 3)
    check(out, want, grid, mode, "sorted move")


@pytest.mark.parametrize("mode", MODES)
def test_engine_matches_oracle_over_steps(gpu, mode):
    """test_offload.cpp:435-462: 4 species x 5000 particles, gem_like_field,
    3 steps through the engine == 3 oracle steps."""
    g = Grid.make(8, 8, 8, 6.4, 6.4, 6.4)
    grid = g.as_tuple()
    f = gem.gem_like_field(g)
    E, B = f.E.ravel(), f.B.ravel()
    from paper_1904_03684_b200.mover import ParticleBatch
    batches, refs, mps = [], [], []
    for s in range(4):
        qom = 1.0 if s % 2 else -25.0
        p0 = random_particles(grid, 5000, 7 + s, vscale=0.1)
        b = ParticleBatch(s, qom, 0.01, 5000, pinned=True)
        b.assign(p0)
        batches.append(b)
        refs.append([a.copy() for a in p0])
        mps.append(MoverParams.make(0.05, qom, 3))
    for schedule in ("pipeline", "prefetch", "sync"):
        eng = B200Engine(g, mode=mode, schedule=schedule, chunk=1536)
        bs = []
        for s in range(4):
            b = ParticleBatch(s, batches[s].qom, 0.01, 5000, pinned=(schedule == "pipeline"))
            b.assign(refs[s])
            bs.append(b)
        eng.prime(f, bs)
        for step in range(3):
            eng.run_mover(f, bs, mps)
        for s in range(4):
            want = [a.copy() for a in refs[s]]
            for step in range(3):
                assert oracle.port_move_batch(want, E, B, grid, 0.05, mps[s].qom, 3) == -1
            if mode == "strict":
                assert_bitwise(bs[s].span(), want, f"{schedule} species {s}")
            else:
                assert_within_contract(bs[s].span(), want, grid, tol=1e-11, what=f"{schedule} s{s}")


@pytest.mark.parametrize("mode", MODES)
def test_engine_fault_poisons(gpu, mode):
    """test_offload.cpp:464-481: a kernel fault surfaces as EngineFault naming
    the particle; the engine stays poisoned."""
    g = Grid.make(8, 8, 8, 6.4, 6.4, 6.4)
    f = gem.gem_like_field(g)
    from paper_1904_03684_b200.mover import ParticleBatch
    bs = []
    for s in range(2):
        b = ParticleBatch(s, -25.0 if s == 0 else 1.0, 0.01, 10)
        b.assign(random_particles(g.as_tuple(), 10, s, 0.1))
        bs.append(b)
    bs[1].arrays[3][3] = np.nan
    eng = B200Engine(g, mode=mode, schedule="sync")
    eng.prime(f, bs)
    mps = [MoverParams.make(0.05, b.qom, 3) for b in bs]
    with pytest.raises(EngineFault, match="particle"):
        eng.run_mover(f, bs, mps)
    with pytest.raises(EngineFault):
        eng.run_mover(f, bs, mps)


def test_full_c2_sampled_parity(gpu):
    """BASELINE config 2 at full size (61,046,784 particles): FAST move of
    the whole GEM state on the GPU; a 200k-particle random sample per species
    is checked against the oracle (the mover is per-particle independent,
    kernels.hpp:46-48), plus size-independent properties on all particles."""
    g = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
    grid = g.as_tuple()
    batches = gem.init_gem_species(g, 216, pinned=True)
    assert sum(b.count() for b in batches) == 61046784
    f = gem.gem_bench_field(g)
    E, B = f.E.ravel(), f.B.ravel()
    st = DeviceStore(g, [b.count() for b in batches], "fast")
    st.upload_field(f)
    for s, b in enumerate(batches):
        st.upload(s, b.span())
    mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
    st.move_all(mps)
    outs = []
    for s, b in enumerate(batches):
        out = [np.empty(b.count()) for _ in range(6)]
        st.download(s, out)
        outs.append(out)
    st.sync()
    r = np.random.default_rng(0)
    for s, b in enumerate(batches):
        out = outs[s]
        for a, L in zip(range(3), grid[3:]):
            assert np.all((out[a] >= 0) & (out[a] < L))
        assert all(np.all(np.isfinite(a)) for a in out)
        idx = np.sort(r.choice(b.count(), size=min(200000, b.count()), replace=False))
        p0 = [a[idx].copy() for a in b.span()]
        want = port_move(p0, E, B, grid, 0.1, b.qom, 3)
        got = [a[idx] for a in out]
        assert_within_contract(got, want, grid, what=f"C2 species {s}")
        np.testing.assert_array_equal(cells_of(got, grid), cells_of(want, grid))


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("n", [1, 31, 127, 128, 129, 4097, 100003])
def test_ragged_sizes(gpu, mode, n):
    """Partial tiles (the TMA box clips the tail) and single particles."""
    grid = (8, 8, 8, 6.4, 6.4, 6.4)
    E, B = random_field(grid, 4, 0.3)
    p0 = random_particles(grid, n, 100 + n)
    check(gpu_move(p0, E, B, grid, 0.1, -25.0, 3, mode), port_move(p0, E, B, grid, 0.1, -25.0, 3),
          grid, mode, f"n={n}")


def test_full_c2_strict_sampled_bitwise(gpu):
    """BASELINE config 2 at full size in STRICT mode: the whole GEM state
    moved on the GPU, with the stock GEM field plus the gem_like E (nonzero
    E); a 100k-particle sample per species is bit-identical to the
    oracle."""
    g = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
    grid = g.as_tuple()
    batches = gem.init_gem_species(g, 216, pinned=True)
    f = gem.gem_bench_field(g)
    E, B = f.E.ravel(), f.B.ravel()
    st = DeviceStore(g, [b.count() for b in batches], "strict")
    st.upload_field(f)
    for s, b in enumerate(batches):
        st.upload(s, b.span())
    st.move_all([MoverParams.make(0.1, b.qom, 3) for b in batches])
    r = np.random.default_rng(1)
    for s, b in enumerate(batches):
        out = [np.empty(b.count()) for _ in range(6)]
        st.download(s, out)
        st.sync()
        idx = np.sort(r.choice(b.count(), size=min(100000, b.count()), replace=False))
        want = port_move([a[idx].copy() for a in b.span()], E, B, grid, 0.1, b.qom, 3)
        assert_bitwise([a[idx] for a in out], want, f"C2 strict species {s}")


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
def test_full_c2_strict_every_particle_vs_reference(gpu):
    """Every one of the 61,046,784 C2 particles, two STRICT steps on the GPU
    (nonzero E), bit-identical to the UNMODIFIED reference pic::move_batch
    run on the host's cores over the same state (oracle/_ref)."""
    import os
    g = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
    grid = g.as_tuple()
    batches = gem.init_gem_species(g, 216, pinned=True)
    f = gem.gem_bench_field(g)
    E, B = f.E.ravel(), f.B.ravel()
    st = DeviceStore(g, [b.count() for b in batches], "strict")
    st.upload_field(f)
    for s, b in enumerate(batches):
        st.upload(s, b.span())
    mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
    st.move_all(mps)
    st.move_all(mps)
    threads = max(1, min(32, os.cpu_count() or 1))
    for s, b in enumerate(batches):
        out = [np.empty(b.count()) for _ in range(6)]
        st.download(s, out)
        st.sync()
        want = [a.copy() for a in b.span()]
        for _ in range(2):
            oracle.ref_move_batch(want, E, B, grid, 0.1, b.qom, 3, threads=threads)
        assert_bitwise(out, want, f"C2 strict species {s}, all particles")


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
def test_full_c2_fast_every_particle_vs_reference(gpu):
    """Every C2 particle, one FAST step, within the 1e-12 contract of the
    UNMODIFIED reference pic::move_batch (oracle/_ref on the host's cores),
    cell indices exact."""
    import os
    g = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
    grid = g.as_tuple()
    batches = gem.init_gem_species(g, 216, pinned=True)
    f = gem.gem_bench_field(g)
    E, B = f.E.ravel(), f.B.ravel()
    st = DeviceStore(g, [b.count() for b in batches], "fast")
    st.upload_field(f)
    for s, b in enumerate(batches):
        st.upload(s, b.span())
    st.move_all([MoverParams.make(0.1, b.qom, 3) for b in batches])
    threads = max(1, min(32, os.cpu_count() or 1))
    for s, b in enumerate(batches):
        out = [np.empty(b.count()) for _ in range(6)]
        st.download(s, out)
        st.sync()
        want = [a.copy() for a in b.span()]
        oracle.ref_move_batch(want, E, B, grid, 0.1, b.qom, 3, threads=threads)
        assert_within_contract(out, want, grid, what=f"C2 fast species {s}, all particles")
        np.testing.assert_array_equal(cells_of(out, grid), cells_of(want, grid))


@pytest.mark.parametrize("mode", MODES)
def test_host_call_context_cache(gpu, mode):
    """b2m_move_batch_host keeps one context per host thread: a fault in one
    call must not leak into the next, and a different grid or a larger batch
    gets a fresh context -- every call still equals the oracle."""
    grid = (8, 8, 8, 6.4, 6.4, 6.4)
    E, B = random_field(grid, 7, 0.3)
    p = random_particles(grid, 1000, 70)
    check(gpu_move(p, E, B, grid, 0.1, 1.0, 3, mode), port_move(p, E, B, grid, 0.1, 1.0, 3),
          grid, mode, "first")
    bad = [a.copy() for a in p]
    bad[3][10] = np.nan
    with pytest.raises(NumericalFault):
        gpu_move(bad, E, B, grid, 0.1, 1.0, 3, mode)
    check(gpu_move(p, E, B, grid, 0.1, 1.0, 3, mode), port_move(p, E, B, grid, 0.1, 1.0, 3),
          grid, mode, "after a fault")
    big = random_particles(grid, 5000, 71)
    check(gpu_move(big, E, B, grid, 0.1, 1.0, 3, mode), port_move(big, E, B, grid, 0.1, 1.0, 3),
          grid, mode, "larger batch")
    g2 = (4, 6, 5, 2.0, 3.0, 2.5)
    E2, B2 = random_field(g2, 8, 0.3)
    p2 = random_particles(g2, 700, 72)
    check(gpu_move(p2, E2, B2, g2, 0.1, 1.0, 3, mode), port_move(p2, E2, B2, g2, 0.1, 1.0, 3),
          g2, mode, "other grid")


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
@pytest.mark.parametrize("mode", MODES)
def test_against_the_reference_library_itself(gpu, mode):
    """Not only the C restatement: the UNMODIFIED reference pic::move_batch
    (oracle/_ref/libminipic_ref.so, built from the reference sources) on the
    same inputs -- STRICT bit-identical, FAST within the contract."""
    grid = (12, 10, 8, 4.8, 3.0, 2.4)
    E, B = random_field(grid, 12, 0.4)
    for qom, pc in ((-25.0, 3), (1.0, 5)):
        p0 = random_particles(grid, 30000, 1200 + pc)
        want = [a.copy() for a in p0]
        oracle.ref_move_batch(want, E, B, grid, 0.1, qom, pc)
        check(gpu_move(p0, E, B, grid, 0.1, qom, pc, mode), want, grid, mode,
              f"vs reference qom={qom} pc={pc}")


def zinvariant_field(grid, seed, scale=0.7):
    """A random field with every node plane k equal to plane 0 (2-D in 3-D)."""
    nx, ny, nz = grid[:3]
    E, B = random_field(grid, seed, scale)
    out = []
    for F in (E, B):
        G = F.reshape(nz + 1, ny + 1, nx + 1, 3).copy()
        G[:] = G[0]
        out.append(np.ascontiguousarray(G.reshape(-1)))
    return out[0], out[1]


@pytest.mark.parametrize("seed,qom,pc", [(11, -25.0, 3), (12, 1.0, 5), (13, -25.0, 1), (14, -25.0, 4)])
def test_zinvariant_kernel_vs_oracle_and_general(gpu, monkeypatch, seed, qom, pc):
    """A z-invariant field runs the column (2-D-in-3-D) FAST kernel: within
    the contract of the oracle, cells exact, and equal to the general 3-D
    FAST kernel (B2M_FAST_3D=1) value for value (the z coefficients it skips
    are exact zeros; only the sign of a zero may differ)."""
    grid = (6, 5, 4, 2.4, 2.0, 1.6)
    E, B = zinvariant_field(grid, seed)
    p0 = random_particles(grid, 50000, seed)
    got = gpu_move(p0, E, B, grid, 0.1, qom, pc, "fast")
    check(got, port_move(p0, E, B, grid, 0.1, qom, pc), grid, "fast", "z-invariant")
    monkeypatch.setenv("B2M_FAST_3D", "1")
    gen = gpu_move(p0, E, B, grid, 0.1, qom, pc, "fast")
    for a, (x, y) in enumerate(zip(got, gen)):
        assert np.array_equal(x, y), f"array {a}: column kernel != general kernel"


def test_zinvariant_kernel_edges_and_faults(gpu):
    """Edge positions (faces, seams, ulps, -0) and a non-finite z velocity
    through the column kernel, against the oracle."""
    grid = (4, 4, 4, 4.0, 4.0, 4.0)
    E, B = zinvariant_field(grid, 21, scale=0.5)
    L = 4.0
    edge = [0.0, -0.0, 1.0, 3.0, np.nextafter(L, 0.0), np.nextafter(1.0, 0.0), 5e-324]
    xs = np.array(np.meshgrid(edge, edge, edge)).reshape(3, -1)
    n = xs.shape[1]
    r = np.random.default_rng(8)
    for vs in (0.3, 1e-18, 4.0):
        p0 = [xs[0].copy(), xs[1].copy(), xs[2].copy()] + [vs * r.standard_normal(n) for _ in range(3)]
        for qom in (-25.0, 1.0):
            check(gpu_move(p0, E, B, grid, 0.1, qom, 3, "fast"),
                  port_move(p0, E, B, grid, 0.1, qom, 3), grid, "fast", f"edges vs={vs}")
    p0 = random_particles(grid, 1000, 4)
    p0[5][617] = np.inf  # w0 = inf: only the z components are non-finite at first
    out = [a.copy() for a in p0]
    with pytest.raises(NumericalFault) as ei:
        move_batch(out, (E, B), Grid.make(*grid), MoverParams.make(0.1, -25.0, 3), mode="fast")
    assert "particle index 617" in str(ei.value)


def test_nearly_zinvariant_field_takes_general_kernel(gpu):
    """One node differing in one plane makes the field 3-D: the general kernel
    must run (the column kernel would ignore the difference)."""
    grid = (6, 5, 4, 2.4, 2.0, 1.6)
    E, B = zinvariant_field(grid, 31)
    nx, ny = grid[:2]
    B[3 * (2 + (nx + 1) * (3 + (ny + 1) * 2)) + 1] += 0.25  # By at node (2, 3, 2)
    p0 = random_particles(grid, 50000, 31)
    check(gpu_move(p0, E, B, grid, 0.1, -25.0, 3, "fast"),
          port_move(p0, E, B, grid, 0.1, -25.0, 3), grid, "fast", "nearly z-invariant")


@pytest.mark.parametrize("path", ["counting", "radix_fallback"])
def test_sort_at_full_capacity_allocates_nothing(gpu, path, monkeypatch):
    """The cell sort's buffers are reserved at context creation
    (device_arena.cpp:20-55: AllocError at creation, never mid-run): sorting
    species filled to exactly their capacity leaves free device memory
    unchanged, and the result is the same multiset in cell order."""
    import torch
    if path == "radix_fallback":
        monkeypatch.setenv("B2M_SORT_FALLBACK", "1")
    g = Grid.make(16, 16, 8, 6.4, 6.4, 3.2)
    grid = g.as_tuple()
    ps = [random_particles(grid, n, 40 + n) for n in (100000, 77777)]
    st = DeviceStore(g, [len(p[0]) for p in ps], "fast")
    st.upload_field(FieldMesh(g, *random_field(grid, 3, 0.3)))
    for s, p in enumerate(ps):
        st.upload(s, p)
    st.sync()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for s in range(len(ps)):
        st.sort(s)
    st.sync()
    assert torch.cuda.mem_get_info()[0] == free0, "the sort allocated device memory mid-run"
    for s, p in enumerate(ps):
        srt = [np.empty_like(a) for a in p]
        assert st.download(s, srt) == len(p[0])
        st.sync()
        np.testing.assert_array_equal(oracle.multiset(srt), oracle.multiset(p))
        assert np.all(np.diff(sort_keys_of(srt, grid)) >= 0)


@pytest.mark.parametrize("seed,qom,pc", [(41, -25.0, 3), (42, 1.0, 5), (43, -25.0, 1)])
def test_strict_column_kernel_bitwise(gpu, monkeypatch, seed, qom, pc):
    """STRICT on a z-invariant field runs the column kernel (4 cached corner
    nodes stand in for 8, the reference's 8 products and sums still formed in
    its order): bit-identical to the oracle and to the general STRICT kernel
    (B2M_FAST_3D=1 disables the z-invariance test), edge positions included;
    one node off the z-invariance takes the general kernel, still bitwise."""
    grid = (6, 5, 4, 2.4, 2.0, 1.6)
    E, B = zinvariant_field(grid, seed)
    p0 = random_particles(grid, 50000, seed)
    L = np.array(grid[3:])
    p0[0][:7] = [0.0, -0.0, np.nextafter(L[0], 0.0), 0.4, np.nextafter(0.4, 0.0), 2.0, 5e-324]
    p0[2][7:14] = [0.0, np.nextafter(L[2], 0.0), 0.4, np.nextafter(0.8, 1.0), 1.2, 0.0, 1.6 / 2]
    want = port_move(p0, E, B, grid, 0.1, qom, pc)
    got = gpu_move(p0, E, B, grid, 0.1, qom, pc, "strict")
    assert_bitwise(got, want, "strict column kernel")
    monkeypatch.setenv("B2M_FAST_3D", "1")
    assert_bitwise(gpu_move(p0, E, B, grid, 0.1, qom, pc, "strict"), want, "strict general")
    monkeypatch.delenv("B2M_FAST_3D")
    nx, ny = grid[:2]
    E2 = E.copy()
    E2[3 * (1 + (nx + 1) * (2 + (ny + 1) * 3)) + 2] += 0.125  # Ez at node (1, 2, 3)
    assert_bitwise(gpu_move(p0, E2, B, grid, 0.1, qom, pc, "strict"),
                   port_move(p0, E2, B, grid, 0.1, qom, pc), "strict nearly z-invariant")
