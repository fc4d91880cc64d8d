"""Pin the oracle (CPU, no GPU): the plain-C restatement in oracle/ must
reproduce the reference's golden vectors bit for bit, and agree bitwise with
the unmodified reference library on fresh inputs when it is available.

Mirrors the reference's own mover tests: test_kernels.cpp:95-230 / :365-403,
test_core.cpp:18-69, test_acceptance.cpp:205-241, SPEC.md KATs.
"""
import numpy as np
import pytest

import oracle
from tests._util import (assert_bitwise, cramer_vbar, digest, from_hex, random_field,
                         random_particles, uniform_field)

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="reference library unavailable")


def _port_gem(gd):
    grid = tuple(gd["grid"])
    return grid, oracle.port_gem_species(grid, gd["ppc"], gd["seed"])


@pytest.mark.parametrize("case", ["c1_init", "desk_init"])
def test_port_gem_init_matches_reference_digests(golden, case):
    gd = golden[case]
    grid, parts = _port_gem(gd)
    assert [len(p[0]) for p in parts] == gd["counts"]
    assert [digest(p) for p in parts] == gd["species_sha"]


@pytest.mark.parametrize("case,init,field", [
    ("c1_move", "c1_init", "like"),
    ("c1_move_gemfield_pc5", "c1_init", "gem"),
    ("c1_move_pc1", "c1_init", "like"),
    ("desk_move", "desk_init", "like+gemB"),
])
def test_port_mover_matches_reference_golden(golden, case, init, field):
    gd = golden[case]
    grid, parts = _port_gem(golden[init])
    if field == "gem":
        ref_parts, E, B = oracle.ref_init_gem(grid, golden[init]["ppc"]) if oracle.ref_available() \
            else (None, None, None)
        if E is None:
            pytest.skip("GEM field needs the reference build")
    else:
        E, B = oracle.port_gem_like_field(grid)
        if field == "like+gemB":
            if not oracle.ref_available():
                pytest.skip("GEM B needs the reference build")
            _, _, B = oracle.ref_init_gem(grid, golden[init]["ppc"])
    assert digest([E, B]) == gd["field_sha"]
    for s, sp in enumerate(gd["species"]):
        p = [a.copy() for a in parts[s]]
        assert digest(p) == sp["in_sha"]
        assert oracle.port_move_batch(p, E, B, grid, gd["dt"], sp["qom"], gd["pc"]) == -1
        for a in range(6):
            np.testing.assert_array_equal(p[a][:16], from_hex(sp["out_prefix"][a]))
        assert digest(p) == sp["out_sha"], f"species {s}"


def test_port_wrap_len_golden(golden):
    for c in golden["wrap_len"]:
        v, l, w = float.fromhex(c["v"]), float.fromhex(c["l"]), float.fromhex(c["w"])
        got = oracle.port_wrap_len(v, l)
        assert got.hex() == w.hex(), (v, l, got, w)
        assert 0.0 <= got < l


def test_port_spec_kat(golden):
    k = golden["kat"]
    grid = tuple(k["grid"])
    E, B = uniform_field(grid, [0, 0, 0], [0, 0, 1])
    p = [np.array([v]) for v in list(from_hex(k["x0"])) + list(from_hex(k["v0"]))]
    assert oracle.port_move_batch(p, E, B, grid, k["dt"], k["qom"], k["pc"]) == -1
    assert [a[0].hex() for a in p[:3]] == [float.fromhex(h).hex() for h in k["x1"]]
    assert [a[0].hex() for a in p[3:]] == [float.fromhex(h).hex() for h in k["v1"]]
    # SPEC.md:189,197-198 decimal values
    np.testing.assert_allclose([p[0][0], p[1][0], p[2][0]], [1.698019801980198, 1.4801980198019802, 1.5],
                               rtol=0, atol=1e-15)
    np.testing.assert_allclose([p[3][0], p[4][0], p[5][0]], [0.98019801980198018, -0.19801980198019803, 0],
                               rtol=0, atol=1e-15)


def test_port_nan_fault_names_first_index_and_leaves_tail(golden):
    gd = golden["nan_fault"]
    grid = (4, 4, 4, 4.0, 4.0, 4.0)
    E, B = uniform_field(grid, [0, 0, 0], [0, 0, 1])
    p = [np.array([1.0, 2.0, 3.0]), np.array([1.0, 2.0, 3.0]), np.array([1.0, 2.0, 3.0]),
         np.array([0.1, np.nan, 0.1]), np.zeros(3), np.zeros(3)]
    assert oracle.port_move_batch(p, E, B, grid, 0.1, 1.0, 2) == 1
    assert gd["message"].endswith("particle index 1")
    for a in range(6):
        want = from_hex(gd["after"][a])
        np.testing.assert_array_equal(np.isnan(p[a]), np.isnan(want))
        np.testing.assert_array_equal(np.nan_to_num(p[a]), np.nan_to_num(want))


def test_port_matches_independent_cramer_oracle_uniform_fields():
    """test_kernels.cpp:183-214 / test_acceptance.cpp:205-241: mover vs an
    independent Cramer-rule solve to 1e-14 on uniform fields."""
    grid = (8, 8, 8, 4.0, 4.0, 4.0)
    rng = np.random.default_rng(23)
    for trial, qom in enumerate([1.0, -25.0, 1.0]):
        E0, B0 = rng.standard_normal(3), rng.standard_normal(3)
        E, B = uniform_field(grid, E0, B0)
        p0 = random_particles(grid, 10000, 100 + trial)
        p = [a.copy() for a in p0]
        dt, pc = 0.1, 3
        assert oracle.port_move_batch(p, E, B, grid, dt, qom, pc) == -1
        beta = qom * dt * 0.5
        v0 = np.stack(p0[3:], axis=1)
        x0 = np.stack(p0[:3], axis=1)
        vbar = cramer_vbar(v0, np.broadcast_to(E0, v0.shape), np.broadcast_to(B0, v0.shape), beta)
        L = np.array(grid[3:])
        x1 = x0 + vbar * dt
        x1 = x1 - L * np.floor(x1 / L)
        v1 = 2 * vbar - v0
        got_x = np.stack(p[:3], axis=1)
        dx = np.abs(got_x - x1)
        dx = np.minimum(dx, L - dx)
        assert np.max(dx) <= 1e-14
        assert np.max(np.abs(np.stack(p[3:], axis=1) - v1)) <= 1e-14


def test_port_gyration_and_exb_drift():
    """test_kernels.cpp:365-403 physics checks on the port."""
    grid = (4, 4, 4, 8.0, 8.0, 8.0)
    N = 32
    dt = 2.0 * np.tan(np.pi / N)
    E, B = uniform_field(grid, [0, 0, 0], [0, 0, 1])
    p = [np.array([4.0]), np.array([4.0]), np.array([4.0]), np.array([0.2]), np.array([0.0]),
         np.array([0.1])]
    s0 = np.hypot(0.2, 0.1)
    for _ in range(100):
        assert oracle.port_move_batch(p, E, B, grid, dt, 1.0, 3) == -1
        assert abs(np.sqrt(p[3][0] ** 2 + p[4][0] ** 2 + p[5][0] ** 2) - s0) <= 1e-13 * s0
    e, bz = 0.02, 1.0
    E, B = uniform_field(grid, [0, e, 0], [0, 0, bz])
    p = [np.array([4.0]), np.array([4.0]), np.array([4.0]), np.zeros(1), np.zeros(1), np.zeros(1)]
    xu, xp = 4.0, 4.0
    for _ in range(N):
        assert oracle.port_move_batch(p, E, B, grid, dt, 1.0, 3) == -1
        d = p[0][0] - xp
        if d < -4.0:
            d += 8.0
        if d > 4.0:
            d -= 8.0
        xu += d
        xp = p[0][0]
    assert abs((xu - 4.0) / (N * dt) - e / bz) <= 0.01 * e / bz


@needs_ref
@pytest.mark.parametrize("seed,qom,pc", [(1, -25.0, 3), (2, 1.0, 3), (3, -25.0, 5), (4, 1.0, 1)])
def test_port_vs_reference_random_fields(seed, qom, pc):
    """Spatially varying random fields (a gap the reference's own tests leave,
    SURVEY §4): port and reference bitwise equal."""
    grid = (6, 5, 4, 2.4, 2.0, 1.6)
    E, B = random_field(grid, seed, scale=0.7)
    p0 = random_particles(grid, 20000, seed)
    a = [x.copy() for x in p0]
    b = [x.copy() for x in p0]
    oracle.ref_move_batch(a, E, B, grid, 0.1, qom, pc)
    assert oracle.port_move_batch(b, E, B, grid, 0.1, qom, pc) == -1
    assert_bitwise(b, a, "port vs reference")


@needs_ref
def test_port_vs_reference_edge_positions():
    """Positions on nodes, seams and one ulp below each length."""
    grid = (4, 4, 4, 4.0, 4.0, 4.0)
    E, B = random_field(grid, 9, scale=0.5)
    L = 4.0
    edge = [0.0, -0.0, 1.0, 2.0, 3.0, np.nextafter(L, 0.0), np.nextafter(1.0, 0.0),
            np.nextafter(3.0, 4.0), 5e-324, 1e-17]
    xs = np.array(np.meshgrid(edge, edge, edge)).reshape(3, -1)
    n = xs.shape[1]
    r = np.random.default_rng(5)
    p0 = [xs[0].copy(), xs[1].copy(), xs[2].copy()] + [0.3 * r.standard_normal(n) for _ in range(3)]
    for qom in (-25.0, 1.0):
        a = [x.copy() for x in p0]
        b = [x.copy() for x in p0]
        oracle.ref_move_batch(a, E, B, grid, 0.1, qom, 3)
        assert oracle.port_move_batch(b, E, B, grid, 0.1, qom, 3) == -1
        assert_bitwise(b, a, "edge positions")


@needs_ref
def test_port_vs_reference_grid_cell_of_known_answers(golden):
    gd = golden["grid_cell_of"]
    grid = tuple(gd["grid"])
    for c in gd["cases"]:
        ijk, f = oracle.ref_grid_cell_of(list(from_hex(c["pos"])), grid)
        assert list(ijk) == c["ijk"]
        np.testing.assert_array_equal(f, from_hex(c["f"]))


# ---- deposit_moments (kernels.cpp:147-183) --------------------------------------

def test_port_deposit_matches_reference_golden(golden):
    """The C restatement of deposit_moments reproduces the reference's C1 GEM
    moment meshes (rho, j, pressure) bit for bit."""
    gd = golden["c1_moments"]
    grid, parts = _port_gem(golden["c1_init"])
    qpp = from_hex(gd["qpp"])
    for s, sp in enumerate(gd["species"]):
        m = oracle.port_deposit_moments(parts[s], grid, float(qpp[s]), True)
        assert [digest([a]) for a in m] == sp["sha"], f"species {s}"
        np.testing.assert_array_equal(m[0][:8], from_hex(sp["rho_prefix"]))


def test_port_deposit_single_particle_and_seam():
    """test_kernels.cpp:232-256: q/V/8 on each corner of cell (0,0,0); a
    particle in the last cell folds its upper corners onto node 0."""
    g = (4, 4, 4, 4.0, 4.0, 4.0)
    q = 0.75
    one = lambda x, u: [np.array([x]), np.array([x]), np.array([x]), np.array([u]),
                        np.zeros(1), np.zeros(1)]
    m = oracle.port_deposit_moments(one(0.5, 2.0), g, q)
    expect = q / 1.0 / 8.0
    for c in range(8):
        idx = (c & 1) + 4 * (((c >> 1) & 1) + 4 * ((c >> 2) & 1))
        assert m[0][idx] == expect and m[1][idx] == 2.0 * expect and m[2][idx] == 0.0
    m2 = oracle.port_deposit_moments(one(3.5, 0.0), g, q)
    for (i, j, k) in [(0, 0, 0), (3, 3, 3), (0, 3, 3)]:
        assert m2[0][i + 4 * (j + 4 * k)] == expect
    assert abs(np.cumsum(m2[0])[-1] - q) < 1e-15


@needs_ref
def test_port_deposit_bitwise_vs_reference_random():
    """test_kernels.cpp:258-280 shape: 5000 particles, pressure on."""
    g = (6, 5, 7, 3.0, 2.5, 3.5)
    p = random_particles(g, 5000, 31, vscale=1.0)
    a = oracle.port_deposit_moments(p, g, -0.0125, True)
    b = oracle.ref_deposit_moments(p, g, -0.0125, True)
    for x, y in zip(a, b):
        assert_bitwise(x, y, "moments")


@needs_ref
def test_reference_deposit_domain_error():
    g = (4, 4, 4, 4.0, 4.0, 4.0)
    p = [np.array([1.0, 4.0]), np.array([1.0, 1.0]), np.array([1.0, 1.0]), np.zeros(2),
         np.zeros(2), np.zeros(2)]
    with pytest.raises(oracle.OracleError) as e:
        oracle.ref_deposit_moments(p, g, 1.0)
    assert e.value.status == 2 and "outside domain" in e.value.msg
    with pytest.raises(oracle.OracleError):
        oracle.port_deposit_moments(p, g, 1.0)


# ---- field_phase_stub (kernels.cpp:185-215) ---------------------------------------

def test_port_field_stub_matches_reference_golden(golden):
    grid = tuple(golden["c1_init"]["grid"])
    E, B = oracle.port_gem_like_field(grid)
    Es, Bs = oracle.port_field_phase_stub(E, B, grid, 3)
    assert digest([Es, Bs]) == golden["c1_field_stub3"]["sha"]
    np.testing.assert_array_equal(Es[:12], from_hex(golden["c1_field_stub3"]["E_prefix"]))


@needs_ref
@pytest.mark.parametrize("passes", [0, 1, 4])
def test_port_field_stub_bitwise_vs_reference(passes):
    g = (7, 5, 6, 1.0, 2.0, 3.0)
    E, B = random_field(g, 9)
    a = oracle.port_field_phase_stub(E, B, g, passes)
    b = oracle.ref_field_phase_stub(E, B, g, passes)
    assert_bitwise(a[0], b[0], "E")
    assert_bitwise(a[1], b[1], "B")
