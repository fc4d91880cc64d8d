"""The product's native GEM generator (csrc/b2m_gem.cpp) against the
reference's init_gem (init.cpp:62-102): bit-identical particles and field.
Host code only -- runs on CPU."""
import pytest

import oracle
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.mover import Grid
from tests._util import assert_bitwise, digest


@pytest.mark.parametrize("case", ["c1_init", "desk_init"])
def test_gem_species_match_reference_digests(built, golden, case):
    gd = golden[case]
    grid = Grid.make(*gd["grid"])
    batches = gem.init_gem_species(grid, gd["ppc"], gd["seed"])
    assert [b.count() for b in batches] == gd["counts"]
    assert [digest(b.span()) for b in batches] == gd["species_sha"]
    f = gem.gem_field(grid)
    assert digest([f.E.ravel(), f.B.ravel()]) == gd["field_sha"]


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library unavailable")
@pytest.mark.parametrize("dims,ppc,seed", [((10, 12, 6, 5.0, 6.0, 3.0), 3, 7),
                                           ((6, 8, 4, 2.4, 3.2, 1.6), 1, 99),
                                           ((5, 10, 3, 2.0, 4.0, 1.2), 5, 12345)])
def test_gem_matches_reference_odd_shapes(built, dims, ppc, seed):
    """Odd ppc and odd cell counts exercise the counter jump-ahead for odd
    particle indices (cached Box-Muller spare across particles)."""
    grid = Grid.make(*dims)
    ours = gem.init_gem_species(grid, ppc, seed, threads=7)
    parts, E, B = oracle.ref_init_gem(dims, ppc, seed)
    for s in range(4):
        assert_bitwise(ours[s].span(), parts[s], f"species {s}")
    f = gem.gem_field(grid)
    assert_bitwise([f.E.ravel(), f.B.ravel()], [E, B], "field")


def test_gem_species_table(built):
    grid = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
    qom, qpp = gem.gem_species_params(grid, 216)
    assert list(qom) == [-25.0, 1.0, -25.0, 1.0]
    v = grid.cell_volume()
    assert qpp[0] == -(0.2 * v / 216) and qpp[2] == -(v / 216)
    # the reference GEM at 216 ppc holds 61,046,784 particles
    assert sum(gem.gem_counts(grid, 216)) == 61046784


def test_gem_like_field_matches_port(built):
    dims = (8, 8, 8, 6.4, 6.4, 6.4)
    f = gem.gem_like_field(Grid.make(*dims))
    E, B = oracle.port_gem_like_field(dims)
    assert_bitwise([f.E.ravel(), f.B.ravel()], [E, B], "gem_like_field")
