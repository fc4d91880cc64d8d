"""GPU parity of the field-phase stand-in (field_phase_stub,
kernels.cpp:185-215): bit-identical to the pinned oracle.  Mirrors
test_kernels.cpp:317-363."""
import numpy as np
import pytest

import oracle
from paper_1904_03684_b200 import FieldMesh, Grid, field_phase_stub
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import MoverParams
from tests._util import assert_bitwise, random_field, random_particles, uniform_field

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("passes", [0, 1, 2, 7])
def test_stub_bitwise_vs_oracle(gpu, passes):
    g = Grid.make(9, 6, 5, 1.0, 2.0, 3.0)
    E, B = random_field(g.as_tuple(), 5)
    out = field_phase_stub(FieldMesh(g, E, B), g, passes)
    Ew, Bw = oracle.port_field_phase_stub(E, B, g.as_tuple(), passes)
    assert_bitwise(out.E.ravel(), Ew, "E")
    assert_bitwise(out.B.ravel(), Bw, "B")


def test_uniform_mesh_is_a_bitwise_fixed_point(gpu):
    """test_kernels.cpp:317-323"""
    g = Grid.make(6, 6, 6, 2.0, 2.0, 2.0)
    E, B = uniform_field(g.as_tuple(), [1.0, -2.0, 0.5], [0.25, 0.5, -1.0])
    out = field_phase_stub(FieldMesh(g, E, B), g, 10)
    assert_bitwise(out.E.ravel(), E, "E")
    assert_bitwise(out.B.ravel(), B, "B")


def test_smoothing_preserves_sum_contracts_extremes_mirrors_seam(gpu):
    """test_kernels.cpp:325-363"""
    g = Grid.make(8, 8, 8, 1.0, 1.0, 1.0)
    m = FieldMesh.make(g)
    r = np.random.default_rng(41)
    G = m.E.reshape(9, 9, 9, 3)
    G[:8, :8, :8, 0] = r.standard_normal((8, 8, 8))
    m.mirror_seams()
    out = field_phase_stub(m, g, 5)
    u0 = m.E.reshape(9, 9, 9, 3)[:8, :8, :8, 0]
    u1 = out.E.reshape(9, 9, 9, 3)[:8, :8, :8, 0]
    assert u1.sum() == pytest.approx(u0.sum(), rel=1e-12, abs=1e-12)
    assert u1.max() <= u0.max() + 1e-12 and u1.min() >= u0.min() - 1e-12
    assert u1.max() - u1.min() < u0.max() - u0.min()
    assert out.E[out.index(8, 3, 3), 0] == out.E[out.index(0, 3, 3), 0]


def test_device_field_stub_then_move(gpu):
    """Engine-level: the stubbed device field is the next mover field
    (runtime.cpp:222): smoothing on the device then moving (FAST tables
    rebuilt) == moving with the oracle-smoothed field (STRICT bitwise)."""
    g = Grid.make(8, 8, 8, 6.4, 6.4, 6.4)
    grid = g.as_tuple()
    field = gem.gem_like_field(g)
    p0 = random_particles(grid, 20000, 3)
    Ew, Bw = oracle.port_field_phase_stub(field.E.ravel(), field.B.ravel(), grid, 3)
    for mode in ("strict", "fast"):
        st = DeviceStore(g, [len(p0[0])], mode)
        st.upload_field(field)
        st.field_stub(3)
        got_f = FieldMesh.make(g)
        st.download_field(got_f)
        assert_bitwise(got_f.E.ravel(), Ew, "device E")
        st.upload(0, p0)
        st.move(0, MoverParams.make(0.1, -25.0, 3))
        out = [np.empty_like(a) for a in p0]
        st.download(0, out)
        st.sync()
        want = [a.copy() for a in p0]
        assert oracle.port_move_batch(want, Ew, Bw, grid, 0.1, -25.0, 3) == -1
        if mode == "strict":
            for a, w in zip(out, want):
                assert_bitwise(a, w, "move after stub")
        else:
            for a, w in zip(out, want):
                np.testing.assert_allclose(a, w, rtol=1e-12, atol=1e-12)
        st.close()


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
def test_stub_against_the_reference_library_itself(gpu):
    g = Grid.make(10, 7, 6, 1.0, 2.0, 3.0)
    E, B = random_field(g.as_tuple(), 13)
    out = field_phase_stub(FieldMesh(g, E, B), g, 4)
    Ew, Bw = oracle.ref_field_phase_stub(E, B, g.as_tuple(), 4)
    assert_bitwise(out.E.ravel(), Ew, "E")
    assert_bitwise(out.B.ravel(), Bw, "B")


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
def test_c2_default_passes_vs_reference(gpu):
    """The C2 mesh (64x64x32, 139,425 nodes) with the reference's default 100
    passes (sim_config field_passes), bit-identical to the unmodified
    reference field_phase_stub."""
    g = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
    E, B = random_field(g.as_tuple(), 21)
    out = field_phase_stub(FieldMesh(g, E, B), g, 100)
    Ew, Bw = oracle.ref_field_phase_stub(E, B, g.as_tuple(), 100)
    assert_bitwise(out.E.ravel(), Ew, "E")
    assert_bitwise(out.B.ravel(), Bw, "B")
