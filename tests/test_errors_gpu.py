"""Error paths of the C ABI on a GPU, in the reference's taxonomy
(errors.hpp:12-44): capacity problems are AllocError at the call that
exceeds them (DeviceArena::configure, device_arena.cpp:20-55; the batch's
fixed capacity, particle_batch.hpp:43-46), bad setups ConfigError
(runtime.cpp:22-37 decompose, kernels.hpp:30-39 MoverParams), and nothing is
silently truncated."""
import pytest
import torch

from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.errors import AllocError, ConfigError, MinipicError
from paper_1904_03684_b200.mover import FieldMesh, Grid, MomentMesh, MoverParams
from paper_1904_03684_b200.partition import DeviceMigration
from tests._util import random_particles

pytestmark = pytest.mark.gpu

G = Grid.make(8, 8, 8, 6.4, 6.4, 6.4)


def test_context_capacity_too_large_is_alloc_error_at_creation(gpu):
    with pytest.raises(AllocError):
        DeviceStore(G, [1 << 40], "fast")   # 48 TB of particles


def test_upload_beyond_capacity_is_alloc_error(gpu):
    st = DeviceStore(G, [100], "fast")
    p = random_particles(G.as_tuple(), 101, 1)
    with pytest.raises(AllocError, match="capacity"):
        st.upload(0, p)
    st.close()


def test_move_before_field_is_config_error(gpu):
    st = DeviceStore(G, [10], "strict")
    st.upload(0, random_particles(G.as_tuple(), 10, 2))
    with pytest.raises(ConfigError, match="no field"):
        st.move(0, MoverParams.make(0.1, 1.0, 3))
    st.close()


def test_bad_pc_iterations_is_config_error(gpu):
    st = DeviceStore(G, [10], "fast")
    st.upload_field(gem.gem_field(G))
    st.upload(0, random_particles(G.as_tuple(), 10, 3))
    mp = MoverParams(0.1, 1.0, 0, 0.05)   # pc_iterations = 0
    with pytest.raises(ConfigError, match="pc_iterations"):
        st.move(0, mp)
    st.close()


@pytest.mark.parametrize("world,msg", [(3, "does not divide"), (8, "at least 2")])
def test_slab_config_validates_like_decompose(gpu, world, msg):
    st = DeviceStore(G, [10], "fast")
    with pytest.raises(ConfigError, match=msg):
        DeviceMigration(st, 0, world)
    st.close()


def test_inbox_beyond_capacity_is_alloc_error(gpu):
    st = DeviceStore(G, [16], "fast")
    st.upload_field(gem.gem_field(G))
    st.upload(0, random_particles(G.as_tuple(), 10, 4))
    mig = DeviceMigration(st, 0, 2)
    recs = torch.zeros((7, 6), dtype=torch.float64, device="cuda")
    recs[:, 0] = 1.0
    with pytest.raises(AllocError):
        mig.inbox_append(0, recs)   # 10 + 7 > 16
    st.close()


def test_moments_without_mesh_is_rejected(gpu):
    st = DeviceStore(G, [10], "fast")
    st.upload(0, random_particles(G.as_tuple(), 10, 5))
    with pytest.raises(ConfigError, match="moments_zero"):
        st.deposit(0, 1.0)
    with pytest.raises((ValueError, MinipicError)):   # B2M_INVALID_ARGUMENT
        st.moments_download(MomentMesh.make(G))
    st.close()


def test_field_node_count_mismatch_is_config_error(gpu):
    st = DeviceStore(G, [10], "fast")
    wrong = FieldMesh(Grid.make(4, 4, 4, 6.4, 6.4, 6.4))
    with pytest.raises(ConfigError, match="node count"):
        st.upload_field(wrong)
    st.close()
