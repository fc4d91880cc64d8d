"""Migration kernels on one B200: several slab ranks as threads of one
process (tests/_fakedist.py), each with its own libb2m context, run SlabWorld
for several cycles.  STRICT mode must reproduce the reference multi-worker
Simulation as a bitwise particle multiset; FAST mode within the 1e-12
contract; every particle must live on the rank that owns its y; CFL and
NaN faults must surface typed on the faulting rank and abort the others."""
import numpy as np
import pytest
import torch

import oracle
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.errors import CflViolation, EngineFault, NumericalFault
from paper_1904_03684_b200.mover import Grid, MoverParams
from paper_1904_03684_b200.partition import DeviceMigration, SlabWorld, owner_of
from tests._fakedist import run_ranks
from tests._util import assert_within_contract

pytestmark = pytest.mark.gpu
GRID_T = (8, 8, 8, 6.4, 6.4, 6.4)


def _rank_fn(mode, cycles, inject=None):
    def fn(rank, dist):
        torch.cuda.set_device(0)
        g = Grid.make(*GRID_T)
        world = dist.get_world_size()
        batches = gem.init_gem_slab(g, 8, rank, world, pinned=False)
        if inject and rank == 0:
            s, a, val = inject
            batches[s].arrays[a][0] = val
        f = gem.gem_field(g)
        caps = [b.count() + 4096 for b in batches]
        store = DeviceStore(g, caps, mode)
        store.upload_field(f)
        for s, b in enumerate(batches):
            store.upload(s, b.span())
        mig = DeviceMigration(store, rank, world)
        sw = SlabWorld(g, mig, 4, dist, torch.device("cuda"))
        sw.set_total()
        mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
        for _ in range(cycles):
            sw.step(mps)
        out = []
        for s in range(4):
            n = store.count(s)
            p6 = [np.empty(n) for _ in range(6)]
            store.download(s, p6)
            out.append(p6)
        store.sync()
        store.close()
        return out
    return fn


def _key_sorted(p6):
    order = np.lexsort([np.round(p6[a], 6) for a in (2, 1, 0)])
    return [a[order] for a in p6]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_gpu_slab_world_matches_reference_simulation(gpu, world, mode):
    res, errs = run_ranks(_rank_fn(mode, 3), world)
    assert not any(errs), errs
    sim = oracle.RefSimulation(GRID_T, 8, workers=world, engine="cpu", field_passes=0)
    sim.run(3)
    g = Grid.make(*GRID_T)
    for s in range(4):
        for r in range(world):
            assert np.all(owner_of(res[r][s][1], g, world) == r)
        mine = [np.concatenate([res[r][s][a] for r in range(world)]) for a in range(6)]
        ref = sim.gather(s)
        assert len(mine[0]) == len(ref[0])
        if mode == "strict":
            np.testing.assert_array_equal(oracle.multiset(mine), oracle.multiset(ref))
        else:
            assert_within_contract(_key_sorted(mine), _key_sorted(ref), GRID_T, tol=1e-11)


def test_gpu_slab_world_cfl_violation(gpu):
    res, errs = run_ranks(_rank_fn("fast", 1, inject=(1, 4, 40.0)), 4)
    assert isinstance(errs[0], CflViolation) and "non-neighbor slab" in str(errs[0]), errs
    assert all(isinstance(e, EngineFault) for e in errs[1:]), errs


def test_gpu_slab_world_nan_fault(gpu):
    res, errs = run_ranks(_rank_fn("strict", 1, inject=(0, 3, float("nan"))), 2)
    assert isinstance(errs[0], NumericalFault) and "particle index 0" in str(errs[0]), errs
    assert isinstance(errs[1], EngineFault), errs
