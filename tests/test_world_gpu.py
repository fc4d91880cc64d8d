"""The native slab world (b2m_world_*: the per-cycle protocol of
Simulation, runtime.cpp:218-288, in the library).  Several ranks as
contexts of one process on one B200 run b2m_world_loopback_step -- the same
native phases as b2m_world_step, device copies standing in for NCCL -- and
must reproduce the reference multi-worker Simulation (STRICT: bitwise
particle multiset, FAST: within contract), keep every particle on its owner
rank, conserve the count, and surface faults typed on the faulting rank with
EngineFault elsewhere.  A world of one runs b2m_world_step itself, through a
real NCCL communicator."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle
from paper_1904_03684_b200 import _capi, gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.errors import CflViolation, EngineFault, NumericalFault
from paper_1904_03684_b200.mover import Grid, MoverParams
from paper_1904_03684_b200.partition import (NativeSlabWorld, loopback_step, loopback_world,
                                             owner_of)
from tests._util import assert_bitwise, assert_within_contract

pytestmark = pytest.mark.gpu
GRID_T = (8, 8, 8, 6.4, 6.4, 6.4)


def _stores(mode, world, inject=None):
    g = Grid.make(*GRID_T)
    stores, batches_all = [], []
    for r in range(world):
        batches = gem.init_gem_slab(g, 8, r, world, pinned=False)
        if inject and r == inject[0]:
            _, s, a, val = inject
            batches[s].arrays[a][0] = val
        st = DeviceStore(g, [b.count() + 4096 for b in batches], mode)
        st.upload_field(gem.gem_field(g))
        for s, b in enumerate(batches):
            st.upload(s, b.span())
        stores.append(st)
        batches_all.append(batches)
    loopback_world(stores, g)
    mps = [MoverParams.make(0.1, b.qom, 3) for b in batches_all[0]]
    return g, stores, mps


def _download(st):
    out = []
    for s in range(st.n_species):
        p6 = [np.empty(st.count(s)) for _ in range(6)]
        st.download(s, p6)
        out.append(p6)
    st.sync()
    return out


def _key_sorted(p6):
    order = np.lexsort([np.round(p6[a], 6) for a in (2, 1, 0)])
    return [a[order] for a in p6]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_loopback_world_matches_reference_simulation(gpu, world, mode):
    g, stores, mps = _stores(mode, world)
    sent = 0
    for _ in range(3):
        sent += loopback_step(stores, mps)
    assert sent > 0   # particles did cross slab boundaries
    res = [_download(st) for st in stores]
    sim = oracle.RefSimulation(GRID_T, 8, workers=world, engine="cpu", field_passes=0)
    sim.run(3)
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
    for st in stores:
        st.close()


def test_loopback_world_cfl_violation(gpu):
    g, stores, mps = _stores("fast", 4, inject=(1, 1, 4, 40.0))
    with pytest.raises(CflViolation, match="non-neighbor slab"):
        loopback_step(stores, mps)
    for st in stores:
        st.close()


def test_loopback_world_nan_fault(gpu):
    g, stores, mps = _stores("strict", 2, inject=(0, 0, 3, float("nan")))
    with pytest.raises(NumericalFault, match="particle index 0"):
        loopback_step(stores, mps)
    for st in stores:
        st.close()


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_world_of_one_over_nccl_equals_plain_mover(gpu, mode):
    """b2m_world_step with a real one-rank NCCL communicator (no exchange):
    the same particles as the plain mover, the count conserved."""
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29547")
    if not dist.is_initialized():
        dist.init_process_group("gloo", rank=0, world_size=1)
    g = Grid.make(*GRID_T)
    batches = gem.init_gem_slab(g, 8, 0, 1, pinned=False)
    mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
    a = DeviceStore(g, [b.count() + 64 for b in batches], mode)
    b_ = DeviceStore(g, [b.count() + 64 for b in batches], mode)
    for st in (a, b_):
        st.upload_field(gem.gem_field(g))
        for s, b in enumerate(batches):
            st.upload(s, b.span())
    uid = (C.c_ubyte * 128)()
    _capi.check(_capi.lib().b2m_world_id(uid))
    _capi.check(_capi.lib().b2m_world_init(a.h, uid, 0, 1))
    w = NativeSlabWorld.__new__(NativeSlabWorld)
    w._capi, w.store, w.ns, w.last_exchange = _capi, a, a.n_species, {}
    total = w.set_total()
    assert total == sum(b.count() for b in batches)
    w.broadcast_field(0)   # a one-rank broadcast: the field (and its tables) unchanged
    for _ in range(3):
        assert w.step(mps) == 0
        assert w.last_exchange["global_count"] == total
        b_.move_all(mps)
    for x, y in zip(_download(a), _download(b_)):
        assert_bitwise(x, y, mode)
    # moments through the world (a one-rank all-reduce) equal the plain deposit
    qpp = [b.q_per_particle for b in batches]
    mine = w.deposit_moments(qpp).cpu().numpy().copy()
    b_.moments_zero(False)
    for s, q in enumerate(qpp):
        b_.deposit(s, q)
    ptr, n = b_.moments_device()
    from paper_1904_03684_b200.partition import _CudaArray
    import torch
    want = torch.as_tensor(_CudaArray(ptr, (n,)), device="cuda").cpu().numpy()
    np.testing.assert_allclose(mine, want, rtol=0, atol=1e-12 * float(np.max(np.abs(want))))
    a.close()
    b_.close()


def test_world_api_misuse_is_config_error(gpu):
    from paper_1904_03684_b200.errors import ConfigError
    g = Grid.make(*GRID_T)
    st = DeviceStore(g, [64], "fast")
    arr = (_capi.b2m_mover_params * 1)(MoverParams.make(0.1, 1.0, 3).to_c())
    with pytest.raises(ConfigError, match="world_init"):
        _capi.check(_capi.lib().b2m_world_step(st.h, arr, None, None))
    with pytest.raises(ConfigError, match="does not divide"):
        _capi.check(_capi.lib().b2m_world_init(st.h, None, 0, 3))
    _capi.check(_capi.lib().b2m_world_init(st.h, None, 0, 2))
    with pytest.raises(ConfigError, match="already"):
        _capi.check(_capi.lib().b2m_world_init(st.h, None, 0, 2))
    with pytest.raises(ConfigError, match="NCCL communicator"):
        _capi.check(_capi.lib().b2m_world_step(st.h, arr, None, None))
    # a world of two without a communicator cannot replicate a field
    with pytest.raises(ConfigError, match="no NCCL communicator"):
        _capi.check(_capi.lib().b2m_world_broadcast_field(st.h, 0))
    st.close()


def test_world_step_per_rank_failure_runs_the_protocol(gpu):
    """A per-rank failure (here: no field on this rank) is carried through the
    collectives like a fault instead of returning before them (so peers never
    wait alone): the typed error comes back, the context is poisoned, and the
    next step reports EngineFault -- again after running the protocol."""
    import torch.distributed as dist
    from paper_1904_03684_b200.errors import ConfigError
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29547")
    if not dist.is_initialized():
        dist.init_process_group("gloo", rank=0, world_size=1)
    g = Grid.make(*GRID_T)
    batches = gem.init_gem_slab(g, 8, 0, 1, pinned=False)
    mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
    st = DeviceStore(g, [b.count() + 64 for b in batches], "fast")
    for s, b in enumerate(batches):
        st.upload(s, b.span())
    uid = (C.c_ubyte * 128)()
    _capi.check(_capi.lib().b2m_world_id(uid))
    _capi.check(_capi.lib().b2m_world_init(st.h, uid, 0, 1))
    arr = (_capi.b2m_mover_params * len(mps))(*[m.to_c() for m in mps])
    with pytest.raises(ConfigError, match="no field"):
        _capi.check(_capi.lib().b2m_world_step(st.h, arr, None, None))
    with pytest.raises(EngineFault):
        _capi.check(_capi.lib().b2m_world_step(st.h, arr, None, None))
    st.close()


@pytest.mark.parametrize("mode,field", [("strict", "gem"), ("fast", "gem+E"),
                                        ("fast", "zvarying")])
def test_loopback_four_ranks_equal_one_context_after_many_steps(gpu, mode, field):
    """1.2M GEM particles split over 4 slab ranks (loopback protocol) for 8
    steps: every particle is on its owner rank, and the union is the bitwise
    multiset of the same particles moved 8 times in one context (the mover is
    per-particle, migration only relocates) -- STRICT, FAST on the
    z-invariant bench field (the column kernel's owner scan) and FAST on a
    z-varying field (the general kernel's)."""
    grid_t = (32, 32, 16, 12.8, 6.4, 3.2)
    g = Grid.make(*grid_t)
    world = 4
    fld = (gem.gem_field(g) if field == "gem" else
           gem.gem_bench_field(g, z_varying=(field == "zvarying")))
    full = gem.init_gem_species(g, 72, pinned=False)
    mps = [MoverParams.make(0.1, b.qom, 3) for b in full]
    ref = DeviceStore(g, [b.count() for b in full], mode)
    ref.upload_field(fld)
    for s, b in enumerate(full):
        ref.upload(s, b.span())
    stores = []
    for r in range(world):
        part = gem.init_gem_slab(g, 72, r, world, pinned=False)
        st = DeviceStore(g, [b.count() * 2 + 4096 for b in part], mode)
        st.upload_field(fld)
        for s, b in enumerate(part):
            st.upload(s, b.span())
        stores.append(st)
    loopback_world(stores, g)
    sent = 0
    for _ in range(8):
        sent += loopback_step(stores, mps)
        ref.move_all(mps)
    assert sent > 1000
    want = _download(ref)
    got = [_download(st) for st in stores]
    for s in range(4):
        for r in range(world):
            assert np.all(owner_of(got[r][s][1], g, world) == r)
        mine = [np.concatenate([got[r][s][a] for r in range(world)]) for a in range(6)]
        np.testing.assert_array_equal(oracle.multiset(mine), oracle.multiset(want[s]))
    for st in stores + [ref]:
        st.close()


def test_loopback_with_an_empty_species(gpu):
    """A species with no particles on any rank rides through the protocol
    (zero counts, zero totals) while the others migrate; counts conserved."""
    g = Grid.make(*GRID_T)
    world = 2
    stores = []
    for r in range(world):
        batches = gem.init_gem_slab(g, 8, r, world, pinned=False)
        st = DeviceStore(g, [b.count() + 4096 for b in batches], "fast")
        st.upload_field(gem.gem_field(g))
        for s, b in enumerate(batches):
            if s != 2:   # species 2 (the electron sheet) left empty everywhere
                st.upload(s, b.span())
        stores.append(st)
    mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
    loopback_world(stores, g)
    total0 = sum(st.count(s) for st in stores for s in range(4))
    for _ in range(4):
        loopback_step(stores, mps)
    assert sum(st.count(2) for st in stores) == 0
    assert sum(st.count(s) for st in stores for s in range(4)) == total0
    for r, st in enumerate(stores):
        for s in range(4):
            y = _download(st)[s][1]
            assert np.all(owner_of(y, g, world) == r)
        st.close()
