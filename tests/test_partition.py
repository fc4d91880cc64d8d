"""Partition layer on CPU (no GPU): the reference's slab rules, and the
SlabWorld exchange protocol over gloo with world sizes 2 and 4, compared as a
bitwise particle multiset with the reference's own multi-worker Simulation
(test_runtime.cpp:214-226 pattern), plus the CFL and count-drift faults."""
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import oracle
from paper_1904_03684_b200.errors import ConfigError
from paper_1904_03684_b200.mover import Grid
from paper_1904_03684_b200.partition import decompose, owner_of

HERE = os.path.dirname(os.path.abspath(__file__))
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="reference library unavailable")


def test_decompose_matches_reference_rules(built):
    g = Grid.make(8, 8, 8, 6.4, 6.4, 6.4)
    subs = decompose(g, 4)
    assert [(s.worker_id, s.j_lo, s.j_hi, s.prev, s.next) for s in subs] == \
        [(0, 0, 2, 3, 1), (1, 2, 4, 0, 2), (2, 4, 6, 1, 3), (3, 6, 8, 2, 0)]
    with pytest.raises(ConfigError, match="workers: 3 does not divide ny=8"):
        decompose(g, 3)
    with pytest.raises(ConfigError, match="slab would be 1 cells"):
        decompose(g, 8)
    with pytest.raises(ConfigError, match="must be >= 1"):
        decompose(g, 0)


@needs_ref
def test_decompose_and_owner_of_vs_reference(built):
    import ctypes as C
    g = Grid.make(8, 16, 4, 3.2, 6.4, 1.6)
    for w in (1, 2, 4, 8):
        out = (C.c_int * (5 * w))()
        buf = C.create_string_buffer(256)
        assert oracle.ref().ref_decompose(8, 16, 4, w, out, buf, 256) == 0
        ref = [tuple(out[5 * i:5 * i + 5]) for i in range(w)]
        assert [(s.worker_id, s.j_lo, s.j_hi, s.prev, s.next) for s in decompose(g, w)] == ref
        ys = np.concatenate([np.random.default_rng(w).random(3000) * 6.4,
                             [0.0, np.nextafter(6.4, 0), 0.4, np.nextafter(0.4, 0), 3.2]])
        mine = owner_of(ys, g, w)
        for y, o in zip(ys, mine):
            assert o == oracle.ref().ref_owner_of(float(y), 8, 16, 4, 3.2, 6.4, 1.6, w)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_world(world, cycles, mode):
    d = tempfile.mkdtemp(prefix="b2m_part_")
    port = str(_free_port())
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "partition_worker.py"), str(r),
                               str(world), port, d, str(cycles), mode],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for r in range(world)]
    for p in procs:
        try:
            p.wait(timeout=240)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise AssertionError("partition workers hung (deadlock in the exchange?)")
    logs = [p.stdout.read().decode(errors="replace") for p in procs]
    return d, logs


@needs_ref
@pytest.mark.parametrize("world", [2, 4])
def test_slab_world_matches_reference_simulation_multiset(built, world):
    """gloo ranks running SlabWorld (migration + count check) for 3 cycles ==
    the reference Simulation with the same worker count, as a bitwise
    multiset per species."""
    d, logs = _run_world(world, 3, "ok")
    for r in range(world):
        assert os.path.exists(os.path.join(d, f"rank{r}.npz")), "\n".join(logs) + \
            (open(os.path.join(d, f"rank{r}.err")).read() if os.path.exists(
                os.path.join(d, f"rank{r}.err")) else "")
    grid_t = (8, 8, 8, 6.4, 6.4, 6.4)
    sim = oracle.RefSimulation(grid_t, 8, workers=world, engine="cpu", field_passes=0)
    sim.run(3)
    per_rank = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    g = Grid.make(*grid_t)
    for s in range(4):
        mine = [np.concatenate([z[f"s{s}a{a}"] for z in per_rank]) for a in range(6)]
        ref = sim.gather(s)
        assert len(mine[0]) == len(ref[0])
        np.testing.assert_array_equal(oracle.multiset(mine), oracle.multiset(ref))
        # every rank holds only particles it owns
        for r, z in enumerate(per_rank):
            assert np.all(owner_of(z[f"s{s}a1"], g, world) == r)


def test_slab_world_cfl_violation_aborts_every_rank(built):
    """test_runtime.cpp:239-252 with 4 workers (slabs of 1.6): a particle
    jumping 4.0 in y lands two slabs away -> CflViolation on its rank, and the
    peers abort instead of deadlocking in the exchange."""
    d, logs = _run_world(4, 1, "cfl")
    errs = [open(os.path.join(d, f"rank{r}.err")).read() for r in range(4)]
    assert errs[0].startswith("CflViolation") and "non-neighbor slab" in errs[0], errs
    assert all(e.startswith("EngineFault") for e in errs[1:]), errs


def test_slab_world_count_drift_is_detected(built):
    d, logs = _run_world(2, 1, "lose")
    errs = [open(os.path.join(d, f"rank{r}.err")).read() for r in range(2)]
    assert all(e.startswith("EngineFault") and "particle count drifted" in e for e in errs), errs


def test_native_world_nccl_probe_is_agreed_by_every_rank(built):
    """NativeSlabWorld probes NCCL on every rank and the ranks agree (over
    torch.distributed, gloo here) before any enters ncclCommInitRank: when
    one rank cannot load NCCL, every rank raises ConfigError -- none is left
    waiting in the communicator setup.  bench.py then falls back to the
    Python SlabWorld on all ranks together."""
    d, logs = _run_world(2, 0, "probe")
    errs = [open(os.path.join(d, f"rank{r}.err")).read() for r in range(2)]
    for e in errs:
        assert e.startswith("ConfigError: native world unavailable (rank "), (errs, logs)

