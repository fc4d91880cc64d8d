"""The native slab world over real NCCL with one process per GPU (ADVICE r1:
the multi-rank exchange had never run).  Skipped unless the box has at least
`world` GPUs -- the round's gpurun boxes have one; the driver's multi-GPU
boxes run it.  STRICT mode: the union of the ranks' particles after the cycles
equals the reference's multi-worker Simulation as a bitwise multiset (the
reference's own worker-count test, test_runtime.cpp:214-226); the reduced
moment mesh is bitwise identical on every rank (rank-ordered sum) and equals
the oracle deposit of all particles to rounding; a NaN on one rank ends the
cycle on every rank with typed errors instead of a hang."""
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest
import torch

import oracle
from paper_1904_03684_b200.mover import Grid
from paper_1904_03684_b200.partition import owner_of

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GRID = (8, 12, 8, 6.4, 9.6, 6.4)


def _gpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, cycles, mode, env=None):
    d = tempfile.mkdtemp(prefix="b2m_nccl_")
    port = str(_free_port())
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "nccl_world_worker.py"),
                               str(r), str(world), port, d, str(cycles), mode],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                              env=dict(os.environ, **(env or {})))
             for r in range(world)]
    for p in procs:
        try:
            p.wait(timeout=300)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise AssertionError("NCCL world ranks hung")
    return d, [p.stdout.read().decode(errors="replace") for p in procs]


def fake_nccl_lib():
    """tests/fake_nccl built into a temporary directory (test infrastructure:
    several native-world ranks on one GPU through host shared memory)."""
    out = os.path.join(tempfile.mkdtemp(prefix="b2m_fake_nccl_"), "libfakenccl.so")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-o", out,
                    os.path.join(HERE, "fake_nccl", "fake_nccl.cpp"), f"-I{cuda}/include",
                    f"-L{cuda}/lib64", "-lcudart", "-lrt"], check=True)
    return out


def _check_world_vs_reference(world, d, logs):
    for r in range(world):
        err = os.path.join(d, f"rank{r}.err")
        assert os.path.exists(os.path.join(d, f"rank{r}.npz")), \
            "\n".join(logs) + (open(err).read() if os.path.exists(err) else "")
    per = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    sim = oracle.RefSimulation(GRID, 8, workers=world, engine="cpu", field_passes=0)
    sim.run(3)
    g = Grid.make(*GRID)
    allp = []
    for s in range(4):
        mine = [np.concatenate([z[f"s{s}a{a}"] for z in per]) for a in range(6)]
        ref = sim.gather(s)
        assert len(mine[0]) == len(ref[0])
        np.testing.assert_array_equal(oracle.multiset(mine), oracle.multiset(ref))
        for r, z in enumerate(per):
            assert np.all(owner_of(z[f"s{s}a1"], g, world) == r)
        allp.append(mine)
    # the rank-ordered reduction: identical on every rank, = oracle to rounding
    for z in per[1:]:
        np.testing.assert_array_equal(z["mesh"], per[0]["mesh"])
    from paper_1904_03684_b200 import gem
    want = [np.zeros(g.cells()) for _ in range(10)]
    qpp = [b.q_per_particle for b in gem.init_gem_species(g, 8)]
    for s, p in enumerate(allp):
        for x, w in zip(oracle.port_deposit_moments(p, GRID, qpp[s], True), want):
            w += x
    got = per[0]["mesh"].reshape(10, -1)
    for a in range(10):
        scale = float(np.max(np.abs(want[a])))
        assert float(np.max(np.abs(got[a] - want[a]))) <= 1e-12 * max(scale, 1e-300)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_native_world_over_fake_nccl_one_gpu(gpu, world):
    """The native slab world's multi-rank protocol (b2m_world_step with real
    peers: counts and records over grouped send/recv, merge, count check;
    the field broadcast; the ordered moments reduction) in separate
    processes on ONE GPU, through tests/fake_nccl (host shared memory, NCCL's
    posting-order matching) -- runnable on this round's one-GPU boxes;
    against the reference's multi-worker Simulation as a bitwise multiset."""
    if not oracle.ref_available():
        pytest.skip("reference library not built")
    d, logs = _run(world, 3, "ok", env={"B2M_NCCL_LIB": fake_nccl_lib()})
    _check_world_vs_reference(world, d, logs)


@pytest.mark.parametrize("mode", ["bcast_zinv", "bcast_zvar"])
@pytest.mark.parametrize("compress", ["1", "0"])
def test_field_broadcast_over_fake_nccl(gpu, mode, compress):
    """b2m_world_broadcast_field at 3 ranks: a z-invariant root field goes
    as plane 0 + a header and is rebuilt on the other ranks, a z-varying one
    (or B2M_BCAST_ZINV=0) as the whole field -- either way every rank ends
    with the root's field bit for bit."""
    lib = fake_nccl_lib()
    d, logs = _run(3, 0, mode, env={"B2M_NCCL_LIB": lib, "B2M_BCAST_ZINV": compress})
    got = []
    for r in range(3):
        f = os.path.join(d, f"rank{r}.npz")
        assert os.path.exists(f), "\n".join(logs)
        got.append(np.load(f))
    from paper_1904_03684_b200 import gem
    want = gem.gem_bench_field(Grid.make(*GRID), z_varying=(mode == "bcast_zvar"))
    for z in got:
        np.testing.assert_array_equal(z["E"].view(np.uint64), want.E.ravel().view(np.uint64))
        np.testing.assert_array_equal(z["B"].view(np.uint64), want.B.ravel().view(np.uint64))


def test_native_world_over_fake_nccl_fault_on_one_rank(gpu):
    d, logs = _run(2, 1, "nan", env={"B2M_NCCL_LIB": fake_nccl_lib()})
    errs = [open(os.path.join(d, f"rank{r}.err")).read() if os.path.exists(
        os.path.join(d, f"rank{r}.err")) else "" for r in range(2)]
    assert errs[1].startswith("NumericalFault"), (errs, logs)
    assert errs[0].startswith("EngineFault"), (errs, logs)


def test_native_world_over_fake_nccl_capacity_overflow_on_one_rank(gpu):
    """Arrivals a rank cannot hold are caught from the counts round, before
    the records round: the step's all-reduced verdict carries the failure,
    so the full rank reports AllocError (the batch capacity is fixed at
    allocation, particle_batch.hpp:43-46) and its peer EngineFault -- both
    return, nobody waits in a collective alone."""
    d, logs = _run(2, 1, "cap", env={"B2M_NCCL_LIB": fake_nccl_lib()})
    errs = [open(os.path.join(d, f"rank{r}.err")).read() if os.path.exists(
        os.path.join(d, f"rank{r}.err")) else "" for r in range(2)]
    assert errs[0].startswith("AllocError") and "capacity" in errs[0], (errs, logs)
    assert errs[1].startswith("EngineFault"), (errs, logs)


@pytest.mark.parametrize("world", [2, 3])
def test_nccl_world_matches_reference_simulation(gpu, world):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs (one rank per GPU), found {_gpus()}")
    if not oracle.ref_available():
        pytest.skip("reference library not built")
    d, logs = _run(world, 3, "ok")
    _check_world_vs_reference(world, d, logs)


def test_nccl_world_fault_on_one_rank_aborts_all(gpu):
    if _gpus() < 2:
        pytest.skip(f"needs 2 GPUs (one rank per GPU), found {_gpus()}")
    d, logs = _run(2, 1, "nan")
    errs = [open(os.path.join(d, f"rank{r}.err")).read() if os.path.exists(
        os.path.join(d, f"rank{r}.err")) else "" for r in range(2)]
    assert errs[1].startswith("NumericalFault"), (errs, logs)
    assert errs[0].startswith("EngineFault"), (errs, logs)
