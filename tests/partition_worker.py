"""One gloo rank of the partition-layer CPU test (launched by test_partition.py).

    python tests/partition_worker.py RANK WORLD PORT OUTDIR CYCLES MODE

MODE: "ok" (plain run), "cfl" (inject a particle jumping two slabs),
"lose" (the store drops a particle -> count-drift EngineFault), "probe"
(NativeSlabWorld when rank 1 cannot load NCCL -> ConfigError on every rank).
Rank r writes OUTDIR/rank{r}.npz with its final particles, or OUTDIR/rank{r}.err.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch  # noqa: E402

from paper_1904_03684_b200 import gem  # noqa: E402
from paper_1904_03684_b200.mover import Grid, MoverParams  # noqa: E402
from paper_1904_03684_b200.partition import SlabWorld  # noqa: E402
from tests._hoststore import HostStore  # noqa: E402


def main():
    rank, world, port, outdir, cycles, mode = (int(sys.argv[1]), int(sys.argv[2]), sys.argv[3],
                                               sys.argv[4], int(sys.argv[5]), sys.argv[6])
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=port, RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo")
    grid = Grid.make(8, 8, 8, 6.4, 6.4, 6.4)          # the reference small_cfg
    if mode == "probe":
        # NativeSlabWorld's NCCL probe when rank 1 has no NCCL: every rank
        # must raise ConfigError (none may enter the communicator setup)
        if rank == 1:
            os.environ["B2M_NCCL_LIB"] = "/nonexistent/libnccl.so.2"
        from paper_1904_03684_b200.partition import NativeSlabWorld

        class _NoStore:
            h, n_species = None, 4
        try:
            NativeSlabWorld(grid, _NoStore(), rank, world, dist)
            msg = "no error"
        except Exception as e:  # noqa: BLE001
            msg = f"{type(e).__name__}: {e}"
        with open(os.path.join(outdir, f"rank{rank}.err"), "w") as fh:
            fh.write(msg)
        dist.destroy_process_group()
        return
    batches = gem.init_gem_slab(grid, 8, rank, world, pinned=False)
    p6s = [b.span() for b in batches]
    if mode == "cfl" and rank == 0:
        p6s[1][4][0] = 40.0    # test_runtime.cpp:241-242: an ion jumping 4.0 in y at dt 0.1
    f = gem.gem_field(grid)
    store = HostStore(grid, p6s, f.E.ravel(), f.B.ravel(), rank, world,
                      lose_one=(mode == "lose" and rank == 1))
    sw = SlabWorld(grid, store, 4, dist, torch.device("cpu"))
    sw.set_total()
    mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
    try:
        for _ in range(cycles):
            sw.step(mps)
        np.savez(os.path.join(outdir, f"rank{rank}.npz"),
                 **{f"s{s}a{a}": store.p[s][a] for s in range(4) for a in range(6)})
    except Exception as e:  # noqa: BLE001 - report the typed fault to the test
        with open(os.path.join(outdir, f"rank{rank}.err"), "w") as fh:
            fh.write(f"{type(e).__name__}: {e}")
    try:
        dist.destroy_process_group()
    except Exception:
        pass


if __name__ == "__main__":
    main()
