"""One NCCL rank of the multi-GPU native-world test (launched by
test_world_nccl_gpu.py, one process per GPU):

    python tests/nccl_world_worker.py RANK WORLD PORT OUTDIR CYCLES MODE

The rank holds its y-slab of the GEM state on GPU RANK (GPU 0 for every rank
with B2M_NCCL_LIB = the fake NCCL of tests/fake_nccl) in a STRICT device
store and runs CYCLES of b2m_world_step (mover + owner scan + compaction +
grouped ncclSend/ncclRecv with prev/next + merge + count all-reduce) through
NativeSlabWorld, then deposits rho/J/pressure and reduces them across ranks
(b2m_world_reduce_moments: all-gather + rank-ordered sum).
MODE "ok", or "nan": rank 1 gets a NaN velocity -> its NumericalFault, and
every peer an EngineFault, nobody hangs; "cap": rank 0 cannot take the
particles rank 1 sends it -> its AllocError, rank 1's EngineFault.  Rank r writes OUTDIR/rank{r}.npz
(particles + reduced mesh) or OUTDIR/rank{r}.err."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1904_03684_b200 import gem  # noqa: E402
from paper_1904_03684_b200.engine import DeviceStore  # noqa: E402
from paper_1904_03684_b200.mover import Grid, MoverParams  # noqa: E402
from paper_1904_03684_b200.partition import NativeSlabWorld  # noqa: E402

GRID = (8, 12, 8, 6.4, 9.6, 6.4)
PPC = 8


def main():
    rank, world, port, outdir, cycles, mode = (int(sys.argv[1]), int(sys.argv[2]), sys.argv[3],
                                               sys.argv[4], int(sys.argv[5]), sys.argv[6])
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=port, RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    # B2M_NCCL_LIB (tests/fake_nccl): every rank on GPU 0, torch.distributed
    # over gloo (it only carries the unique id); else one GPU per rank
    fake = bool(os.environ.get("B2M_NCCL_LIB"))
    dev = 0 if fake else rank
    torch.cuda.set_device(dev)
    if fake:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    grid = Grid.make(*GRID)
    batches = gem.init_gem_slab(grid, PPC, rank, world, pinned=False)
    p6s = [b.span() for b in batches]
    if mode == "nan" and rank == 1:
        p6s[0][3][5] = np.nan
    caps = [int(b.count() * 1.5) + 4096 for b in batches]
    if mode == "cap":
        # rank 1 hands 64 species-0 particles to rank 0 (y just below its own
        # slab), and rank 0 has no room for arrivals: its capacity is its count
        if rank == 1:
            p6s[0][1][:64] = grid.ly / world - 1e-3
        else:
            caps[0] = batches[0].count()
    st = DeviceStore(grid, caps, "strict", device=dev)
    st.upload_field(gem.gem_field(grid))
    for s, p in enumerate(p6s):
        st.upload(s, p)
    if mode in ("bcast_zinv", "bcast_zvar"):
        # rank 0's field (z-invariant, or varying in z) broadcast over fields
        # the other ranks scrambled: every rank must end with rank 0's bits
        f = gem.gem_bench_field(grid, z_varying=(mode == "bcast_zvar"))
        if rank != 0:
            f.E[:] = -7.0
            f.B[:] = 3.0
        st.upload_field(f)
        sw = NativeSlabWorld(grid, st, rank, world, dist)
        sw.broadcast_field(0)
        from paper_1904_03684_b200.mover import FieldMesh
        out = FieldMesh(grid, np.zeros_like(f.E.ravel()), np.zeros_like(f.B.ravel()))
        st.download_field(out)
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), E=out.E.ravel(), B=out.B.ravel())
        st.close()
        dist.destroy_process_group()
        return
    sw = NativeSlabWorld(grid, st, rank, world, dist)
    sw.set_total()
    mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
    try:
        for _ in range(cycles):
            sw.broadcast_field(0)
            sw.step(mps)
        mesh = sw.deposit_moments([b.q_per_particle for b in batches], with_pressure=True)
        out = {"mesh": mesh.cpu().numpy()}
        for s in range(len(batches)):
            n = st.count(s)
            p = [np.empty(n) for _ in range(6)]
            st.download(s, p)
            st.sync()
            for a in range(6):
                out[f"s{s}a{a}"] = p[a]
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    except Exception as e:  # noqa: BLE001 - report the typed fault to the test
        with open(os.path.join(outdir, f"rank{rank}.err"), "w") as fh:
            fh.write(f"{type(e).__name__}: {e}")
    st.close()
    try:
        dist.destroy_process_group()
    except Exception:
        pass


if __name__ == "__main__":
    main()
