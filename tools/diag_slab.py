"""Where the partition-layer step spends its time at N = 1 (no migration):
host wall time per phase of SlabWorld.step, and device time of the mover."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29531")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import Grid, MoverParams
from paper_1904_03684_b200.partition import DeviceMigration, SlabWorld
grid = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
batches = gem.init_gem_slab(grid, 216, 0, 1)
mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
st = DeviceStore(grid, [int(b.count() * 1.05) + 65536 for b in batches], "fast")
st.set_stream(stream.cuda_stream)
st.upload_field(gem.gem_field(grid))
for s, b in enumerate(batches): st.upload(s, b.span()); st.sort(s)
mig = DeviceMigration(st, 0, 1)
sw = SlabWorld(grid, mig, 4, dist, torch.device("cuda", 0))
sw.set_total()
for _ in range(3): sw.step(mps)
torch.cuda.synchronize()
# phases
T = {}
def tick(name, t0):
    T[name] = T.get(name, 0.0) + time.perf_counter() - t0
    return time.perf_counter()
K = 10
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t_all = time.perf_counter()
for _ in range(K):
    t = time.perf_counter()
    mig.move_migrate_all(mps); t = tick("launch move_migrate_all", t)
    mig.sync(); t = tick("sync (mover + compaction)", t)
    outs = [(mig.outbox(s, 0), mig.outbox(s, 1)) for s in range(4)]; t = tick("outbox", t)
    ins = sw._exchange(outs); t = tick("exchange", t)
    for s in range(4): mig.inbox_append(s, ins[s].contiguous())
    t = tick("inbox_append", t)
    sw._reduce_count(sw._count_all(), 0)
    t = tick("count all-reduce", t)
e1.record(); torch.cuda.synchronize()
wall = (time.perf_counter() - t_all) / K * 1e3
print(f"step wall {wall:.3f} ms, device {e0.elapsed_time(e1) / K:.3f} ms")
for k, v in T.items(): print(f"  {k:28s} {v / K * 1e3:.3f} ms")
st.record(2); st.move_all(mps); st.record(3); st.sync()
print(f"plain move_all: {st.elapsed_ms(2, 3):.3f} ms")
# the same step in the library (b2m_world_step over a one-rank NCCL communicator)
from paper_1904_03684_b200.partition import NativeSlabWorld
st2 = DeviceStore(grid, [int(b.count() * 1.05) + 65536 for b in batches], "fast")
st2.set_stream(stream.cuda_stream)
st2.upload_field(gem.gem_field(grid))
for s, b in enumerate(batches): st2.upload(s, b.span()); st2.sort(s)
nw = NativeSlabWorld(grid, st2, 0, 1, dist)
nw.set_total()
for _ in range(3): nw.step(mps)
torch.cuda.synchronize()
e0.record(); t0 = time.perf_counter()
for _ in range(K): nw.step(mps)
e1.record(); torch.cuda.synchronize()
print(f"native b2m_world_step: wall {(time.perf_counter() - t0) / K * 1e3:.3f} ms, "
      f"device {e0.elapsed_time(e1) / K:.3f} ms")
dist.destroy_process_group()
