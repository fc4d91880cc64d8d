"""C2 at N = 1: K native b2m_world_step cycles (one-rank world, no NCCL
communicator: mover + owner scan + compaction + count check), for a launch
list under ncu, next to K plain move_all cycles."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import Grid, MoverParams
from paper_1904_03684_b200.partition import NativeSlabWorld
grid = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
batches = gem.init_gem_slab(grid, 216, 0, 1)
mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
st = DeviceStore(grid, [int(b.count() * 1.05) + 65536 for b in batches], "fast")
st.upload_field(gem.gem_bench_field(grid))
for s, b in enumerate(batches): st.upload(s, b.span()); st.sort(s)
nw = NativeSlabWorld(grid, st, 0, 1, None)
nw.set_total()
K = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(K): nw.step(mps)
st.sync()
for _ in range(K): st.move_all(mps)
st.sync()
st.record(2)
for _ in range(10): nw.step(mps)
st.record(3); st.sync()
a = st.elapsed_ms(2, 3) / 10
st.record(2)
for _ in range(10): st.move_all(mps)
st.record(3); st.sync()
print(f"world step {a:.3f} ms, plain move_all {st.elapsed_ms(2, 3) / 10:.3f} ms")
# the mover with the owner scan + compaction alone (b2m_move_migrate_all)
from paper_1904_03684_b200 import _capi
arr = (_capi.b2m_mover_params * len(mps))(*[m.to_c() for m in mps])
for _ in range(3): _capi.check(_capi.lib().b2m_move_migrate_all(st.h, arr))
st.sync()
st.record(2)
for _ in range(10): _capi.check(_capi.lib().b2m_move_migrate_all(st.h, arr))
st.record(3); st.sync()
print(f"move_migrate_all (mover + owner scan + compaction) {st.elapsed_ms(2, 3) / 10:.3f} ms")
# interleaved: plain mover vs mover + owner scan + compaction, same drift
ta = tb = 0.0
for _ in range(10):
    st.record(2); st.move_all(mps); st.record(3); st.sync(); ta += st.elapsed_ms(2, 3)
    st.record(2); _capi.check(_capi.lib().b2m_move_migrate_all(st.h, arr)); st.record(3); st.sync()
    tb += st.elapsed_ms(2, 3)
print(f"interleaved: move_all {ta / 10:.3f} ms, move_migrate_all {tb / 10:.3f} ms")
