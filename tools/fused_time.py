"""C2: per-launch times of the plain FAST mover, the separate deposit and the
fused mover+deposit (b2m_move_deposit_all), right after a sort and after
drift.  Each timed with CUDA events on the store's stream, synchronised."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import Grid, MoverParams
grid = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
batches = gem.init_gem_species(grid, 216, pinned=True)
mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
qs = [b.q_per_particle for b in batches]
st = DeviceStore(grid, [b.count() for b in batches], "fast")
st.upload_field(gem.gem_bench_field(grid))
for s, b in enumerate(batches): st.upload(s, b.span())
for s in range(4): st.sort(s)
st.moments_zero(False)
st.move_all(mps); st.sync()

def t(fn):
    st.record(2); fn(); st.record(3); st.sync(); return st.elapsed_ms(2, 3)

def dep():
    for s in range(4): st.deposit(s, qs[s])

for rnd in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    st.moments_zero(False)
    a = t(lambda: st.move_all(mps))
    b = t(dep)
    c = t(lambda: st.move_deposit_all(mps, qs))
    print(f"round {rnd}: mover {a:.3f}  deposit {b:.3f}  fused {c:.3f} ms", flush=True)
