"""Average step time (mover + amortised cell re-sort every N steps) over 64 steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import Grid, MoverParams
grid = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
batches = gem.init_gem_species(grid, 216, pinned=True)
field = gem.gem_field(grid)
mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
st = DeviceStore(grid, [b.count() for b in batches], "fast")
st.upload_field(field)
for s, b in enumerate(batches): st.upload(s, b.span())
st.sync()
for s in range(4): st.sort(s)
st.sync()
st.record(0)
for s in range(4): st.sort(s)
st.record(1)
print(f"sort all species: {st.elapsed_ms(0, 1):.3f} ms")
for N in (4, 8, 16, 32, 10000):
    for s in range(4): st.sort(s)
    st.record(2)
    for k in range(64):
        if k % N == 0 and k > 0:
            for s in range(4): st.sort(s)
        st.move_all(mps)
    st.record(3)
    print(f"resort every {N:5d}: {st.elapsed_ms(2, 3) / 64:.3f} ms/step")
