"""Diagnostics: mover time vs steps since the last cell sort; sort cost."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import Grid, MoverParams

grid = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
batches = gem.init_gem_species(grid, 216, pinned=True)
field = gem.gem_field(grid)
n = sum(b.count() for b in batches)
mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
st = DeviceStore(grid, [b.count() for b in batches], "fast")
st.upload_field(field)
for s, b in enumerate(batches):
    st.upload(s, b.span())
st.sync()
for rep in range(2):
    st.record(0)
    for s in range(4):
        st.sort(s)
    st.record(1)
    print(f"sort all species: {st.elapsed_ms(0, 1):.3f} ms")
    ts = []
    for k in range(60):
        st.record(2); st.move_all(mps); st.record(3)
        ts.append(st.elapsed_ms(2, 3))
    print("move ms after sort:", " ".join(f"{t:.2f}" for t in ts))
