"""Fresh-after-sort vs 40-steps-later mover launches (for ncu -s/-c)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import Grid, MoverParams
grid = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
batches = gem.init_gem_species(grid, 216, pinned=True, species=(0,))
field = gem.gem_field(grid)
mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
st = DeviceStore(grid, [b.count() for b in batches], "fast")
st.upload_field(field)
for s, b in enumerate(batches): st.upload(s, b.span())
st.sort(0); st.sync()
for k in range(int(os.environ.get("NSTEPS", "41"))):
    st.record(2); st.move_all(mps); st.record(3)
    if k in (0, 10, 40): print(k, st.elapsed_ms(2, 3))
st.sync()
