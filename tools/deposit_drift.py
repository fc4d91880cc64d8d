"""C2: moment deposition time vs mover steps since the last cell sort (FAST context)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import Grid, MoverParams
grid = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
batches = gem.init_gem_species(grid, 216, pinned=True)
mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
st = DeviceStore(grid, [b.count() for b in batches], "fast")
st.upload_field(gem.gem_field(grid))
for s, b in enumerate(batches): st.upload(s, b.span())
for s in range(4): st.sort(s)
n = sum(b.count() for b in batches)
done = 0
for target in (0, 1, 4, 8, 16, 32):
    while done < target:
        st.move_all(mps); done += 1
    st.moments_zero(False)
    st.record(2)
    for s, b in enumerate(batches): st.deposit(s, b.q_per_particle)
    st.record(3)
    st.sync()
    ms = st.elapsed_ms(2, 3)
    print(f"steps since sort {target:3d}: deposit {ms:.3f} ms", flush=True)
