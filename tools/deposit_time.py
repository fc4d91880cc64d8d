"""C2 GEM state: time moment deposition (all species) fresh-sorted, on the device."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import Grid, MoverParams
grid = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
batches = gem.init_gem_species(grid, 216, pinned=True)
st = DeviceStore(grid, [b.count() for b in batches], "strict")
st.upload_field(gem.gem_field(grid))
for s, b in enumerate(batches): st.upload(s, b.span())
n = sum(b.count() for b in batches)
for sort in (False, True):
    if sort:
        for s in range(4): st.sort(s)
    for pressure in (False, True):
        ts = []
        for k in range(5):
            st.moments_zero(pressure)
            st.record(2)
            for s, b in enumerate(batches): st.deposit(s, b.q_per_particle)
            st.record(3)
            st.sync()
            ts.append(st.elapsed_ms(2, 3))
        best = min(ts)
        print(f"sorted={sort} pressure={pressure}: {best:.3f} ms  {n / best / 1e3:.0f} MPA/s "
              f"({n * 48 / best / 1e6:.0f} GB/s of particle reads)", flush=True)
# FAST-mode context: reciprocal scaling + FMA
st.set_mode("fast")
for pressure in (False, True):
    ts = []
    for k in range(5):
        st.moments_zero(pressure)
        st.record(2)
        for s, b in enumerate(batches): st.deposit(s, b.q_per_particle)
        st.record(3)
        st.sync()
        ts.append(st.elapsed_ms(2, 3))
    best = min(ts)
    print(f"[fast ctx] sorted=True pressure={pressure}: {best:.3f} ms  {n / best / 1e3:.0f} MPA/s", flush=True)
