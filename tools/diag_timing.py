"""Diagnostics: host launch cost vs device time of the mover on C2."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import Grid, MoverParams

mode = sys.argv[1] if len(sys.argv) > 1 else "fast"
fieldkind = sys.argv[2] if len(sys.argv) > 2 else "gem"
grid = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
batches = gem.init_gem_species(grid, 216, pinned=True)
field = gem.gem_field(grid) if fieldkind == "gem" else gem.gem_bench_field(grid)
n = sum(b.count() for b in batches)
mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
st = DeviceStore(grid, [b.count() for b in batches], mode)
st.upload_field(field)
for s, b in enumerate(batches):
    st.upload(s, b.span())
for s in range(4):
    st.sort(s)
st.sync()
for _ in range(3):
    st.move_all(mps)
st.sync()
t0 = time.perf_counter()
st.record(0)
for _ in range(20):
    st.move_all(mps)
st.record(1)
t1 = time.perf_counter()
ms = st.elapsed_ms(0, 1)
t2 = time.perf_counter()
print(f"host enqueue {1e3*(t1-t0)/20:.3f} ms/call, device {ms/20:.3f} ms/step, wall {1e3*(t2-t0)/20:.3f}")
for s in range(4):
    st.record(2); st.move(s, mps[s]); st.record(3)
    print(f"species {s}: n={batches[s].count()} {st.elapsed_ms(2,3):.3f} ms  -> {batches[s].count()/st.elapsed_ms(2,3)/1e3:.0f} MPA/s")
