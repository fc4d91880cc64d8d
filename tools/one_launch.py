"""C2 state, cell-sorted, then N FAST mover launches (for ncu captures of one launch).
SW_3D=1: z-varying bench field (general 3-D kernel), else the GEM bench field."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import Grid, MoverParams
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
grid = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
batches = gem.init_gem_species(grid, 216, pinned=True)
mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
st = DeviceStore(grid, [b.count() for b in batches], os.environ.get("B2M_MODE", "fast"))
st.upload_field(gem.gem_bench_field(grid, z_varying=os.environ.get("SW_3D") == "1"))
for s, b in enumerate(batches): st.upload(s, b.span())
for s in range(4): st.sort(s)
st.sync()
for k in range(n):
    st.record(2); st.move_all(mps); st.record(3)
    print(os.environ.get("B2M_LIB", "libb2m.so"), "launch", k, "%.3f ms" % st.elapsed_ms(2, 3), flush=True)
