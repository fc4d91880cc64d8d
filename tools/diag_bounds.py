"""Upper-bound experiments for the FAST kernel (see DESIGN.md / profiles)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import Grid, MoverParams
grid = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
n = 28311552
field = gem.gem_field(grid)
mp = MoverParams.make(0.1, -25.0, 3)
def run(p6, label):
    st = DeviceStore(grid, [n], "fast")
    st.upload_field(field); st.upload(0, p6); st.sync()
    st.move(0, mp); st.sync()
    st.record(0)
    for _ in range(5): st.move(0, mp)
    st.record(1)
    print(f"{os.path.basename(os.environ.get('B2M_LIB','default'))} {label}: {st.elapsed_ms(0,1)/5:.3f} ms per {n} particles", flush=True)
    st.close()
r = np.random.default_rng(0)
# (1) every particle inside one cell (0.2..0.3 of cell (10,20,10)), thermal-ish velocity
one = [10.2 * 0.4 + r.random(n) * 0.04, 20.2 * 0.2 + r.random(n) * 0.02, 10.2 * 0.2 + r.random(n) * 0.02,
       0.001 * r.standard_normal(n), 0.001 * r.standard_normal(n), 0.001 * r.standard_normal(n)]
run(one, "one-cell")
b = gem.init_gem_species(grid, 216, species=(0,))[0]
run(b.span(), "gem-bg-electrons (cell order)")
