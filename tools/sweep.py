"""Tuning sweep: mover time fresh-after-sort and after N steps, per lib variant."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import os, sys
sys.path.insert(0, %r)
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
for s in range(4): st.sort(s)
st.sync()
ts = []
for k in range(41):
    st.record(2); st.move_all(mps); st.record(3); ts.append(st.elapsed_ms(2, 3))
print(os.environ.get("B2M_LIB"), "fresh %%.2f  step5 %%.2f  step10 %%.2f  step20 %%.2f  step40 %%.2f" %% (ts[0], ts[5], ts[10], ts[20], ts[40]))
''' % ROOT
for v in sys.argv[1:]:
    env = dict(os.environ, B2M_LIB=os.path.join(ROOT, "paper_1904_03684_b200", f"libb2m_{v}.so"))
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-2000:], flush=True)
