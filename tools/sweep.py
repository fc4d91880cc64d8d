"""Tuning sweep: C2 mover time fresh-after-sort and after N steps, per lib variant.

  python tools/sweep.py VARIANT[:3d] ...
VARIANT names paper_1904_03684_b200/libb2m_VARIANT.so ("default" = libb2m.so);
":3d" moves in a z-varying field (the general 3-D kernel), else the GEM bench
field (z-invariant: the 2-D-in-3-D kernel)."""
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
field = gem.gem_bench_field(grid, z_varying=os.environ.get("SW_3D") == "1")
mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
st = DeviceStore(grid, [b.count() for b in batches], os.environ.get("B2M_MODE", "fast"))
st.upload_field(field)
for s, b in enumerate(batches): st.upload(s, b.span())
for s in range(4): st.sort(s)
st.sync()
ts = []
for k in range(41):
    st.record(2); st.move_all(mps); st.record(3); ts.append(st.elapsed_ms(2, 3))
avg = sum(ts[:32]) / 32  # the bench's cycle: a re-sort every 32 steps
print("%%-28s fresh %%.3f  step5 %%.3f  step10 %%.3f  step20 %%.3f  step40 %%.3f  avg0-31 %%.3f" %% (os.environ["SW_NAME"], ts[0], ts[5], ts[10], ts[20], ts[40], avg))
''' % ROOT
for v in sys.argv[1:]:
    name, _, opt = v.partition(":")
    lib = "libb2m.so" if name == "default" else f"libb2m_{name}.so"
    env = dict(os.environ, B2M_LIB=os.path.join(ROOT, "paper_1904_03684_b200", lib),
               SW_3D="1" if opt == "3d" else "0", SW_NAME=v)
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-2000:], flush=True)
