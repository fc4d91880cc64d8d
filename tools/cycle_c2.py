"""A device-resident PIC cycle at C2 on one B200, the reference's cycle order
(runtime.cpp:218-262): field phase stand-in (field_phase_stub, 100 passes =
the reference default cfg.field_passes) -> mover (FAST) -> moments (rho+J, + the pressure tensor by default),
with a cell sort every --resort cycles.  Prints per-phase device times."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_03684_b200 import gem  # noqa: E402
from paper_1904_03684_b200.engine import DeviceStore  # noqa: E402
from paper_1904_03684_b200.mover import Grid, MoverParams  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cycles", type=int, default=16)
ap.add_argument("--passes", type=int, default=100)
ap.add_argument("--resort", type=int, default=8)
ap.add_argument("--pressure", type=int, default=1,
                help="deposit the pressure tensor too (the reference Simulation default, sim_config.hpp:46)")
a = ap.parse_args()
grid = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
batches = gem.init_gem_species(grid, 216, pinned=True)
mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
st = DeviceStore(grid, [b.count() for b in batches], "fast")
st.upload_field(gem.gem_like_field(grid))
for s, b in enumerate(batches):
    st.upload(s, b.span())
n = sum(b.count() for b in batches)
phases = {"sort": 0.0, "field_stub": 0.0, "mover": 0.0, "moments": 0.0}
st.moments_zero(bool(a.pressure))
for c in range(a.cycles + 1):
    times = {}
    st.record(0)
    if c % a.resort == 0:
        for s in range(4):
            st.sort(s)
    st.record(1)
    st.field_stub(a.passes)
    st.record(2)
    st.move_all(mps)
    st.record(3)
    st.moments_zero(bool(a.pressure))
    for s, b in enumerate(batches):
        st.deposit(s, b.q_per_particle)
    st.record(4)
    st.sync()
    if c == 0:
        continue  # warm-up
    for k, (i, j) in zip(phases, [(0, 1), (1, 2), (2, 3), (3, 4)]):
        phases[k] += st.elapsed_ms(i, j) / a.cycles
total = sum(phases.values())
print(json.dumps({"config": "C2 61M particles, FAST, field_passes=%d, sort every %d cycles, "
                  "pressure %d" % (a.passes, a.resort, a.pressure), "ms_per_cycle": total,
                  "phases_ms": phases, "mover_mpa_s": n / (phases["mover"] * 1e-3) / 1e6}))
