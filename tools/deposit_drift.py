"""C2: moment deposition time vs mover steps since the last cell sort (FAST
context), the separate deposit and the fused mover+deposit, with the state's
disorder: the fraction of particles whose cell differs from the cell of the
particle before them in memory order, and of rows of 32 in one cell.
FIELD=gem: E = 0 (the reference's init_gem field); default gem+E (bench).
PRESSURE=1: rho, J and the pressure tensor."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import Grid, MoverParams
from paper_1904_03684_b200.partition import _CudaArray
grid = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
batches = gem.init_gem_species(grid, 216, pinned=True)
mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
qs = [b.q_per_particle for b in batches]
st = DeviceStore(grid, [b.count() for b in batches], "fast")
field = gem.gem_field(grid) if os.environ.get("FIELD") == "gem" else gem.gem_bench_field(grid)
st.upload_field(field)
for s, b in enumerate(batches): st.upload(s, b.span())
for s in range(4): st.sort(s)
n = sum(b.count() for b in batches)


def disorder():
    ch = rows = nrows = 0
    for s in range(4):
        c = st.count(s)
        x, y, z = [torch.as_tensor(_CudaArray(p, (c,)), device="cuda") for p in st.device_ptrs(s)[:3]]
        key = ((x * (64 / 25.6)).long().clamp(max=63) + 64 * ((y * (64 / 12.8)).long().clamp(max=63)
               + 64 * (z * (32 / 6.4)).long().clamp(max=31)))
        ch += int((key[1:] != key[:-1]).sum())
        m = c // 32 * 32
        r = key[:m].view(-1, 32)
        rows += int((r == r[:, :1]).all(1).sum())
        nrows += r.shape[0]
    return ch / n, rows / nrows


PRESSURE = os.environ.get("PRESSURE") == "1"
st.moments_zero(PRESSURE)   # warm-up: the first deposit call sets the kernel up
for s, b in enumerate(batches): st.deposit(s, b.q_per_particle)
st.sync()
done = 0
for target in (0, 1, 4, 8, 16, 32):
    while done < target:
        st.move_all(mps); done += 1
    st.sync()
    chg, pure = disorder()
    st.moments_zero(PRESSURE)
    st.record(2)
    for s, b in enumerate(batches): st.deposit(s, b.q_per_particle)
    st.record(3)
    st.sync()
    ms = st.elapsed_ms(2, 3)
    print(f"steps since sort {target:3d}: deposit {ms:.3f} ms; cell changes along memory "
          f"order {chg * 100:5.1f} %, rows of 32 in one cell {pure * 100:5.1f} %", flush=True)
