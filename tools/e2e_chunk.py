import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import B200Engine
from paper_1904_03684_b200.mover import Grid, MoverParams
g = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
batches = gem.init_gem_species(g, 216, pinned=True)
field = gem.gem_field(g)
mps = [MoverParams.make(0.1, b.qom, 3) for b in batches]
n = sum(b.count() for b in batches)
for ch in (1 << 20, 1 << 21, 1 << 22, 1 << 23):
    eng = B200Engine(g, mode="fast", schedule="pipeline", chunk=ch)
    eng.prime(field, batches)
    eng.run_mover(field, batches, mps)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        eng.run_mover(field, batches, mps)
    dt = (time.perf_counter() - t) / 3
    print(f"chunk {ch}: {dt*1e3:.1f} ms/step  {n/dt/1e6:.0f} MPA/s", flush=True)
    eng.close()
