"""Diagnostics: per-launch device time vs clocks/power (NVML) on C2 species 0."""
import os, sys, time, threading, statistics, functools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml, torch
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import Grid, MoverParams

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()
def poll():
    while not stop.is_set():
        samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h),
                        pynvml.nvmlDeviceGetPerformanceState(h)))
        time.sleep(0.002)
th = threading.Thread(target=poll, daemon=True); th.start()

x = torch.empty(2**28, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); [y.copy_(x) for _ in range(10)]; e1.record(); torch.cuda.synchronize()
print(f"torch copy: {2*8*2**28*10/e0.elapsed_time(e1)/1e6:.0f} GB/s")
del x, y

mode = sys.argv[1] if len(sys.argv) > 1 else "fast"
fieldkind = sys.argv[2] if len(sys.argv) > 2 else "gem"
grid = Grid.make(64, 64, 32, 25.6, 12.8, 6.4)
b = gem.init_gem_species(grid, 216, pinned=True, species=(0,))[0]
field = gem.gem_field(grid) if fieldkind == "gem" else gem.gem_bench_field(grid)
mp = MoverParams.make(0.1, b.qom, 3)
st = DeviceStore(grid, [b.count()], mode)
st.upload_field(field); st.upload(0, b.span()); st.sync()
t_start = time.perf_counter()
res = []
for i in range(40):
    st.record(0); st.move(0, mp); st.record(1)
    res.append((time.perf_counter(), st.elapsed_ms(0, 1)))
time.sleep(2.0)
for i in range(3):
    st.record(0); st.move(0, mp); st.record(1)
    res.append((time.perf_counter(), st.elapsed_ms(0, 1)))
    time.sleep(1.0)
stop.set(); th.join()
print("per-launch ms:", " ".join(f"{m:.2f}" for _, m in res))
busy = [s for s in samples if s[0] >= t_start]
print("sm clocks during:", sorted(set(s[1] for s in busy)))
print("mem clocks during:", sorted(set(s[2] for s in busy)))
print("power W max/median:", max(s[3] for s in busy), statistics.median(s[3] for s in busy))
print("reasons OR:", hex(functools.reduce(lambda a, s: a | s[4], busy, 0)), "pstates", sorted(set(s[5] for s in busy)))
