"""C3 (or C4 / C5) state, cell-sorted, then N FAST mover launches, each timed
(for ncu captures of one launch and per-launch times at the large configs).
  python tools/one_launch_big.py N [c3|c4|c5]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1904_03684_b200 import gem
from paper_1904_03684_b200.engine import DeviceStore
from paper_1904_03684_b200.mover import Grid, MoverParams
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = sys.argv[2] if len(sys.argv) > 2 else "c3"
grid, ppc = {"c3": (Grid.make(128, 128, 64, 51.2, 25.6, 12.8), 235),
             "c4": (Grid.make(64, 64, 32, 25.6, 12.8, 6.4), 905),
             "c5": (Grid.make(128, 128, 64, 51.2, 25.6, 12.8), 460)}[cfg]
counts = gem.gem_counts(grid, ppc)
qom, _ = gem.gem_species_params(grid, ppc)
st = DeviceStore(grid, counts, "fast")
st.upload_field(gem.gem_bench_field(grid))
bench.load_gem_chunked(st, grid, ppc)
for s in range(4):
    st.sort(s)
st.sync()
mps = [MoverParams.make(0.1, float(qom[s]), 3) for s in range(4)]
tot = sum(counts)
# per launch: time, SM clock / power / HBM temperature, throttle reasons (NVML)
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:
    h = None
for k in range(n):
    st.record(2); st.move_all(mps); st.record(3)
    ms = st.elapsed_ms(2, 3)
    info = ""
    if h is not None:
        clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        mem = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)
        pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
        t = pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU)
        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        info = f"sm {clk} MHz mem {mem} MHz {pw:.0f} W {t} C reasons 0x{r:x}"
    print(cfg, "launch", k, "%.3f ms" % ms, "%.1f MPA/s" % (tot / ms / 1e3), info, flush=True)
