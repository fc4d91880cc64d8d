"""Mover benchmark: MPA/s on the GEM challenge config (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A *step* is one mover cycle: every particle of the four GEM species advanced
once (pc_iterations = 3, dt = 0.1) on the GEM field -- exactly the work the
reference times as t_mover per cycle (runtime.cpp:227-229).  Particles are
device-resident (the north star's SoA); the field is staged outside the timed
region as in the reference's prefetch engine (engines.cpp:169-173).

N = 1: 64x64x32 cells, 216 ppc -> 61,046,784 particles.
N > 1 (torchrun, one rank per GPU): y-slab partition with per-cycle NCCL
particle migration and count check; weak scaling, ny = 64*N so every GPU holds
a C2-sized slab.

Prints ONE JSON line (rank 0).  `value` is device time (CUDA events) of the K
timed steps, max over ranks; `e2e` goes through the reference-facing engine
API (B200Engine.run_mover) with pinned host batches, host<->device copies
inside the timed region; `cpu_baseline` is the reference's own mover
(oracle/_ref, all host threads) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DT = 0.1
PC = 3
PPC = 216
NX, NY, NZ = 64, 64, 32
LX, LY, LZ = 25.6, 12.8, 6.4
BYTES_PER_PARTICLE = 96  # 48 B read + 48 B write of x,y,z,u,v,w


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """Polls NVML in a thread while the GPU works (SM clock + throttle reasons)."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index: int, period_s: float = 0.0005):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self._err = str(e)
        self.period = period_s

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self._ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        r = [name for bit, name in self.REASONS.items() if self.reasons & bit and bit != 0x1]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples), "reasons": r}


def measured_traffic(mode: str):
    """dram__bytes_read + dram__bytes_write of the mover launch at C2 from the
    committed `ncu --set full` capture (profiles/r01_c2_bench.json), per launch."""
    p = os.path.join(ROOT, "profiles", "r01_c2_bench.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    want = "0>(" if mode == "fast" else "1>("
    for k in d.get("kernels", []):
        if "warp_tile_kernel" in k["kernel"] and want in k["kernel"]:
            rd, wr = k["dram__bytes_read.sum"], k["dram__bytes_write.sum"]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            return float(rd[0]) * scale[rd[1]] + float(wr[0]) * scale[wr[1]]
    return None


def host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return os.cpu_count() or 1, model


# ---------------------------------------------------------------------------
# reference CPU mover (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------

def cpu_mover_setup(grid_t, sample_total, field="gem"):
    """Bounded sample of the GEM workload for the CPU mover: the first
    particles of each species in proportion to the species sizes, generated by
    the reference's own init_gem when it was built (else the C port)."""
    import oracle
    kind = "reference" if os.path.exists(oracle.REF_SO) else "port"
    if kind == "reference":
        parts, E, B = oracle.ref_init_gem(grid_t, PPC)
    else:
        parts = oracle.port_gem_species(grid_t, PPC)
        from paper_1904_03684_b200 import gem as _g  # field only (host generator)
        from paper_1904_03684_b200.mover import Grid
        f = _g.gem_field(Grid.make(*grid_t))
        E, B = f.E.ravel().copy(), f.B.ravel().copy()
    if field == "gem+E":
        E, _ = oracle.port_gem_like_field(grid_t)
    total = sum(len(p[0]) for p in parts)
    frac = min(1.0, sample_total / total)
    qoms = [-25.0, 1.0, -25.0, 1.0]
    sample = []
    for s, p in enumerate(parts):
        m = max(1, int(len(p[0]) * frac))
        sample.append(([a[:m].copy() for a in p], qoms[s]))
    return kind, sample, E, B, total


def cpu_mover_step(kind, sample, E, B, grid_t, threads):
    import oracle
    n = 0
    t0 = time.perf_counter()
    for p6, qom in sample:
        if kind == "reference":
            oracle.ref_move_batch(p6, E, B, grid_t, DT, qom, PC, threads=threads)
        else:
            oracle.port_move_batch(p6, E, B, grid_t, DT, qom, PC)
        n += len(p6[0])
    return n, time.perf_counter() - t0


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads, model = host_info()
    grid_t = (NX, NY, NZ, LX, LY, LZ)
    kind, sample, E, B, total = cpu_mover_setup(grid_t, sample_total=2_000_000 * threads,
                                                field=args.field)
    if kind == "port":
        threads = 1
    n_s = sum(len(p[0][0]) for p in sample)
    for _ in range(args.warmup):
        cpu_mover_step(kind, sample, E, B, grid_t, threads)
    times = []
    for _ in range(args.steps):
        n, t = cpu_mover_step(kind, sample, E, B, grid_t, threads)
        times.append(t)
    mean = sum(times) / len(times)
    value = n_s / mean / 1e6
    line = {
        "impl": "reference", "metric": "MPA/s in mover", "value": value, "unit": "MPA/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": mean * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic GEM (reference init_gem)",
        "config": {"workload": "GEM 64x64x32, 216 ppc, 4 species, pc 3, dt 0.1 (C2)",
                   "particles_total": total, "sample_particles_per_step": n_s},
        "cpu_baseline": {"value": value, "unit": "MPA/s", "cores": threads, "kind": kind,
                         "cpu_model": model,
                         "sample": f"first {n_s} of {total} GEM particles (species-proportional), "
                                   f"pic::move_batch on {threads} threads over disjoint spans"},
        "e2e": {"value": value, "unit": "MPA/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    from paper_1904_03684_b200 import _capi, gem
    from paper_1904_03684_b200.engine import B200Engine, DeviceStore
    from paper_1904_03684_b200.mover import Grid, MoverParams

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # B2M_SLAB_PATH=1 runs the partition-layer step (mover fused with the
    # owner scan + compaction + exchange + count all-reduce) even at N = 1, to
    # measure what the multi-GPU step adds over the plain mover
    if world > 1 or os.environ.get("B2M_SLAB_PATH") == "1":
        from paper_1904_03684_b200 import partition
        return partition.bench_world(args)

    torch.cuda.set_device(local)
    lib = _capi.lib()
    grid = Grid.make(NX, NY, NZ, LX, LY, LZ)
    t_init = time.perf_counter()
    batches = gem.init_gem_species(grid, PPC, pinned=True)
    t_init = time.perf_counter() - t_init
    field = gem.gem_field(grid) if args.field == "gem" else gem.gem_bench_field(grid)
    n_total = sum(b.count() for b in batches)
    mps = [MoverParams.make(DT, b.qom, PC) for b in batches]

    store = DeviceStore(grid, [b.count() for b in batches], args.mode, device=local)
    store.upload_field(field)
    for s, b in enumerate(batches):
        store.upload(s, b.span())
    if args.sort:
        for s in range(len(batches)):
            store.sort(s)
    store.sync()

    # ---- device-resident timed region ----
    # Work runs on torch's current stream so torch events can bracket every
    # launch.  A step = one mover cycle over all species; every `resort`
    # steps the step also re-sorts every species by cell (the optional
    # cell-sort pass) -- its cost is inside the timed region.
    stream = torch.cuda.Stream()           # a real stream handle (the legacy default is 0)
    torch.cuda.set_stream(stream)
    store.set_stream(stream.cuda_stream)
    step_no = [0]

    def step():
        if args.resort and step_no[0] % args.resort == 0:
            for s in range(len(batches)):
                store.sort(s)
        store.move_all(mps)
        step_no[0] += 1

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    store.sync()
    launches0 = lib.b2m_launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record()
        for k in range(args.steps):
            if args.resort and step_no[0] % args.resort == 0:
                for s in range(len(batches)):
                    store.sort(s)
            ev[k][0].record()
            store.move_all(mps)
            ev[k][1].record()
            step_no[0] += 1
        t1.record()
        torch.cuda.synchronize()
    store.sync()
    total_ms = t0.elapsed_time(t1)
    launches = lib.b2m_launch_count() - launches0
    ms = total_ms / args.steps
    value = n_total / (ms * 1e-3) / 1e6
    # the mover launch alone (events bracket exactly the one move_all launch)
    mover_ms = [a.elapsed_time(b) for a, b in ev]
    kernel_ms = sum(mover_ms) / len(mover_ms)
    sort_share = 1.0 - sum(mover_ms) / total_ms

    # STRICT (bit-exact) mode on the same resident state, for reference
    strict_value = None
    if args.strict_too:
        store.set_mode("strict")
        store.move_all(mps)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            store.move_all(mps)
        b.record()
        torch.cuda.synchronize()
        strict_value = n_total / (a.elapsed_time(b) / 3 * 1e-3) / 1e6
        store.sync()
        store.set_mode(args.mode)

    # Moment deposition (deposit_moments, kernels.cpp:147-183)
    # of the resident state after the timed steps, rho + J for all species
    moments = None
    if args.moments:
        def deposit_ms():
            store.moments_zero(False)
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for s, b in enumerate(batches):
                store.deposit(s, b.q_per_particle)
            b_.record()
            torch.cuda.synchronize()
            store.sync()
            return a.elapsed_time(b_)
        deposit_ms()  # warm-up
        drifted = deposit_ms()   # the state the timed steps left (drifted since the last sort)
        for s in range(len(batches)):
            store.sort(s)
        fresh = deposit_ms()     # right after a cell sort
        moments = {"value": n_total / (fresh * 1e-3) / 1e6, "unit": "MPA/s", "ms": fresh,
                   "what": "deposit_moments rho+J, all species, device-resident C2 state right "
                           "after a cell sort",
                   "ms_drifted": drifted,
                   "drifted_what": "the same on the state left by the timed steps (particles "
                                   "drifted out of cell order: more per-run mesh updates)",
                   "hbm_frac": 48 * n_total / (fresh * 1e-3) / 1e9 / load_peaks()[0]}
    store.close()

    peak, peak_src = load_peaks()
    alg_bytes = BYTES_PER_PARTICLE * n_total
    achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9

    # ---- e2e through the reference-facing engine API, host batches ----
    e2e = None
    if args.e2e_steps > 0:
        eng = B200Engine(grid, mode=args.mode, schedule="pipeline")
        eng.prime(field, batches)
        eng.run_mover(field, batches, mps)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev0 = torch.cuda.Event(enable_timing=True)
        for _ in range(args.e2e_steps):
            eng.run_mover(field, batches, mps)
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        e2e = {"value": n_total / e2e_s / 1e6, "unit": "MPA/s",
               "h2d_bytes_per_step": alg_bytes // 2 + 2 * 24 * grid.nodes(),
               "d2h_bytes_per_step": alg_bytes // 2,
               "ms_per_step": e2e_s * 1e3,
               "path": "B200Engine.run_mover (pic::Engine contract) with pinned host batches; "
                       "chunked H2D / kernel / D2H on three streams"}
        eng.close()

    # ---- CPU baseline (reference mover on host cores, bounded sample) ----
    cpu = None
    if args.cpu_baseline:
        threads, model = host_info()
        grid_t = grid.as_tuple()
        kind, sample, E, B, total = cpu_mover_setup(grid_t, sample_total=1_000_000 * threads,
                                                    field=args.field)
        if kind == "port":
            threads = 1
        n_s, t = cpu_mover_step(kind, sample, E, B, grid_t, threads)
        cpu = {"value": n_s / t / 1e6, "unit": "MPA/s", "cores": threads, "kind": kind,
               "cpu_model": model,
               "sample": f"first {n_s} of {total} GEM particles (species-proportional), one "
                         f"mover cycle, pic::move_batch on {threads} threads"}

    line = {
        "metric": "MPA/s in mover", "value": value, "unit": "MPA/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic GEM state bit-identical to the reference's init_gem (seed 12345): "
                 "Harris B, E = 0, as the reference's own run_benchmark sees it")
                if args.field == "gem" else
                "synthetic GEM particles (reference init_gem) + gem_like_field E",
        "config": {"workload": "GEM 64x64x32, 216 ppc, 4 species (C2), pc 3, dt 0.1",
                   "particles": n_total, "mode": args.mode,
                   "cell_sort": f"every {args.resort} steps, inside the timed region"
                                if args.resort else "once before timing",
                   "l2": "inputs larger than L2 (2.93 GB SoA vs 126 MB)",
                   "parallelism": "single GPU"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": args.traffic if args.traffic is not None
                                else measured_traffic(args.mode),
                     "traffic_source": "ncu --set full, profiles/r01_c2_bench.json",
                     "kernel": "warp_tile_kernel<4,0> (FAST)" if args.mode == "fast"
                               else "warp_tile_kernel<4,1> (STRICT)",
                     "kernel_ms": kernel_ms, "bytes_per_launch": alg_bytes,
                     "sort_share_of_step": sort_share,
                     "peak_source": peak_src},
        # the resource that actually binds this kernel: FP64 dependency
        # latency at 12 warps/SM (profiles/README.md).  225 FP64 instructions
        # per particle (ncu, FAST) against the FP64 FMA rate measured by
        # tools/micro/dfma.cu (56 lane-ops/clk/SM x 148 SMs x 1.965 GHz)
        "fp64_pipe": ({"ops_per_particle": 225, "achieved_tops": 225 * n_total / (kernel_ms * 1e-3)
                       / 1e12, "peak_tops": 56 * 148 * 1.965e9 / 1e12,
                       "frac": 225 * n_total / (kernel_ms * 1e-3) / (56 * 148 * 1.965e9),
                       "peak_source": "tools/micro/dfma.cu on this B200 (FP64 FMA, ILP 8)"}
                      if args.mode == "fast" else None),
        "clocks": clk.summary(),
        "e2e": e2e,
        "cpu_baseline": cpu,
        "strict_value": strict_value,
        "moments": moments,
        "init_s": t_init,
    }
    print(json.dumps(line), flush=True)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="fast", choices=["fast", "strict"])
    ap.add_argument("--sort", type=int, default=1, help="cell-sort species once before timing")
    ap.add_argument("--resort", type=int, default=32,
                    help="re-sort every N steps inside the timed region (0: never)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-baseline", type=int, default=1)
    ap.add_argument("--strict-too", type=int, default=1)
    ap.add_argument("--moments", type=int, default=1)
    ap.add_argument("--field", default="gem", choices=["gem", "gem+E"],
                    help="gem: the reference's init_gem field (E=0, static B) that its own "
                         "benchmark moves particles in; gem+E: add the gem_like_field E")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per launch from an ncu --set full capture")
    args = ap.parse_args(argv)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
