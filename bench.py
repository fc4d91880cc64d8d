"""Mover benchmark: MPA/s on the GEM challenge config (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A *step* is one mover cycle: every particle of the four GEM species advanced
once (pc_iterations = 3, dt = 0.1) -- the work the reference times as t_mover
per cycle (runtime.cpp:227-229) -- preceded by the cycle's field change (the
field buffers marked rewritten, so the mover's derived gather tables and the
field's z-invariance test are redone inside the step).  Particles are
device-resident (the north star's SoA).

N = 1: 64x64x32 cells, 216 ppc -> 61,046,784 particles, field
= init_gem's Harris B + the gem_like_field E (test_offload.cpp:60-71).
N > 1: one rank per GPU over NCCL.  `--gpus N` launches the N ranks itself
(torch.distributed.run) when it is not already under torchrun.  Weak scaling
headline: y-slab partition (runtime.cpp:22-76), every rank a C2-sized slab,
per cycle the field broadcast (runtime.cpp:143) + mover + NCCL particle
migration + count check; plus a C4 strong-scaling leg (255.8M
particles, fixed, on 1 and on N GPUs, efficiency S/N as bench.cpp:53-59).

Prints ONE JSON line (rank 0).  `value` is device time (CUDA events) of the K
timed steps, max over ranks; it equals the harmonic mean of the per-repetition
MPA/s over the timed repetitions of 10 cycles (bench.cpp:13-45; the warm-up
steps play the dropped first repetition).  `e2e` goes through the
reference-facing engine API (B200Engine.run_mover) with pinned host batches,
host<->device copies inside the timed region; `cpu_baseline` is the
reference's own mover (oracle/_ref, all host threads) on the same bounded
sample and field as the `--impl reference` arm.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DT = 0.1
PC = 3
PPC = 216
NX, NY, NZ = 64, 64, 32
LX, LY, LZ = 25.6, 12.8, 6.4
C4_PPC = 905           # 64x64x32 cells, 255,774,720 particles
C3_GRID = (128, 128, 64, 51.2, 25.6, 12.8)   # SURVEY §8d C3 (BASELINE configs[2])
C3_PPC = 235                                 # -> 512,081,920 particles
BYTES_PER_PARTICLE = 96  # 48 B read + 48 B write of x,y,z,u,v,w
REP_CYCLES = 10          # cycles per repetition (bench.cpp:13-45)
CPU_SAMPLE_PER_THREAD = 2_000_000


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
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


PROFILE = os.path.join(ROOT, "profiles", "r02_c2_bench.json")


def measured_traffic(kernel_tag: str):
    """dram__bytes_read + dram__bytes_write per launch of the kernel whose ncu
    name contains `kernel_tag`, from the committed `ncu --set full` capture of
    this round (profiles/r02_c2_bench.json)."""
    if not os.path.exists(PROFILE):
        return None
    with open(PROFILE) as f:
        d = json.load(f)
    for k in d.get("kernels", []):
        if kernel_tag in k["kernel"]:
            rd, wr = k["dram__bytes_read.sum"], k["dram__bytes_write.sum"]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            return float(rd[0]) * scale[rd[1]] + float(wr[0]) * scale[wr[1]]
    return None


def measured_ncu(kernel_tag: str):
    """FP64-pipe / issue / occupancy figures of the same ncu capture
    (profiles/r02_c2_bench.json) for the kernel whose name contains
    `kernel_tag` -- the regime the roofline fraction sits in."""
    if not os.path.exists(PROFILE):
        return None
    with open(PROFILE) as f:
        d = json.load(f)
    keys = {"fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
            "registers": "launch__registers_per_thread",
            "ncu_ms": "gpu__time_duration.sum"}
    for k in d.get("kernels", []):
        if kernel_tag in k["kernel"]:
            return {name: float(k[m][0]) for name, m in keys.items() if m in k}
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


def harmonic_reps(step_ms, particles, rep=REP_CYCLES):
    """Per-repetition MPA/s over consecutive groups of `rep` timed cycles and
    their harmonic mean (bench.cpp:13-45); equal work per repetition, so the
    harmonic mean is total particles / total time."""
    reps = [step_ms[i:i + rep] for i in range(0, len(step_ms), rep)]
    mpas = [particles * len(r) / (sum(r) * 1e-3) / 1e6 for r in reps if r]
    hm = len(mpas) / sum(1.0 / m for m in mpas) if mpas else None
    return {"cycles_per_rep": rep, "mpas": mpas, "harmonic_mean": hm}


# ---------------------------------------------------------------------------
# the reference CPU mover (the --impl reference arm and our cpu_baseline key)
# ---------------------------------------------------------------------------

def cpu_mover_setup(grid_t, sample_total, field="gem+E"):
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
        sample.append(([a[:m].copy() if m < len(a) else a for a in p], qoms[s]))
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


def cpu_reference_measure(field, steps, warmup, whole_budget_s=0.0):
    """The reference's pic::move_batch (oracle/_ref: its own sources, all host
    threads over disjoint spans) on a bounded species-proportional sample of
    the C2 state: `warmup` untimed then `steps` timed cycles of the sample.
    Used by both the reference arm and our line's cpu_baseline, so the two
    report the same method and field.  whole_budget_s > 0: the WHOLE C2 state
    when (warmup + steps) cycles of it are estimated to fit that many seconds
    (~5 M particles/s per host thread)."""
    threads, model = host_info()
    grid_t = (NX, NY, NZ, LX, LY, LZ)
    n_sample = CPU_SAMPLE_PER_THREAD * threads
    if whole_budget_s > 0 and (warmup + max(1, steps)) * 61046784 / (5e6 * threads) <= whole_budget_s:
        n_sample = 1 << 62
    kind, sample, E, B, total = cpu_mover_setup(grid_t, n_sample, field=field)
    if kind == "port":
        threads = 1
    n_s = sum(len(p[0][0]) for p in sample)
    for _ in range(warmup):
        cpu_mover_step(kind, sample, E, B, grid_t, threads)
    times = [cpu_mover_step(kind, sample, E, B, grid_t, threads)[1] for _ in range(max(1, steps))]
    mean = sum(times) / len(times)
    return {"value": n_s / mean / 1e6, "unit": "MPA/s", "cores": threads, "kind": kind,
            "cpu_model": model, "ms_per_step": mean * 1e3, "steps": len(times),
            "particles_total": total, "sampled": n_s,
            "sample": (f"the whole C2 state ({total} GEM particles)" if n_s == total else
                       f"first {n_s} of {total} C2 GEM particles (species-proportional, "
                       f"{CPU_SAMPLE_PER_THREAD} per thread)") + f", field {field}, "
                      f"pic::move_batch on {threads} threads over disjoint spans, "
                      f"{warmup} warm-up + {len(times)} timed cycles"}


def reference_simulation_measure(field, cycles=3):
    """SURVEY §8(d) CPU baseline (i): the reference's own pic::Simulation
    (runtime.cpp, the path bench.cpp's run_benchmark times) with the cpu
    engine on the whole C2 state and field, workers = the largest divisor of
    ny not above the host's threads (runtime.cpp:24-30); MPA/s from the mean
    per-cycle t_mover (max over workers, bench.cpp:78-81).  None when the
    reference library was not built."""
    import oracle
    if not os.path.exists(oracle.REF_SO):
        return None
    threads, model = host_info()
    grid_t = (NX, NY, NZ, LX, LY, LZ)
    workers = max(w for w in range(1, min(threads, NY // 2) + 1) if NY % w == 0 and NY // w >= 2)
    parts, E, B = oracle.ref_init_gem(grid_t, PPC)
    if field == "gem+E":
        E, _ = oracle.port_gem_like_field(grid_t)
    total = sum(len(p[0]) for p in parts)
    t0 = time.perf_counter()
    sim = oracle.RefSimulation(grid_t, PPC, workers=workers, engine="cpu", pc=PC, dt=DT,
                               inject=(parts, E, B))
    sim.run(cycles)
    t_mover = sim.mean_mover_s()
    wall = time.perf_counter() - t0
    del sim
    return {"value": total / t_mover / 1e6, "unit": "MPA/s", "workers": workers,
            "cycles": cycles, "t_mover_s": t_mover, "wall_s": wall, "cpu_model": model,
            "what": f"pic::Simulation (cpu engine, {workers} workers) on the whole C2 state "
                    f"({total} particles), field {field}; MPA/s = particles / mean per-cycle "
                    f"t_mover (max over workers), as bench.cpp's run_benchmark reports"}


def run_reference_arm(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    cpu = cpu_reference_measure(args.field, args.steps, args.warmup, whole_budget_s=240.0)
    try:
        sim = reference_simulation_measure(args.field) if args.ref_sim else None
    except Exception as e:  # noqa: BLE001 - an extra figure; the arm's value stands
        sim = {"unavailable": f"{type(e).__name__}: {e}"}
    whole = cpu.get("sampled") == cpu["particles_total"]
    line = {
        "impl": "reference", "metric": "MPA/s in mover", "value": cpu["value"], "unit": "MPA/s",
        "n_gpus": args.gpus, "steps": cpu["steps"], "warmup": args.warmup,
        "ms_per_step": cpu["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic GEM (reference init_gem) + gem_like_field E" if args.field == "gem+E"
                else "synthetic GEM (reference init_gem), E = 0",
        "config": {"workload": "GEM 64x64x32, 216 ppc, 4 species, pc 3, dt 0.1 (C2)",
                   "particles_total": cpu["particles_total"], "same_config": whole,
                   "note": ("the whole C2 state every step" if whole else
                            "a bounded sample of the C2 state per step (the whole state would "
                            "not fit the run's time budget); same metric, unit and field")},
        "cpu_baseline": cpu,
        "reference_simulation": sim,
        "e2e": {"value": cpu["value"], "unit": "MPA/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm, one GPU
# ---------------------------------------------------------------------------

def time_steps(store, mps, steps, refresh, events):
    """`steps` cycles, each: the field marked changed (z-invariance test and
    gather tables rebuilt inside the move call) then the mover over all
    species, enqueued back to back without host syncs.  With events: per step
    (step ms, mover-kernel ms) from CUDA events on the launching stream --
    torch's current stream around the step, the library's kernel-timing log
    (b2m_kernel_timing_*) around the mover launches alone."""
    import torch
    ev = []
    if events:
        store.kernel_timing_begin(steps)
    for _ in range(steps):
        if events:
            e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            e[0].record()
        if refresh:
            store.field_changed()
        store.move_all(mps)
        if events:
            e[1].record()
            ev.append(e)
    if not events:
        return []
    kms = store.kernel_timing_read(steps)
    return [(a.elapsed_time(b), k) for (a, b), k in zip(ev, kms)]


def fused_cycle(store, mps, qs, ns, reps=3, drift=32):
    """Mover + moment deposition (rho, J) of all species: one fused launch
    (b2m_move_deposit_all: the deposit from the mover's shared-memory tile
    through FP64 DMMA) against b2m_move_all + b2m_deposit per species and
    against the plain mover, right after a cell sort and `drift` cycles
    later.  Every call advances the state one cycle; the three are
    interleaved so they see the same drift."""
    import torch

    def timed(fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    def mover():
        store.move_all(mps)

    def separate():
        store.moments_zero(False)
        store.move_all(mps)
        for s in range(ns):
            store.deposit(s, qs[s])

    def fused():
        store.moments_zero(False)
        store.move_deposit_all(mps, qs)

    def measure():
        t = {"mover": [], "separate": [], "fused": []}
        for _ in range(reps):
            t["mover"].append(timed(mover))
            t["separate"].append(timed(separate))
            t["fused"].append(timed(fused))
        store.sync()
        return {k: sum(v) / len(v) for k, v in t.items()}

    for s in range(ns):
        store.sort(s)
    fused()  # warm-up
    store.sync()
    fresh = measure()
    for _ in range(drift):
        store.move_all(mps)
    drifted = measure()
    return {"fresh_ms": fresh, f"after_{drift}_cycles_ms": drifted,
            "what": "ms per cycle of all C2 species: 'mover' = b2m_move_all alone; "
                    "'separate' = b2m_move_all + b2m_deposit (rho, J) per species; 'fused' = "
                    "b2m_move_deposit_all (one launch, deposit from the mover's tile via FP64 "
                    "DMMA); fresh = right after a cell sort"}


def load_gem_chunked(store, grid, ppc, chunk=1 << 24):
    """The reference GEM state straight into a device store without holding it
    on the host: background species generated in index ranges by the
    counter-RNG jump-ahead and uploaded chunk by chunk, the (domain-size
    independent) sheet species whole."""
    import ctypes as C
    import numpy as np
    from paper_1904_03684_b200 import _capi, gem
    counts = gem.gem_counts(grid, ppc)
    g = grid.to_c()
    for s in range(4):
        if s >= 2:
            b = gem.init_gem_species(grid, ppc, species=(s,))[0]
            store.upload(s, b.span())
            continue
        for m0 in range(0, counts[s], chunk):
            m1 = min(counts[s], m0 + chunk)
            arrs = [np.empty(m1 - m0) for _ in range(6)]
            _capi.check(_capi.lib().b2m_gem_fill_species_range(
                C.byref(g), ppc, gem.DEFAULT_SEED, s, m0, m1, _capi.ptr6(arrs), 0))
            _capi.check(_capi.lib().b2m_species_upload_range(store.h, s, _capi.ptr6(arrs), m0,
                                                             m1 - m0))
        _capi.check(_capi.lib().b2m_species_set_count(store.h, s, counts[s]))
    store.sync()
    return counts


def c3_single_gpu(args, local, field_kind):
    """SURVEY C3 (BASELINE configs[2]: 128x128x64 cells, 235 ppc, 512,081,920
    particles, 24.6 GB of SoA) on this one GPU: field refresh + mover, the
    same step as the headline."""
    import torch
    from paper_1904_03684_b200 import gem
    from paper_1904_03684_b200.engine import DeviceStore
    from paper_1904_03684_b200.mover import Grid, MoverParams
    grid = Grid.make(*C3_GRID)
    t0 = time.perf_counter()
    counts = gem.gem_counts(grid, C3_PPC)
    qom, _ = gem.gem_species_params(grid, C3_PPC)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    store = DeviceStore(grid, counts, args.mode, device=local)
    store.set_stream(stream.cuda_stream)
    store.upload_field(gem.gem_bench_field(grid) if field_kind == "gem+E" else gem.gem_field(grid))
    load_gem_chunked(store, grid, C3_PPC)
    t_init = time.perf_counter() - t0
    for s in range(4):
        store.sort(s)
    mps = [MoverParams.make(DT, float(qom[s]), PC) for s in range(4)]
    time_steps(store, mps, args.warmup, True, False)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev = time_steps(store, mps, args.steps, True, True)
        torch.cuda.synchronize()
    store.sync()
    store.close()
    n = sum(counts)
    ms = sum(t for t, k in ev) / len(ev)
    kms = sum(k for t, k in ev) / len(ev)
    peak, _ = load_peaks()
    return {"particles": n, "n_gpus": 1, "ms_per_step": ms, "value": n / (ms * 1e-3) / 1e6,
            "unit": "MPA/s", "kernel_ms": kms,
            "roofline_frac": BYTES_PER_PARTICLE * n / (kms * 1e-3) / 1e9 / peak,
            "step_ms": [round(t, 4) for t, k in ev], "clocks": clk.summary(),
            "init_s": t_init,
            "workload": "GEM 128x128x64, L = (51.2, 25.6, 12.8), 235 ppc (SURVEY C3, BASELINE "
                        "configs[2]) on one GPU: field refresh + mover"}


def c4_single_gpu(args, local, field_kind):
    """SURVEY C4 (255.8M particles) on this one GPU: the strong-scaling
    baseline T1 (plain mover + field refresh, no exchange)."""
    import torch
    from paper_1904_03684_b200 import gem
    from paper_1904_03684_b200.engine import DeviceStore
    from paper_1904_03684_b200.mover import Grid, MoverParams
    grid = Grid.make(NX, NY, NZ, LX, LY, LZ)
    t0 = time.perf_counter()
    batches = gem.init_gem_species(grid, C4_PPC, pinned=True)
    t_init = time.perf_counter() - t0
    field = gem.gem_bench_field(grid) if field_kind == "gem+E" else gem.gem_field(grid)
    n = sum(b.count() for b in batches)
    mps = [MoverParams.make(DT, b.qom, PC) for b in batches]
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    store = DeviceStore(grid, [b.count() for b in batches], args.mode, device=local)
    store.set_stream(stream.cuda_stream)
    store.upload_field(field)
    for s, b in enumerate(batches):
        store.upload(s, b.span())
        store.sort(s)
    del batches
    time_steps(store, mps, args.warmup, True, False)
    torch.cuda.synchronize()
    ev = time_steps(store, mps, args.steps, True, True)
    torch.cuda.synchronize()
    store.sync()
    store.close()
    step_ms = [t for t, k in ev]
    ms = sum(step_ms) / len(step_ms)
    return {"particles": n, "n_gpus": 1, "ms_per_step": ms, "value": n / (ms * 1e-3) / 1e6,
            "unit": "MPA/s", "init_s": t_init,
            "workload": "GEM 64x64x32, 905 ppc (SURVEY C4), one GPU, field refresh + mover"}


def run_ours(args):
    import torch
    from paper_1904_03684_b200 import _capi, gem
    from paper_1904_03684_b200.engine import B200Engine, DeviceStore
    from paper_1904_03684_b200.mover import Grid, MoverParams

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    lib = _capi.lib()
    grid = Grid.make(NX, NY, NZ, LX, LY, LZ)
    t_init = time.perf_counter()
    batches = gem.init_gem_species(grid, PPC, pinned=True)
    t_init = time.perf_counter() - t_init
    field = gem.gem_bench_field(grid) if args.field == "gem+E" else gem.gem_field(grid)
    n_total = sum(b.count() for b in batches)
    mps = [MoverParams.make(DT, b.qom, PC) for b in batches]

    store = DeviceStore(grid, [b.count() for b in batches], args.mode, device=local)
    stream = torch.cuda.Stream()           # a real stream handle (the legacy default is 0)
    torch.cuda.set_stream(stream)
    store.set_stream(stream.cuda_stream)

    def load_state(f):
        store.upload_field(f)
        for s, b in enumerate(batches):
            store.upload(s, b.span())
            if args.sort:
                store.sort(s)
        store.sync()

    load_state(field)

    # ---- device-resident timed region: K cycles of (field refresh + mover) ----
    time_steps(store, mps, args.warmup, args.refresh, False)
    torch.cuda.synchronize()
    store.sync()
    launches0 = lib.b2m_launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record()
        ev = time_steps(store, mps, args.steps, args.refresh, True)
        t1.record()
        torch.cuda.synchronize()
    store.sync()
    total_ms = t0.elapsed_time(t1)
    launches = lib.b2m_launch_count() - launches0
    ms = total_ms / args.steps
    value = n_total / (ms * 1e-3) / 1e6
    step_ms = [t for t, k in ev]
    mover_ms = [k for t, k in ev]
    kernel_ms = sum(mover_ms) / len(mover_ms)
    reps = harmonic_reps(step_ms, n_total)
    peak, peak_src = load_peaks()
    alg_bytes = BYTES_PER_PARTICLE * n_total

    # Moment deposition (deposit_moments, kernels.cpp:147-183)
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
        drifted = deposit_ms()   # the state the steps above left (drifted since the last sort)
        for s in range(len(batches)):
            store.sort(s)
        fresh = deposit_ms()     # right after a cell sort
        moments = {"value": n_total / (fresh * 1e-3) / 1e6, "unit": "MPA/s", "ms": fresh,
                   "what": "deposit_moments rho+J, all species, device-resident C2 state right "
                           "after a cell sort",
                   "ms_drifted": drifted,
                   "drifted_what": "the same on the state the timed steps left",
                   "hbm_frac": 48 * n_total / (fresh * 1e-3) / 1e9 / peak,
                   "fused": fused_cycle(store, mps, [b.q_per_particle for b in batches],
                                        len(batches)) if args.mode == "fast" else None}
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

    # ---- the general 3-D kernel on the same particles, z-varying field ----
    general = None
    if args.general_3d and args.mode == "fast":
        load_state(gem.gem_bench_field(grid, z_varying=True))
        time_steps(store, mps, args.warmup, args.refresh, False)
        g_steps = min(args.steps, 10)
        gev = time_steps(store, mps, g_steps, args.refresh, True)
        torch.cuda.synchronize()
        store.sync()
        g_ms = [k for t, k in gev]
        g_step = [t for t, k in gev]
        gk = sum(g_ms) / len(g_ms)
        general = {"value": n_total / (sum(g_step) / len(g_step) * 1e-3) / 1e6, "unit": "MPA/s",
                   "kernel": "warp_tile_kernel<4,0,3,0> (FAST, general trilinear gather)",
                   "kernel_ms": gk, "steps": g_steps,
                   "roofline_frac": alg_bytes / (gk * 1e-3) / 1e9 / peak,
                   "traffic": measured_traffic("<4, 0, 3, 0>"),
                   "field": "the bench field + Ez 1e-3 sin(2 pi z/lz) (not z-invariant), same "
                            "particles, re-sorted, after the same warm-up"}

    store.close()

    # ---- e2e through the reference-facing engine API, host batches ----
    e2e = None
    if args.e2e_steps > 0:
        eng = B200Engine(grid, mode=args.mode, schedule="pipeline")
        eng.prime(field, batches)
        eng.run_mover(field, batches, mps)  # warm-up
        torch.cuda.synchronize()
        e2e_t = []
        for _ in range(args.e2e_steps):
            t = time.perf_counter()
            eng.run_mover(field, batches, mps)
            e2e_t.append(time.perf_counter() - t)
        e2e_s = sum(e2e_t) / len(e2e_t)
        e2e = {"value": n_total / e2e_s / 1e6, "unit": "MPA/s",
               "h2d_bytes_per_step": alg_bytes // 2 + 2 * 24 * grid.nodes(),
               "d2h_bytes_per_step": alg_bytes // 2,
               "ms_per_step": e2e_s * 1e3, "steps": len(e2e_t),
               "step_ms": [t * 1e3 for t in e2e_t],
               "path": "B200Engine.run_mover (pic::Engine contract) with pinned host batches; "
                       "chunked H2D / kernel / D2H on three streams (PCIe-bound)"}
        eng.close()
    del batches

    # ---- strong-scaling baseline (C4 on this GPU) ----
    strong = c4_single_gpu(args, local, args.field) if args.strong else None
    c3 = c3_single_gpu(args, local, args.field) if args.c3 else None

    # ---- CPU baseline: the reference arm's own measurement ----
    cpu = cpu_reference_measure(args.field, 2, 1, whole_budget_s=30.0) if args.cpu_baseline else None

    kname = "warp_tile_kernel<4,0,2,0> (FAST, z-invariant column gather)" \
        if args.mode == "fast" and args.field in ("gem", "gem+E") else "warp_tile_kernel"
    line = {
        "metric": "MPA/s in mover", "value": value, "unit": "MPA/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic GEM state bit-identical to the reference's init_gem (seed 12345) "
                 "+ gem_like_field E (SURVEY §8d)") if args.field == "gem+E" else
                "synthetic GEM state (reference init_gem), E = 0",
        "config": {"workload": "GEM 2-D-in-3-D, 64x64x32 cells, 216 ppc, 4 species (C2), "
                               "pc 3, dt 0.1",
                   "particles": n_total, "mode": args.mode, "field": args.field,
                   "step": "field marked rewritten (z-invariance test + gather tables rebuilt) "
                           "+ mover over all species" if args.refresh else "mover over all species",
                   "cell_sort": "once, before the warm-up (not in the timed region)"
                                if args.sort else "never (init_gem order)",
                   "l2": "inputs larger than L2 (2.93 GB SoA vs 126 MB)",
                   "parallelism": "single GPU"},
        "repetitions": reps,
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": alg_bytes / (kernel_ms * 1e-3) / 1e9,
                     "peak": peak, "unit": "GB/s",
                     "frac": alg_bytes / (kernel_ms * 1e-3) / 1e9 / peak,
                     "traffic": measured_traffic("<4, 0, 2, 0>") if args.mode == "fast" else None,
                     "ncu": measured_ncu("<4, 0, 2, 0>") if args.mode == "fast" else None,
                     "traffic_source": "ncu --set full, profiles/r02_c2_bench.json",
                     "kernel": kname, "kernel_ms": kernel_ms,
                     "bytes_per_launch": alg_bytes, "bytes_per_particle": BYTES_PER_PARTICLE,
                     "kernel_share_of_step": sum(mover_ms) / sum(step_ms),
                     "peak_source": peak_src},
        "general_3d": general,
        "clocks": clk.summary(),
        "e2e": e2e,
        "cpu_baseline": cpu,
        "strict_value": strict_value,
        "strict_what": "STRICT (bit-identical to the reference) mover, same state and field "
                       "(z-invariant: warp_tile_kernel<4,1,2,0>), 3 cycles",
        "moments": moments,
        "strong_scaling": strong,
        "c3": c3,
        "init_s": t_init,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm, N GPUs (one rank per GPU)
# ---------------------------------------------------------------------------

def verify_sample(store, sw_step, field, grid, rank, world, dist, gather, m=2048):
    """One untimed partitioned step checked against the reference mover: the
    first m particles of every species on every rank are moved on the host by
    pic::move_batch (oracle/_ref -- the particles are independent), then the
    distributed step runs; every expected particle must be found on exactly
    one rank, within the 1e-12 contract (positions |dx| <= 1e-12 L, velocities
    |dv| <= 1e-12 |v|).  Particles within 1e-9 of a periodic wall are not
    sampled (a wrap could put the GPU and host copies at 0 and at L)."""
    import numpy as np
    import torch
    import oracle
    from paper_1904_03684_b200.partition import _CudaArray
    gt = grid.as_tuple()
    L = np.array(gt[3:6])
    exp = []
    for s in range(store.n_species):
        k = min(m, store.count(s))
        if k == 0:
            exp.append(np.empty((0, 6)))
            continue
        p6 = [np.empty(k) for _ in range(6)]
        store.download_range(s, p6, 0, k)
        store.sync()
        qom = [-25.0, 1.0, -25.0, 1.0][s]
        if os.path.exists(oracle.REF_SO):
            oracle.ref_move_batch(p6, field.E.ravel(), field.B.ravel(), gt, DT, qom, PC)
        else:
            oracle.port_move_batch(p6, field.E.ravel(), field.B.ravel(), gt, DT, qom, PC)
        e = np.stack(p6, axis=1)
        near = np.any((e[:, :3] < 1e-9 * L) | (e[:, :3] > L - 1e-9 * L), axis=1)
        exp.append(e[~near])
    sw_step()
    allexp = gather(exp)                      # every rank's expected particles
    found = 0
    want = 0
    for s in range(store.n_species):
        e = np.concatenate([x[s] for x in allexp]) if allexp else np.empty((0, 6))
        want += len(e)
        n = store.count(s)
        if n == 0 or len(e) == 0:
            continue
        ptrs = store.device_ptrs(s)
        cols = [torch.as_tensor(_CudaArray(p, (n,)), device="cuda") for p in ptrs]
        xs, perm = torch.sort(cols[0])
        et = torch.as_tensor(e, device="cuda")
        tol_x = 1e-12 * float(L[0])
        lo = torch.searchsorted(xs, et[:, 0] - tol_x)
        hit = torch.zeros(len(e), dtype=torch.bool, device="cuda")
        vn = et[:, 3:].norm(dim=1)
        for c in range(4):                    # the few candidates inside the x window
            idx = (lo + c).clamp(max=n - 1)
            j = perm[idx]
            ok = torch.ones(len(e), dtype=torch.bool, device="cuda")
            for a in range(3):
                ok &= (cols[a][j] - et[:, a]).abs() <= 1e-12 * float(L[a])
            dv = torch.stack([cols[a][j] - et[:, a] for a in range(3, 6)], 1).norm(dim=1)
            ok &= dv <= 1e-12 * vn.clamp(min=1e-300)
            hit |= ok
        found += int(hit.sum().item())
    del xs, perm
    return found, want


def run_world(args):
    # the communicator lines (one per rank) go to stderr, not the JSON stream
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1904_03684_b200 import _capi, gem
    from paper_1904_03684_b200.engine import B200Engine, DeviceStore
    from paper_1904_03684_b200.mover import Grid, MoverParams
    from paper_1904_03684_b200.errors import ConfigError
    from paper_1904_03684_b200.partition import DeviceMigration, NativeSlabWorld, SlabWorld

    world_env = int(os.environ["WORLD_SIZE"])
    ndev = torch.cuda.device_count()
    shared = ndev < world_env   # ranks sharing GPUs: a functional run (NCCL needs one GPU each)
    backend = os.environ.get("B2M_DIST_BACKEND") or ("gloo" if shared else "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, ndev)
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", local)

    def reduce(x, op):
        t = torch.tensor([x], dtype=torch.float64)
        if backend == "nccl":
            t = t.to(dev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    def gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    # the native world over NCCL; B2M_NATIVE_WORLD=force also with a gloo
    # process group (ranks sharing a GPU with B2M_NCCL_LIB = tests/fake_nccl)
    nw_env = os.environ.get("B2M_NATIVE_WORLD", "1")
    native = nw_env == "force" or (backend == "nccl" and nw_env != "0")
    native_why = None
    field_of = (lambda g: gem.gem_bench_field(g)) if args.field == "gem+E" \
        else (lambda g: gem.gem_field(g))

    def setup(grid, ppc, pinned=True):
        """This rank's slab of the GEM state in a device store + its slab world."""
        batches = gem.init_gem_slab(grid, ppc, rank, world, pinned=pinned)
        field = field_of(grid)
        mps = [MoverParams.make(DT, b.qom, PC) for b in batches]
        caps = [int(b.count() * 1.05) + 65536 for b in batches]
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        store = DeviceStore(grid, caps, args.mode, device=local)
        store.set_stream(stream.cuda_stream)
        store.upload_field(field)
        for s, b in enumerate(batches):
            store.upload(s, b.span())
            if args.sort:
                store.sort(s)
        nonlocal native, native_why
        if native:
            try:
                sw = NativeSlabWorld(grid, store, rank, world, dist, comm=True)
            except ConfigError as e:
                # raised on EVERY rank together (NativeSlabWorld's NCCL probe
                # is agreed over dist): the same protocol in Python instead
                native, native_why = False, str(e)
        if not native:
            sw = SlabWorld(grid, DeviceMigration(store, rank, world), len(batches), dist, dev)
        sw.set_total()
        # field replication every cycle (runtime.cpp:143 / :221-223): rank 0's
        # device field broadcast to every rank, the gather tables rebuilt
        fE = fB = None
        if not native:
            fE = torch.as_tensor(field.E.ravel().copy(), device=dev)
            fB = torch.as_tensor(field.B.ravel().copy(), device=dev)

        def replicate():
            if native:
                sw.broadcast_field(0)
                return
            for t in (fE, fB):
                if backend == "nccl":
                    dist.broadcast(t, 0)
                else:
                    h = t.cpu()
                    dist.broadcast(h, 0)
                    t.copy_(h.to(dev))
            store.upload_field_device(fE.data_ptr(), fB.data_ptr())

        def step():
            if args.refresh:
                replicate()
            sw.step(mps)
        return batches, field, mps, store, sw, step

    def timed(store, step, steps):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        l0 = _capi.lib().b2m_launch_count()
        per = []
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            step()
            b.record()
            per.append((a, b))
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / steps
        launches = _capi.lib().b2m_launch_count() - l0
        step_ms = [a.elapsed_time(b) for a, b in per]
        # the native step's phase events (slots 13-15: mover + scan + compaction,
        # then exchange + merge) hold the LAST step; reading them inside the
        # loop would add a host sync per step
        if native:
            return ms, step_ms, store.elapsed_ms(13, 14), store.elapsed_ms(14, 15), launches
        return ms, step_ms, None, None, launches

    # ---- weak scaling: every rank a C2-sized slab ----
    grid = Grid.make(NX, NY * world, NZ, LX, LY * world, LZ)
    batches, field, mps, store, sw, step = setup(grid, PPC)
    n_local = sum(store.count(s) for s in range(len(batches)))
    with ClockSampler(local) as clk:
        ms, step_ms, mover_ms, exch_ms, launches = timed(store, step, args.steps)
    ms_max = reduce(ms, dist.ReduceOp.MAX)
    n_total = int(reduce(n_local, dist.ReduceOp.SUM))
    peak, peak_src = load_peaks()
    mine = {"rank": rank, "particles": n_local, "ms_per_step": ms, "mover_ms": mover_ms,
            "exchange_ms": exch_ms,
            "roofline_frac": (BYTES_PER_PARTICLE * n_local / (mover_ms * 1e-3) / 1e9 / peak)
            if mover_ms else None}
    ranks = gather(mine)
    reps = harmonic_reps([reduce(t, dist.ReduceOp.MAX) for t in step_ms], n_total)
    verify = None
    if args.verify:
        found, want = verify_sample(store, step, field, grid, rank, world, dist, gather)
        found = int(reduce(found, dist.ReduceOp.SUM))
        verify = {"sampled": want, "found_within_1e-12": found, "ok": found == want,
                  "how": "first 2048 particles of every species on every rank moved by the "
                         "reference pic::move_batch on the host; after one partitioned step "
                         "each must be on exactly one rank within the contract"}
        assert found == want, f"sampled reference check failed: {found} of {want}"
    counts_ok = True   # every step checked the global count (runtime.cpp:264-269)
    store.close()
    dist.barrier()

    # ---- e2e through the engine API on this rank's host batches ----
    e2e = None
    if args.e2e_steps > 0:
        eng = B200Engine(grid, mode=args.mode, schedule="pipeline", device=local)
        eng.prime(field, batches)
        eng.run_mover(field, batches, mps)  # warm-up
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            eng.run_mover(field, batches, mps)
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        eng.close()
        e2e_s = reduce(e2e_s, dist.ReduceOp.MAX)
        n_e2e = int(reduce(sum(b.count() for b in batches), dist.ReduceOp.SUM))
        e2e = {"value": n_e2e / e2e_s / 1e6, "unit": "MPA/s",
               "h2d_bytes_per_step": 48 * n_e2e + world * 2 * 24 * grid.nodes(),
               "d2h_bytes_per_step": 48 * n_e2e, "ms_per_step": e2e_s * 1e3,
               "steps": args.e2e_steps,
               "path": "B200Engine.run_mover per rank (pic::Engine contract) on the rank's "
                       "pinned host batches; max over ranks"}
    del batches

    # ---- strong scaling: C4 fixed (255.8M particles) on 1 and on N GPUs ----
    strong = None
    if args.strong:
        t1 = c4_single_gpu(args, local, args.field) if rank == 0 else None
        dist.barrier()
        g4 = Grid.make(NX, NY, NZ, LX, LY, LZ)
        b4, f4, mps4, st4, sw4, step4 = setup(g4, C4_PPC)
        n4 = int(reduce(sum(st4.count(s) for s in range(len(b4))), dist.ReduceOp.SUM))
        del b4
        ms4, _, mv4, ex4, _ = timed(st4, step4, args.steps)
        per4 = gather({"rank": rank, "ms_per_step": ms4, "mover_ms": mv4, "exchange_ms": ex4,
                       "particles": sum(st4.count(s) for s in range(st4.n_species))})
        ms4 = reduce(ms4, dist.ReduceOp.MAX)
        st4.close()
        if rank == 0:
            sp = t1["ms_per_step"] / ms4
            strong = {"workload": "GEM 64x64x32, 905 ppc (SURVEY C4), fixed; y-slabs of "
                                  f"{NY // world} cells", "particles": n4,
                      "t1": t1, "n_gpus": world, "ms_per_step": ms4,
                      "value": n4 / (ms4 * 1e-3) / 1e6, "unit": "MPA/s",
                      "speedup": sp, "efficiency": sp / world,
                      "efficiency_def": "S/N with S = T1/TN (bench.cpp:53-59)", "ranks": per4}
        dist.barrier()

    # ---- C3 (BASELINE configs[2]): 512M particles in N y-slabs of 128/N cells ----
    c3 = None
    if args.c3:
        g3 = Grid.make(*C3_GRID)
        b3, f3, mps3, st3, sw3, step3 = setup(g3, C3_PPC, pinned=False)
        n3 = int(reduce(sum(st3.count(s) for s in range(len(b3))), dist.ReduceOp.SUM))
        del b3
        ms3, _, mv3, ex3, _ = timed(st3, step3, args.steps)
        per3 = gather({"rank": rank, "ms_per_step": ms3, "mover_ms": mv3, "exchange_ms": ex3,
                       "particles": sum(st3.count(s) for s in range(st3.n_species))})
        ms3 = reduce(ms3, dist.ReduceOp.MAX)
        st3.close()
        if rank == 0:
            c3 = {"workload": "GEM 128x128x64, L = (51.2, 25.6, 12.8), 235 ppc (SURVEY C3, "
                              f"BASELINE configs[2]); y-slabs of {C3_GRID[1] // world} cells",
                  "particles": n3, "n_gpus": world, "ms_per_step": ms3,
                  "value": n3 / (ms3 * 1e-3) / 1e6, "unit": "MPA/s", "ranks": per3}
        dist.barrier()

    cpu = (cpu_reference_measure(args.field, 2, 1, whole_budget_s=30.0)
           if args.cpu_baseline and rank == 0 else None)
    if rank == 0:
        mv = [r["mover_ms"] for r in ranks if r["mover_ms"] is not None]
        kernel_ms = max(mv) if mv else None
        line = {"metric": "MPA/s in mover", "value": n_total / (ms_max * 1e-3) / 1e6,
                "unit": "MPA/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic GEM state (reference init_gem generator) per-rank C2-sized "
                        "slab" + (" + gem_like_field E" if args.field == "gem+E" else ""),
                "config": {"workload": f"GEM 2-D-in-3-D, 64x{64 * world}x32 cells, 216 ppc, "
                                       f"y-slabs of 64 cells (C2 per GPU)",
                           "particles": n_total, "mode": args.mode, "field": args.field,
                           "step": ("field broadcast from rank 0 + gather tables rebuilt + "
                                    if args.refresh else "") +
                                   "mover fused with the owner scan + compaction + NCCL P2P "
                                   "migration of all species + count all-reduce",
                           "cell_sort": "once, before the warm-up" if args.sort else "never",
                           "parallelism": f"y-slab x{world}, {backend}"
                                          + (" (ranks share GPUs: functional run)" if shared
                                             else "") + (", native b2m_world_step" if native
                                                         else ", Python SlabWorld")
                                          + (f" (native world unavailable: {native_why})"
                                             if native_why else "")},
                "repetitions": reps,
                "ranks": ranks,
                "gpu_launches": int(launches),
                "roofline": ({"bound": "hbm", "unit": "GB/s", "peak": peak,
                              "achieved": BYTES_PER_PARTICLE * ranks[0]["particles"]
                              / (ranks[0]["mover_ms"] * 1e-3) / 1e9,
                              "frac": ranks[0]["roofline_frac"],
                              "kernel": "rank 0: mover + gather-table rebuild + owner scan + "
                                        "compaction (b2m_world_step slots 13-14)",
                              "kernel_ms": ranks[0]["mover_ms"], "max_kernel_ms": kernel_ms,
                              "traffic": None, "peak_source": peak_src}
                             if mv else None),
                "verify": verify, "counts_conserved": counts_ok,
                "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
                "strong_scaling": strong, "c3": c3}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# launcher
# ---------------------------------------------------------------------------

def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(argv, n):
    """`--gpus N` outside torchrun: start N ranks (one process per GPU) with
    torch.distributed.run and relay rank 0's JSON line.  NCCL_DEBUG=INFO by
    default, to stderr, so the communicator lines show the N ranks."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + list(argv)
    p = subprocess.run(cmd, env=env, stdout=subprocess.PIPE, text=True)
    for ln in p.stdout.splitlines():
        (sys.stdout if ln.lstrip().startswith("{") else sys.stderr).write(ln + "\n")
    sys.stdout.flush()
    return p.returncode


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="fast", choices=["fast", "strict"])
    ap.add_argument("--sort", type=int, default=1, help="cell-sort species once before warm-up")
    ap.add_argument("--refresh", type=int, default=1,
                    help="every step marks the field rewritten (tables rebuilt in the step)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-baseline", type=int, default=1)
    ap.add_argument("--strict-too", type=int, default=1)
    ap.add_argument("--moments", type=int, default=1)
    ap.add_argument("--general-3d", type=int, default=1,
                    help="also time the general 3-D kernel on a z-varying field")
    ap.add_argument("--ref-sim", type=int, default=1,
                    help="reference arm: also time the reference's own Simulation (cpu engine)")
    ap.add_argument("--c3", type=int, default=1,
                    help="the C3 leg (BASELINE configs[2]: 512M particles, 128x128x64)")
    ap.add_argument("--strong", type=int, default=1,
                    help="the C4 strong-scaling leg (255.8M particles)")
    ap.add_argument("--verify", type=int, default=1,
                    help="N > 1: sampled check of one step against the reference mover")
    ap.add_argument("--field", default="gem+E", choices=["gem", "gem+E"],
                    help="gem+E: init_gem's B + the gem_like_field E (SURVEY §8d); gem: E = 0")
    return ap.parse_args(argv)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.impl == "reference":
        return run_reference_arm(args)
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:
        return self_launch(argv, args.gpus)
    # B2M_BENCH_WORLD=1 under a one-rank torchrun: the N > 1 code path (slab
    # world over a one-rank NCCL communicator) -- a check of that path on a
    # one-GPU box
    if world > 1 or (world == 1 and os.environ.get("B2M_BENCH_WORLD") == "1"):
        return run_world(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
