"""Compare ncu reports: duration, pipes, stalls per issued instruction, L1/L2 traffic."""
import csv, io, subprocess, sys
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__inst_executed.sum", "warp instr"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 inst %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data pipe %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "LDG requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_miss.sum", "LDG sector misses"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("sm__warps_active.avg.per_cycle_active", "warps active"),
]
STALLS = ["long_scoreboard", "wait", "short_scoreboard", "math_pipe_throttle", "branch_resolving",
          "no_instruction", "selected", "not_selected", "dispatch_stall", "mio_throttle", "lg_throttle",
          "barrier", "membar", "sleeping", "tex_throttle", "drain", "misc"]

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[2]))

reps = sys.argv[1:]
data = [raw(r) for r in reps]
print(f"{'':34s}" + "".join(f"{r.split('/')[-1][:22]:>24s}" for r in reps))
for k, name in KEYS:
    print(f"{name:34s}" + "".join(f"{d.get(k, '-'):>24s}" for d in data))
for s in STALLS:
    k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
    print(f"stall {s:28s}" + "".join(f"{d.get(k, '-'):>24s}" for d in data))
