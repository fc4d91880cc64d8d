"""Key metrics + instruction mix + stall summary of one kernel in an ncu report.
  python tools/ncu_brief.py REPORT.ncu-rep [particles]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
nparts = float(sys.argv[2]) if len(sys.argv) > 2 else 61046784
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
for w in want:
    if w in h:
        print(f"{w:70s} {v[h.index(w)]} {rows[1][h.index(w)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]; data = rows[2:]
ix = {k: i for i, k in enumerate(h)}
P = nparts / 32
byop = collections.Counter(); stall = collections.Counter(); tot = 0; samples = 0
scols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
for r in data:
    n = int(r[ix["Instructions Executed"]] or 0)
    srcl = r[ix["Source"]].strip().split()
    if not srcl: continue
    op = srcl[1] if srcl[0].startswith("@") else srcl[0]
    byop[op.split(".")[0]] += n; tot += n
    for c in scols: stall[c] += int(r[ix[c]] or 0)
    samples += int(r[ix["# Samples"]] or 0)
print(f"warp instructions per 32 particles: {tot / P:.1f}")
print(" ".join(f"{op}:{n / P:.1f}" for op, n in byop.most_common(30)))
print(" ".join(f"{c[6:]}:{n / max(samples, 1):.3f}" for c, n in stall.most_common(12)))
