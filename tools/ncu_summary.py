"""Summarise ncu captures into profiles/ (tracked): key metrics per kernel and
the launch-list time shares.  Usage:
  python tools/ncu_summary.py OUT_PREFIX launches.csv prof1.ncu-rep [prof2.ncu-rep ...]"""
import collections
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def main():
    prefix, launches, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    summary = {"kernels": [], "launch_shares": {}}
    for rep in reps:
        rows, units = raw(rep)
        for r in rows:
            summary["kernels"].append({"report": rep.split("/")[-1],
                                       "kernel": r.get("Kernel Name", "")[:120],
                                       **{k: (r.get(k), units.get(k)) for k in KEYS if k in r}})
    rows = [r for r in csv.reader(open(launches)) if len(r) > 5]
    hdr = rows[0]
    iN, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
             "second": 1e6, "s": 1e6}
    for r in rows[1:]:
        name = r[iN].split("(")[0].replace("void ", "")[:80]
        tot[name] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        cnt[name] += 1
    T = sum(tot.values())
    summary["launch_shares"] = {n: {"us": round(tot[n], 1), "share": round(tot[n] / T, 4),
                                    "launches": cnt[n]}
                                for n in sorted(tot, key=lambda n: -tot[n])}
    with open(prefix + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1)[:4000])


if __name__ == "__main__":
    main()
