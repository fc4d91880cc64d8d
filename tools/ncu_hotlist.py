"""Per-instruction SASS listing (exec count per 32 particles, stall samples) of an ncu report.
  python tools/ncu_hotlist.py REPORT.ncu-rep [min_exec_per_batch] [particles]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
P = (float(sys.argv[3]) if len(sys.argv) > 3 else 61046784) / 32
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]; data = rows[2:]
ix = {k: i for i, k in enumerate(h)}
cols = ['stall_wait', 'stall_long_sb', 'stall_short_sb', 'stall_branch_resolving', 'stall_math', 'stall_selected']
for k, r in enumerate(data):
    n = int(r[ix['Instructions Executed']] or 0)
    s = int(r[ix['# Samples']] or 0)
    if n / P < mn and s < 50: continue
    st = ' '.join(f"{c[6:10]}={r[ix[c]]}" for c in cols if int(r[ix[c]] or 0) >= 100)
    print(f"{k:5d} {n / P:6.2f} {s:6d} {r[ix['Source']].strip()[:72]:72s} {st}")
