"""Top SASS instructions of an ncu report by warp-stall samples:
python tools/ncu_hot.py REPORT [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
body = rows[2:]
ci = h.index("Warp Stall Sampling (All Samples)")
ei = h.index("Instructions Executed")
def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0
tot = sum(f(r[ci]) for r in body)
inst = sum(f(r[ei]) for r in body)
print(f"samples {tot:.0f}  warp instructions {inst:.0f}")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_")]
for r in sorted(body, key=lambda r: -f(r[ci]))[:n]:
    top = sorted(((f(r[i]), h[i][6:]) for i in stall_cols), reverse=True)[:2]
    print(f"{r[0]:>6} {100 * f(r[ci]) / tot:5.1f}%  {r[1][:60]:60s} "
          + " ".join(f"{k}={v:.0f}" for v, k in top))
