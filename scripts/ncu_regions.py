"""Per-region breakdown of an ncu --set full capture (source page, SASS):
instructions grouped by execution count (a loop body executes its
instructions equally often), with warp-stall samples by reason.
Usage: python scripts/ncu_regions.py <report.ncu-rep> [min_share]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
min_share = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
iS, iW, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ist = [h.index(c) for c in stalls]
tot_s = sum(int(r[iW]) for r in data) or 1
tot_e = sum(int(r[iE]) for r in data) or 1
groups = {}
for j, r in enumerate(data):
    e = int(r[iE])
    g = groups.setdefault(e, {"n": 0, "s": 0, "first": j, "src": r[iS].strip(), "st": [0] * len(stalls)})
    g["n"] += 1
    g["s"] += int(r[iW])
    for q, i in enumerate(ist):
        g["st"][q] += int(r[i] or 0)
print(f"samples {tot_s} warp-instructions {tot_e}")
for e, g in sorted(groups.items(), key=lambda kv: -kv[1]["s"]):
    if g["s"] / tot_s < min_share and e * g["n"] / tot_e < min_share:
        continue
    top = sorted(zip(stalls, g["st"]), key=lambda x: -x[1])[:4]
    print(f"exec {e:9d} x{g['n']:4d} instr {100 * e * g['n'] / tot_e:5.1f}%  samples {100 * g['s'] / tot_s:5.1f}%  "
          f"line {g['first']:5d} {g['src'][:34]:34s} | " +
          " ".join(f"{k[6:]}={100 * v / tot_s:.1f}" for k, v in top))
