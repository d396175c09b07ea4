"""Summary of one ncu --set full capture of the bench's snapshot sweep
(k3_sweep_rec): duration, DRAM bytes, FP64 instruction mix per candidate,
pipe utilisation and stalls -> JSON (profiles/r2_k6_sweep_ncu_summary.json,
read by bench.py for roofline.traffic and issued_fp64_per_candidate).
Usage: python scripts/ncu_sweep_summary.py <report.ncu-rep> <candidates> <out.json> [source]"""
import csv
import io
import json
import subprocess
import sys

rep, cands, out = sys.argv[1], float(sys.argv[2]), sys.argv[3]
source = sys.argv[4] if len(sys.argv) > 4 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))
u = dict(zip(h, units))


def num(k):
    x = float(str(d[k]).replace(",", ""))
    unit = u.get(k, "")
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e-3, "msecond": 1.0,
             "nsecond": 1e-6, "us": 1e-3, "ms": 1.0, "ns": 1e-6, "MB": 1e6, "KB": 1e3, "GB": 1e9}.get(unit, 1.0)
    return x * scale


cyc = num("sm__cycles_elapsed.avg")
per = lambda k: num(k) * cyc / cands  # noqa: E731  (per-cycle-elapsed sums -> totals per candidate)
dadd = per("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed")
dmul = per("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed")
fp64_pct = num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
nsm = 148
# FP64 pipe: 64 lanes per SM per cycle; thread-level ops issued to it
fp64_ops = fp64_pct / 100.0 * 64 * nsm * num("sm__cycles_active.avg") / cands
stalls = {k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]: float(d[k])
          for k in h if k.startswith("smsp__average_warps_issue_stalled_") and
          k.endswith("_per_issue_active.ratio") and float(d[k] or 0) > 0.02}
res = {
    "source": source,
    "kernel": d.get("Kernel Name", ""),
    "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size"),
    "candidates_per_launch": cands,
    "duration_ms": num("gpu__time_duration.sum"),
    "dram_bytes_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
    "dadd_per_candidate": dadd,
    "dmul_per_candidate": dmul,
    "issued_fp64_per_candidate": fp64_ops,
    "fp64_pipe_pct_active": fp64_pct,
    "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_per_sm": num("sm__warps_active.avg.per_cycle_active"),
    "warp_instructions_per_candidate": num("smsp__inst_executed.sum") / cands,
    "registers": num("launch__registers_per_thread"),
    "stalls_per_issue": stalls,
}
with open(out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res, indent=1))
