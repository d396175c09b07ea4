"""Summarise the K3P lines of scripts/k3_timeline.py (last launch only).

Usage: k3_timeline_stats.py log [ctas_per_item] [items (item-minor map)]

Line format (k3_sweep, -DK3_PROFILE): K3P block smid t_start t_staged t_loop_end t_end
(globaltimer ns).  Prints start/staging/loop/end spreads and per-item loop-end spread.
"""
import collections
import statistics
import sys

cpi = int(sys.argv[2]) if len(sys.argv) > 2 else 4
nitems = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # > 0: item-minor CTA map
rows = [l.split()[1:] for l in open(sys.argv[1]) if l.startswith("K3P ")]
rows = [tuple(int(x) for x in r) for r in rows]
nblk = max(r[0] for r in rows) + 1
last = rows[-nblk:]
t0 = min(r[2] for r in last)
rel = lambda v: (v - t0) / 1000.0
st = [rel(r[2]) for r in last]
stg = [rel(r[3]) - rel(r[2]) for r in last]
loop = [rel(r[4]) - rel(r[3]) for r in last]
end = [rel(r[5]) for r in last]
def q(v):
    v = sorted(v)
    return "min %.2f p10 %.2f p50 %.2f p90 %.2f max %.2f" % (
        v[0], v[len(v) // 10], v[len(v) // 2], v[9 * len(v) // 10], v[-1])
print("CTAs", len(last))
print("start  ", q(st))
print("staging", q(stg))
print("loop   ", q(loop))
print("end    ", q(end))
items = collections.defaultdict(list)
for r in last:
    items[r[0] % nitems if nitems else r[0] // cpi].append(rel(r[4]))
spread = [max(v) - min(v) for v in items.values()]
iend = [max(v) for v in items.values()]
print("item loop-end", q(iend))
print("intra-item loop-end spread", q(spread))
per_sm = collections.Counter(r[1] for r in last)
print("CTAs per SM", collections.Counter(per_sm.values()))
single = {sm for sm, c in per_sm.items() if c == 1}
print("loop time on single-CTA SMs", q([l for r, l in zip(last, loop) if r[1] in single] or [0]))
