"""Per-CTA timeline of one C4 gp_replan graph (needs the -DGP_TIMELINE build:
make -C paper_2505_15536_b200/csrc timeline).  Prints, per kernel, first
entry / last post-wait / last exit relative to the first CTA entry."""
import ctypes as C
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("GP_ENGINE_LIB", os.path.join(HERE, "paper_2505_15536_b200",
                                                    "libgeopipe_b200_tl.so"))
sys.path.insert(0, HERE)
import numpy as np  # noqa: E402
from paper_2505_15536_b200 import instances  # noqa: E402
from paper_2505_15536_b200.engine import Engine, lib  # noqa: E402
from paper_2505_15536_b200.layout import PackedInstance  # noqa: E402

REC = np.dtype([("t0", "<u8"), ("tw", "<u8"), ("t1", "<u8"), ("kid", "<u4"), ("blk", "<u4"),
                ("smid", "<u4"), ("pad", "<u4")])
NAMES = {51: "detail phases", 5: "arena_pull", 10: "k1p1 intervals", 11: "k1p1 groups", 12: "k1p1 gateways", 20: "k1p2 stages",
         21: "k1p2 boundary", 30: "k3_sweep", 40: "fixup", 50: "solve_detail"}


def drain():
    buf = np.zeros(65536, REC)
    n = C.c_uint32(0)
    lib().gp_diag_timeline(C.c_void_p(buf.ctypes.data), 65536, C.byref(n))
    return buf[: n.value]


which = sys.argv[1] if len(sys.argv) > 1 else "c4"
packs = [PackedInstance(*instances.load(which, snapshot=j), 1.25) for j in range(4)]
eng = Engine(0)
eng.replan_timing(True)
for i in range(30):
    eng.replan(packs[i % 4])
for rep in range(3):
    drain()
    eng.replan(packs[rep % 4])
    tl = drain()
    base = int(tl["t0"].min())
    print(f"--- replan {rep}: graph device {eng.replan_timing(True) * 1e3:.1f} us; "
          f"{len(tl)} CTA records; times in us from the first CTA entry")
    fs = tl[tl["kid"] == 23]
    if len(fs):  # register-path stage threads: smid field = clock64 cycles
        d = (fs["t1"] - fs["t0"]).astype(float)
        print(f"  fast stage threads: {len(fs)}, p50 {np.median(d) / 1e3:.2f} us, "
              f"p50 {np.median(fs['smid']):.0f} cycles -> {np.median(fs['smid'] / d) * 1e3:.0f} MHz")
        tl = tl[tl["kid"] != 23]
    th = tl[tl["kid"] == 22]
    tl = tl[tl["kid"] != 22]
    if len(th):  # per-thread K1 phase-2 stage records (kind = pad)
        d = (th["t1"] - th["t0"]) / 1e3
        print(f"  stage threads: first start {(int(th['t0'].min()) - base) / 1e3:.2f} "
              f"last start {(int(th['t0'].max()) - base) / 1e3:.2f} us")
        for kind in sorted(set(th["pad"].tolist())):
            sel = d[th["pad"] == kind]
            sp = ((th["tw"] - th["t0"]) / 1e3)[th["pad"] == kind]
            print(f"  stage kind {kind}: threads {len(sel)} p50 {np.median(sel):.2f} "
                  f"max {sel.max():.2f} us; choose_split p50 {np.median(sp):.2f} us")
        slow = np.argsort(-d)[:5]
        for j in slow:
            b = int(th["blk"][j])
            print(f"  slow: f {b >> 16} a {(b >> 8) & 255} b {b & 255} kind {th['pad'][j]} "
                  f"{d[j]:.2f} us")
    for kid in sorted(set(tl["kid"].tolist())):
        r = tl[tl["kid"] == kid]
        f = lambda v: (int(v) - base) / 1e3
        print(f"{NAMES.get(kid, kid):>16}: ctas {len(r):4d} first-entry {f(r['t0'].min()):7.2f} "
              f"last-entry {f(r['t0'].max()):7.2f} last-wait {f(r['tw'].max()):7.2f} "
              f"first-exit {f(r['t1'].min()):7.2f} last-exit {f(r['t1'].max()):7.2f} "
              f"max-cta {(r['t1'] - r['tw']).max() / 1e3:6.2f}")
