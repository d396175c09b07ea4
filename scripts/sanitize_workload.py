#!/usr/bin/env python3
"""Small workload touching every engine kernel, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).

  compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize_workload.py

Each section checks its answer against the golden fixtures so that a run
under a tool is also a parity run.  GP_K3_CLUSTER=2 in the environment
exercises the thread-block-cluster multicast staging of the sweep.
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from cases import enumerate_encoded, golden_costs, load_case, same_bits  # noqa: E402
import paper_2505_15536_b200 as P  # noqa: E402
from paper_2505_15536_b200 import instances as I  # noqa: E402
from paper_2505_15536_b200 import replan as R  # noqa: E402
from paper_2505_15536_b200 import simulate as SM  # noqa: E402
from paper_2505_15536_b200 import schedule as SCH  # noqa: E402
from paper_2505_15536_b200 import grouping as GR  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402
from paper_2505_15536_b200.layout import PackedInstance  # noqa: E402


def section(name):
    print(f"-- {name}", flush=True)


def main():
    eng = Engine(0)
    doc, model, topo, groups = load_case("c2j")
    packed = PackedInstance(model, topo, groups, 1.25)
    gc, gs = golden_costs("c2j")
    eng.load(packed)
    total = eng.space_size()
    exp = doc["exhaustive"]["result"]["breakdown"]["plan_cost"]

    section("K1 + K3 sweep / tile / generic / record kernels")
    for mode in (-1, 0, 1, 2, 3, 5):
        eng.set_k3_mode(mode)
        assert eng.argmin_range(0, total).cost == exp, mode
        b = eng.argmin_range(1000, 9000)
        assert same_bits(b.cost, gc[1000:9000].min())
    eng.set_k3_mode(-1)
    assert eng.argmin_items(3, 11).evaluated > 0

    section("verify sink")
    eng.verify_begin(0, total)
    eng.argmin_range(0, total)
    v = eng.verify_end()
    assert same_bits(v, gc).all()

    section("gp_replan graph (arena pull, K1, sweep, detail; PDL)")
    for _ in range(3):
        b, info = eng.replan(packed)
        assert b.cost == exp and info.plan_cost == exp

    section("K2 small and large batches")
    order, counts, bm = enumerate_encoded(packed)
    c, s = eng.eval_batch(order[:500], counts[:500], bm[:500])
    assert same_bits(c, gc[:500]).all()
    reps = (1 << 16) // order.shape[0] + 1
    c, s = eng.eval_batch(np.tile(order, (reps, 1)), np.tile(counts, (reps, 1)), np.tile(bm, reps))
    assert same_bits(c, np.tile(gc, reps)).all()

    section("K6 snapshots (fast path + zero-bandwidth slow path)")
    spec = I.config("c2")
    m2, t2, g2 = I.build(spec)
    p2 = PackedInstance(m2, t2, g2, 1.25)
    eng.load(p2)
    mults = [I.snapshot_multipliers(spec, j) for j in range(3)]
    ids = sorted(d.id for d in t2.devices)
    mz = dict(mults[0])
    mz[(ids[0], ids[1])] = 0.0
    bws = R.bandwidth_matrices(p2, mults + [mz])
    bests, st = eng.replan_snapshots(bws)
    assert list(st[:3]) == [0, 0, 0] and st[3] != 0

    section("K4 branch-and-bound")
    eng.load(packed)
    assert eng.argmin_bnb().cost == exp

    section("drop-in exhaustive_plan / search_plan / plan_cost")
    r = P.exhaustive_plan(model, topo, groups, P.SearchConfig(seed=0), engine=eng)
    assert r.breakdown.plan_cost == exp
    P.search_plan(model, topo, groups, P.SearchConfig(seed=1), engine=eng)
    from paper_2505_15536_b200 import costmodel as CM
    CM.plan_cost(r.plan, topo, model, groups, engine=eng)
    eng.plan_timing(order[:64], counts[:64], bm[:64])
    eng.sim_candidates(order[:64], counts[:64], bm[:64], 2, 0.0)

    section("K5 1F1B + full event engine + schedules, K8 validation")
    tims = [SM.make_timing(fwd=[1.0, 1.5, 0.7], bwd=[2.0, 2.5, 1.1], wgt=[0.5, 0.4, 0.3],
                           transfer=[0.8, 1.3], microbatch=4, micro_count=m, latency=0.05,
                           sync=[0.1, 0.2, 0.1], opt=[0.05, 0.05, 0.05]) for m in (3, 5, 8)]
    arr = SM.pack_timings(tims)
    eng.sim_1f1b(arr, 3, 2)
    trace = [{"0-1": [[2.0, 0.25], [9.0, 1.0]], "1-2": [[4.0, 0.5]]}]
    tr = SM.pack_traces(trace)
    eng.simulate(arr, 3, 3, 2, tr, 1, [0, 0, 0])
    eng.simulate_report(arr, 3, 3, 3, tr, 1, [0, 0, 0], adapter=True, async_iterations=True)
    sched = SCH.generate_schedules(tims, "zb_compact", trace, [0, 0, 0], adapter_enabled=True,
                                   config=SM.SimConfig(iterations=2, async_iterations=True),
                                   engine=eng)
    SCH.validate_schedules([s_ for s_, _ in sched], tims, engine=eng)

    section("K7 grouping")
    _, t1, _ = I.load("c1")
    ids1, pt, bw, pc = GR.topology_arrays(t1)
    GR.group_hierarchies(np.stack([pt, pt * 1.5]), bw, pc, engine=eng)
    eng.close()
    print("sanitize workload ok", flush=True)


if __name__ == "__main__":
    main()
