#!/usr/bin/env python3
"""Generate tests/golden/ fixtures from the UNMODIFIED reference (build container only).

The reference (/root/reference/pkg/src, pure Python) is imported read-only; its
outputs are frozen into JSON / .npy files so that the GPU box - which has no
/root/reference - can check the engine against the reference's own answers.

Cases
  c1, c1j, c2, c2j   App. D configs (integer / jittered): every candidate's
                     _evaluate cost in exhaustive_plan enumeration order, the
                     exhaustive_plan result, search_plan results for seeds 0-5
  c4, c4j            App. D config C4: 20,000 sampled candidates' costs
                     (random.Random(4).sample), search_plan seeds 0-1, and the
                     full 11.4M exhaustive arg-min computed by the C oracle
                     (the oracle is first checked bit-exact on the sample)
  small, rand*       reference test fixtures (tests/conftest.py small_setup,
                     tests/test_acceptance.py:_random_instance)
  err_*              error behaviour: all-infeasible memory, zero intra-group
                     bandwidth, zero-bandwidth gateway
  k5n9 .. k8n9       k = 5..8 stage groups (instances.many_group_config):
                     every candidate's reference cost, exhaustive_plan, search
  k5n24 .. k6n40     k = 5..8, larger spaces (up to 1.66e9 candidates, the
                     K4 regime): a 2,000-candidate reference sample that pins
                     the oracle on that instance, then the oracle's arg-min
Usage: python scripts/make_golden.py [--skip-c4] [--only many:k5n9]
"""

from __future__ import annotations

import argparse
import itertools
import json
import logging
import os
import random
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import golden_io as G  # noqa: E402
from refbridge import AVAILABLE, build_reference, geopipe  # noqa: E402

from paper_2505_15536_b200 import instances as I  # noqa: E402
from paper_2505_15536_b200.layout import PackedInstance  # noqa: E402

logging.disable(logging.CRITICAL)


def enumerate_all(model, groups):
    """Candidates in exhaustive_plan order (src/planner.py:389-392)."""
    from geopipe.planner import Candidate, _compositions
    fg_ids = sorted(groups.fgs)
    n = model.num_layers
    for bi, b in enumerate(model.global_batch_candidates):
        for mi, m in enumerate(model.microbatch_candidates):
            for order in itertools.permutations(fg_ids):
                for cuts in _compositions(n, len(order)):
                    yield bi * len(model.microbatch_candidates) + mi, b, m, Candidate(order, cuts)


ERR_CODE = {"InputFileError": 1, "InfeasibleSplitError": 2, "NoFeasiblePlanError": 3,
            "DegenerateGroupError": 4, "InvalidTopologyError": 5}


def ref_cost(model, topo, groups, cand, b, m, cfg):
    """(cost, status): status is the C-ABI code of the exception _evaluate raises."""
    from geopipe.planner import _evaluate
    try:
        return _evaluate(cand, b, m, groups, topo, model, cfg, {})[0], 0
    except Exception as e:
        return float("nan"), ERR_CODE[type(e).__name__]


def run_or_error(fn):
    try:
        return {"result": G.result_to_dict(fn())}
    except Exception as e:  # reference exception class name is the golden
        return {"error": type(e).__name__}


def dump_case(name, model, topo, groups, seeds, all_costs=True, beam_width=8, max_iter=20):
    gp = geopipe()
    doc = {"instance": G.instance_to_dict(model, topo, groups)}
    t = time.time()
    if all_costs:
        cfg = gp.SearchConfig(seed=0)
        out = [ref_cost(model, topo, groups, c, b, m, cfg)
               for _, b, m, c in enumerate_all(model, groups)]
        costs = np.array([c for c, _ in out], dtype=np.float64)
        status = np.array([s for _, s in out], dtype=np.uint8)
        np.save(os.path.join(G.GOLDEN, f"{name}.costs.npy"), costs)
        np.save(os.path.join(G.GOLDEN, f"{name}.status.npy"), status)
        doc["n_candidates"] = int(costs.size)
    cfg0 = gp.SearchConfig(seed=0, beam_width=beam_width, max_iter=max_iter)
    doc["exhaustive"] = run_or_error(lambda: gp.exhaustive_plan(model, topo, groups, cfg0))
    doc["search"] = {}
    for s in seeds:
        cfg = gp.SearchConfig(seed=s, beam_width=beam_width, max_iter=max_iter)
        doc["search"][str(s)] = run_or_error(lambda: gp.search_plan(model, topo, groups, cfg))
    doc["search_config"] = {"beam_width": beam_width, "max_iter": max_iter}
    G.save(f"{name}.json", doc)
    print(f"{name}: {time.time() - t:.1f}s", flush=True)


def dump_c4(name, jitter):
    gp = geopipe()
    from oracle import oracle as O
    spec = I.config("c4", jitter)
    model, topo, groups = build_reference(spec)
    doc = {"instance": G.instance_to_dict(model, topo, groups)}
    packed = PackedInstance(model, topo, groups, 1.25)
    total = O.space_size(packed)
    idx = sorted(random.Random(4).sample(range(total), 20000))
    cfg = gp.SearchConfig(seed=0)
    t = time.time()
    fg_ids = sorted(groups.fgs)
    from geopipe.planner import Candidate
    costs = []
    for i in idx:
        o, c, bm = O.decode(packed, i)
        b = model.global_batch_candidates[bm // len(model.microbatch_candidates)]
        m = model.microbatch_candidates[bm % len(model.microbatch_candidates)]
        cand = Candidate(tuple(fg_ids[x] for x in o), tuple(int(x) for x in c))
        costs.append(ref_cost(model, topo, groups, cand, b, m, cfg)[0])
    costs = np.array(costs, dtype=np.float64)
    # pin the oracle on this sample before trusting its full sweep
    oc = []
    for i in idx:
        o, c, bm = O.decode(packed, i)
        st, v = O.evaluate(packed, o, c, bm)
        assert st == 0
        oc.append(v)
    oc = np.array(oc)
    assert (oc.view(np.uint64) == costs.view(np.uint64)).all(), "oracle != reference on C4 sample"
    np.save(os.path.join(G.GOLDEN, f"{name}.sample_idx.npy"), np.array(idx, dtype=np.uint64))
    np.save(os.path.join(G.GOLDEN, f"{name}.sample_costs.npy"), costs)
    print(f"{name}: sample {time.time() - t:.1f}s", flush=True)
    t = time.time()
    st, best = O.argmin_range(packed, 0, total, threads=os.cpu_count())
    doc["oracle_argmin"] = {"status": st, "cost": best.cost, "index": best.index,
                            "order": list(best.order[:best.k]),
                            "counts": list(best.counts[:best.k]),
                            "batch_index": best.batch_index, "micro_index": best.micro_index,
                            "evaluated": total,
                            "cpu_seconds_8threads": time.time() - t}
    print(f"{name}: oracle argmin {time.time() - t:.1f}s", flush=True)
    doc["search"] = {}
    for s in (0, 1):
        t = time.time()
        doc["search"][str(s)] = run_or_error(
            lambda: gp.search_plan(model, topo, groups, gp.SearchConfig(seed=s)))
        print(f"{name}: search seed {s} {time.time() - t:.1f}s", flush=True)
    doc["search_config"] = {"beam_width": 8, "max_iter": 20}
    G.save(f"{name}.json", doc)


def timing_to_dict(t):
    return {"batch": t.batch, "microbatch": t.microbatch,
            "stages": [[st.fwd_per_sample, st.bwd_per_sample, st.wgt_per_sample,
                        st.sync_seconds, st.opt_seconds] for st in t.stages],
            "boundaries": [[b.latency_seconds, b.bandwidth_bytes_per_s,
                            b.act_bytes_per_sample, b.grad_bytes_per_sample]
                           for b in t.boundaries]}


def dump_sim():
    """1F1B makespans (simulate_timing, ONE_F_ONE_B) of random and plan timings."""
    gp = geopipe()
    sys.path.insert(0, "/root/reference/pkg/tests")
    from test_schedule import random_timing
    from test_acceptance import _random_instance
    rng = random.Random(2024)
    cases = [random_timing(rng) for _ in range(1500)]
    # timings of real plans: winners and random candidates of the golden configs
    for seed in range(100, 130):
        topo, groups, model = _random_instance(seed)
        res = gp.search_plan(model, topo, groups, gp.SearchConfig(seed=seed))
        cases.append(gp.build_plan_timing(res.plan, topo, model, groups))
    for cfg_name, jit in [("c1", False), ("c2", True), ("c4", False)]:
        model, topo, groups = build_reference(I.config(cfg_name, jit))
        res = gp.search_plan(model, topo, groups, gp.SearchConfig(seed=0))
        for opt in (0.0, 0.25):
            cases.append(gp.build_plan_timing(res.plan, topo, model, groups, opt_seconds=opt))
    out = {"timings": [timing_to_dict(t) for t in cases], "makespan": {}}
    t0 = time.time()
    for it in (1, 2, 3):
        ms = []
        for t in cases:
            try:
                ms.append(gp.simulate_timing(t, gp.Policy.ONE_F_ONE_B,
                                             config=gp.SimConfig(iterations=it)).makespan)
            except Exception as e:
                ms.append(type(e).__name__)
        out["makespan"][str(it)] = ms
    G.save("sim.json", out)
    print(f"sim: {len(cases)} timings x 3 iteration counts, {time.time() - t0:.1f}s", flush=True)


def dump_sim_policies():
    """makespans under all four policies with random breakpoint traces."""
    gp = geopipe()
    sys.path.insert(0, "/root/reference/pkg/tests")
    from test_schedule import random_timing
    rng = random.Random(77)
    cases = [random_timing(rng) for _ in range(400)]
    traces = []
    for t in cases:
        bps = {}
        for b in range(t.num_stages - 1):
            if rng.random() < 0.75:
                pts = sorted(set(round(rng.uniform(0.0, 25.0), 3) for _ in range(rng.randint(1, 8))))
                bps[f"{b}-{b + 1}"] = [[x, rng.choice([0.25, 0.4, 0.5, 0.6, 0.8, 1.0, 1.5, 2.0])]
                                       for x in pts]
        traces.append(bps)
    out = {"timings": [timing_to_dict(t) for t in cases], "traces": traces, "makespan": {}}
    t0 = time.time()
    for pol in gp.Policy:
        for it in (1, 2):
            ms = []
            for t, bps in zip(cases, traces):
                tr = gp.NetworkTrace(breakpoints={k: tuple(tuple(p) for p in v)
                                                  for k, v in bps.items()})
                try:
                    ms.append(gp.simulate_timing(t, pol, tr,
                                                 config=gp.SimConfig(iterations=it)).makespan)
                except Exception as e:
                    ms.append(type(e).__name__)
            out["makespan"][f"{pol.value}:{it}"] = ms
    G.save("sim_policies.json", out)
    print(f"sim policies: {time.time() - t0:.1f}s", flush=True)


def dump_sim_reports():
    """simulate_timing reports with the adapter and asynchronous iterations:
    makespan, throughput, steady_throughput, bubble_fractions, iteration_ends
    and the action / transfer / op counts, under degrading traces."""
    gp = geopipe()
    rng = random.Random(91)
    cases, traces = [], []
    for _ in range(160):
        S = rng.randint(1, 5)
        micro = rng.choice([1, 2, 4, 8])
        cases.append(gp.make_timing(
            fwd=[rng.uniform(0.2, 2.0) for _ in range(S)], bwd=[rng.uniform(0.2, 2.0) for _ in range(S)],
            wgt=[rng.uniform(0.05, 1.0) for _ in range(S)],
            transfer=[rng.uniform(0.05, 2.5) for _ in range(S - 1)], microbatch=micro,
            micro_count=rng.randint(1, 16), sync=[rng.uniform(0, 0.5) for _ in range(S)],
            opt=[rng.uniform(0, 0.3) for _ in range(S)], latency=rng.uniform(0.0, 0.2)))
        bps = {}
        for b in range(S - 1):
            if rng.random() < 0.8:
                pts = sorted(set(round(rng.uniform(0.0, 60.0), 3) for _ in range(rng.randint(1, 6))))
                bps[f"{b}-{b + 1}"] = [[x, rng.choice([0.25, 0.4, 0.5, 0.6, 1.0])] for x in pts]
        traces.append(bps)
    out = {"timings": [timing_to_dict(t) for t in cases], "traces": traces, "reports": {}}
    t0 = time.time()
    combos = [(ad, asy, pol.value, it, 1.2, 1.05) for ad in (0, 1) for asy in (0, 1)
              for pol in gp.Policy for it in (1, 3)]
    combos += [(1, 0, "zb_compact", 3, 1.1, 1.02), (1, 1, "1f1b", 4, 1.5, 1.2)]
    for ad, asy, pol, it, deg, rec in combos:
        cfg = gp.SimConfig(iterations=it, async_iterations=bool(asy),
                           adapter=gp.AdapterConfig(degrade_factor=deg, recover_factor=rec))
        rows = []
        for t, bps in zip(cases, traces):
            tr = gp.NetworkTrace(breakpoints={k: tuple(tuple(p) for p in v) for k, v in bps.items()})
            try:
                r = gp.simulate_timing(t, gp.Policy(pol), tr, adapter_enabled=bool(ad), config=cfg)
            except Exception as e:
                rows.append(type(e).__name__)
                continue
            rows.append([r.makespan, r.throughput, r.steady_throughput, list(r.bubble_fractions),
                         list(r.iteration_ends), len(r.adapter_actions), len(r.transfers),
                         sum(len(o) for o in r.schedule.ops)])
        out["reports"][f"{ad}:{asy}:{pol}:{it}:{deg}:{rec}"] = rows
    G.save("sim_reports.json", out)
    print(f"sim reports: {time.time() - t0:.1f}s", flush=True)


def dump_sim_candidates():
    """simulate(build_plan(candidate), ONE_F_ONE_B) makespans of candidates."""
    gp = geopipe()
    from geopipe.planner import build_plan, memory_feasible
    out = {}
    t0 = time.time()
    for name, cfg_name, jit, nsample in [("c1", "c1", False, None), ("c2j", "c2", True, 600),
                                         ("c4", "c4", False, 300)]:
        model, topo, groups = build_reference(I.config(cfg_name, jit))
        allc = list(enumerate_all(model, groups))
        rng = random.Random(17)
        idx = range(len(allc)) if nsample is None else sorted(rng.sample(range(len(allc)), nsample))
        rows = []
        for i in idx:
            bm, b, m, cand = allc[i]
            plan = build_plan(cand, b, m, groups, topo, model, 1.25)
            if not memory_feasible(plan, model, groups, topo):
                rows.append([i, "infeasible", "infeasible"])
                continue
            vals = []
            for it, opt in ((1, 0.0), (2, 0.5)):
                r = gp.simulate(plan, topo, model, groups, gp.Policy.ONE_F_ONE_B,
                                config=gp.SimConfig(iterations=it, opt_seconds=opt))
                vals.append(r.makespan)
            rows.append([i] + vals)
        out[name] = rows
    G.save("sim_cands.json", out)
    print(f"sim candidates: {time.time() - t0:.1f}s", flush=True)


def dump_snapshots():
    """C3: exhaustive re-plan of C2 per bandwidth snapshot (App. D recipe).

    Each snapshot is rebuilt with the reference's own constructors and
    grouping (CS4 composition); the arg-min comes from the pinned oracle,
    itself checked against the reference's exhaustive_plan on 3 snapshots."""
    from oracle import oracle as O
    gp = geopipe()
    spec = I.config("c2")
    out = {"config": "c2", "snapshots": []}
    t0 = time.time()
    for j in range(200):
        mult = I.snapshot_multipliers(spec, j)
        model, topo, groups = build_reference(spec, mult)
        packed = PackedInstance(model, topo, groups, 1.25)
        st, best = O.argmin_range(packed, 0, O.space_size(packed), threads=os.cpu_count())
        rec = {"j": j, "status": st, "cost": best.cost, "index": best.index,
               "min_bw": {f: groups.fgs[f].min_intra_bandwidth for f in sorted(groups.fgs)}}
        if j < 3:
            r = gp.exhaustive_plan(model, topo, groups, gp.SearchConfig(seed=0))
            assert r.breakdown.plan_cost == best.cost, (j, r.breakdown.plan_cost, best.cost)
            rec["reference"] = G.result_to_dict(r)
        out["snapshots"].append(rec)
    G.save("c3_snapshots.json", out)
    print(f"snapshots: {time.time() - t0:.1f}s", flush=True)


# k >= 5 stage groups (the regime exhaustive_plan hands to K4 above 5e8
# candidates): small spaces with every candidate's reference cost, larger
# ones with the pinned oracle's arg-min (pinned on a reference sample).
MANY_SMALL = [("k5n9", 5, 9, 51, (64, 128), (8, 16)), ("k6n8", 6, 8, 61, (64, 128), (8, 16)),
              ("k7n8", 7, 8, 71, (64, 128), (8,)), ("k8n9", 8, 9, 81, (64, 128), (16,))]
MANY_BIG = [("k5n24", 5, 24, 100, (64, 128), (8, 16)), ("k6n20", 6, 20, 100, (64, 128), (8, 16)),
            ("k7n16", 7, 16, 72, (64, 128), (8,)), ("k8n14", 8, 14, 82, (64, 128), (16,)),
            ("k6n40", 6, 40, 100, (64, 128), (8, 16))]


def _many_ref(k, n, seed, batches, micros):
    spec = I.many_group_config(k, n, seed, batches, micros)
    model, topo, groups = build_reference(spec)
    assert len(groups.fgs) == k, (k, n, seed, len(groups.fgs))
    return model, topo, groups


def dump_many(which=None):
    for name, k, n, seed, bs, ms in MANY_SMALL:
        if which and name != which:
            continue
        model, topo, groups = _many_ref(k, n, seed, bs, ms)
        dump_case(name, model, topo, groups, seeds=[0, 1])
    from oracle import oracle as O
    gp = geopipe()
    from geopipe.planner import Candidate
    for name, k, n, seed, bs, ms in MANY_BIG:
        if which and name != which:
            continue
        model, topo, groups = _many_ref(k, n, seed, bs, ms)
        doc = {"instance": G.instance_to_dict(model, topo, groups)}
        packed = PackedInstance(model, topo, groups, 1.25)
        total = O.space_size(packed)
        idx = sorted(random.Random(seed).sample(range(total), 2000))
        cfg = gp.SearchConfig(seed=0)
        fg_ids = sorted(groups.fgs)
        costs, stats = [], []
        t = time.time()
        for i in idx:
            o, c, bm = O.decode(packed, i)
            b = model.global_batch_candidates[bm // len(model.microbatch_candidates)]
            m = model.microbatch_candidates[bm % len(model.microbatch_candidates)]
            cand = Candidate(tuple(fg_ids[x] for x in o), tuple(int(x) for x in c))
            cv, sv = ref_cost(model, topo, groups, cand, b, m, cfg)
            st_o, v_o = O.evaluate(packed, o, c, bm)
            assert st_o == sv and (sv != 0 or np.float64(v_o).view(np.uint64) ==
                                   np.float64(cv).view(np.uint64)), (name, i)
            costs.append(cv)
            stats.append(sv)
        doc["sample"] = {"index": idx, "cost": [G._f(x) for x in costs], "status": stats}
        print(f"{name}: reference sample {time.time() - t:.1f}s (oracle pinned)", flush=True)
        t = time.time()
        st, best = O.argmin_range(packed, 0, total, threads=os.cpu_count())
        doc["oracle_argmin"] = {"status": st, "cost": best.cost, "index": best.index,
                                "order": list(best.order[:best.k]),
                                "counts": list(best.counts[:best.k]),
                                "batch_index": best.batch_index, "micro_index": best.micro_index,
                                "evaluated": total,
                                "cpu_seconds": time.time() - t, "threads": os.cpu_count()}
        print(f"{name}: oracle argmin over {total} candidates {time.time() - t:.1f}s", flush=True)
        doc["search"] = {}
        for s_ in (0,):
            doc["search"][str(s_)] = run_or_error(
                lambda: gp.search_plan(model, topo, groups, gp.SearchConfig(seed=s_)))
        doc["search_config"] = {"beam_width": 8, "max_iter": 20}
        G.save(f"{name}.json", doc)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c4", action="store_true")
    ap.add_argument("--only-sim", action="store_true")
    ap.add_argument("--only", default=None, help="run one dump_* function, e.g. sim_reports")
    args = ap.parse_args()
    if not AVAILABLE:
        sys.exit("reference not available at /root/reference")
    gp = geopipe()
    sys.path.insert(0, "/root/reference/pkg/tests")
    import conftest as rc  # reference test fixtures (read-only import)
    os.makedirs(G.GOLDEN, exist_ok=True)
    if args.only:
        if args.only.startswith("many:"):
            dump_many(args.only[5:])
            return
        globals()["dump_" + args.only]()
        return
    ap_only = args.only_sim
    if ap_only:
        dump_sim_reports()
        dump_sim_policies()
        dump_sim()
        dump_sim_candidates()
        dump_snapshots()
        return
    dump_sim()
    dump_sim_policies()
    dump_sim_reports()
    dump_sim_candidates()
    dump_snapshots()
    dump_grouping()
    dump_schedules()
    dump_cli()
    dump_plan_costs()
    dump_region_sweep()
    dump_search_seeds()
    dump_regroup_replan()

    for name, cfg_name, jit in [("c1", "c1", False), ("c1j", "c1", True),
                                ("c2", "c2", False), ("c2j", "c2", True)]:
        model, topo, groups = build_reference(I.config(cfg_name, jit))
        dump_case(name, model, topo, groups, seeds=range(6))

    # tests/test_planner.py small_setup
    topo = rc.clique_topology([[4.0, 4.0], [2.0], [1.0]], intra=0.01, cross=0.5,
                              bandwidth=1e8, latency=0.001)
    groups = rc.make_groups(topo)
    model = rc.uniform_model(6, flops=8.0, act_bytes=1e5, param_bytes=1e6,
                             batches=(8,), micros=(2, 4))
    dump_case("small", model, topo, groups, seeds=[2, 3, 5, 11])

    # tests/test_acceptance.py:_random_instance (seeds with <= 4 groups)
    sys.path.insert(0, "/root/reference/pkg/tests")
    from test_acceptance import _random_instance
    for seed in range(1, 16):
        topo, groups, model = _random_instance(seed)
        if len(groups.fgs) > 4:
            continue
        dump_case(f"rand{seed}", model, topo, groups, seeds=[seed], beam_width=16)

    # error behaviour
    topo = rc.clique_topology([[2.0], [1.0]], memory=10.0, bandwidth=1e8, latency=0.001)
    groups = rc.make_groups(topo)
    model = rc.uniform_model(4, param_bytes=1e9, batches=(4,), micros=(2,))
    dump_case("err_memory", model, topo, groups, seeds=[0])

    # zero intra-group bandwidth: one link of a 2-device clique carries 0 B/s
    devs = [rc.device("a0", 1.0), rc.device("a1", 1.0), rc.device("b0", 1.0), rc.device("b1", 1.0)]
    links = []
    for u, v in itertools.combinations(devs, 2):
        same = u.id[0] == v.id[0]
        bw = (0.0 if (u.id, v.id) == ("a0", "a1") else 1e8) if same else 1e7
        links.append(rc.link(u.id, v.id, 0.01 if same else 1.0, bandwidth=bw, latency=0.001))
    topo = gp.build_topology(devs, links)
    groups = rc.make_groups(topo)
    model = rc.uniform_model(4, batches=(4,), micros=(2,))
    dump_case("err_intra_bw", model, topo, groups, seeds=[0])

    # zero-bandwidth gateway between the two groups
    links = []
    for u, v in itertools.combinations(devs, 2):
        same = u.id[0] == v.id[0]
        bw = 1e8 if same else (0.0 if (u.id, v.id) == ("a0", "b0") else 1e7)
        pt = 0.01 if same else (0.5 if (u.id, v.id) == ("a0", "b0") else 1.0)
        links.append(rc.link(u.id, v.id, pt, bandwidth=bw, latency=0.001))
    topo = gp.build_topology(devs, links)
    groups = rc.make_groups(topo)
    dump_case("err_gateway", model, topo, groups, seeds=[0])

    # single group (k = 1) and more groups than layers
    topo = rc.clique_topology([[2.0, 1.0, 1.0]], bandwidth=1e8, latency=0.001)
    groups = rc.make_groups(topo)
    dump_case("single_fg", rc.uniform_model(5, batches=(4, 8), micros=(1, 2)), topo, groups,
              seeds=[0, 1])
    topo = rc.clique_topology([[1.0], [2.0], [4.0]], bandwidth=1e8, latency=0.001)
    groups = rc.make_groups(topo)
    dump_case("too_few_layers", rc.uniform_model(2, batches=(4,), micros=(2,)), topo, groups,
              seeds=[0])

    if not args.skip_c4:
        dump_c4("c4", False)
        dump_c4("c4j", True)




def dump_grouping():
    """group_first_level / group_second_level of the reference on the
    topologies of tests/grouping_cases.py (rebuilt as reference objects)."""
    gp = geopipe()
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import grouping_cases as GC
    from geopipe.profiling import ClusterTopology, CommMetric, ComputeMetric, LinkInfo
    out = {}
    t0 = time.time()
    for name in GC.names():
        pt, bw, pc, tn, tc = GC.build(name)
        n = len(pc)
        ids = [f"d{i:04d}" for i in range(n)]  # string order == rank order
        devices = tuple(gp.DeviceSpec(id=i, memory_bytes=1e12, benchmark_times=(("b", 1.0),))
                        for i in ids)
        compute = {ids[i]: ComputeMetric(p_c=float(pc[i])) for i in range(n)}
        links = {frozenset((ids[i], ids[j])): LinkInfo(metric=CommMetric(p_t=float(pt[i, j])),
                                                        latency_seconds=0.0,
                                                        bandwidth_bytes_per_s=float(bw[i, j]))
                 for i in range(n) for j in range(i + 1, n)}
        topo = ClusterTopology(devices=devices, compute=compute, links=links)
        fgs = gp.group_first_level(topo, tn)
        rank = {d: i for i, d in enumerate(ids)}
        rows = []
        for fg in fgs:
            sgs = gp.group_second_level(fg, topo, tc)
            rows.append([[rank[d] for d in fg.member_device_ids], fg.intra_metric,
                         fg.aggregate_capacity, fg.min_intra_bandwidth,
                         [[[rank[d] for d in sg.member_device_ids], sg.aggregate_capacity]
                          for sg in sgs]])
        out[name] = rows
    G.save("grouping.json", out)
    print(f"grouping: {time.time() - t0:.1f}s", flush=True)


def dump_schedules():
    """Schedule digests (ops + transfers) of the sim_reports timings under
    every policy / adapter / async combination, and validate_schedule
    messages of seeded perturbations (tests/schedule_cases.py)."""
    gp = geopipe()
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import schedule_cases as SC
    from geopipe.timing import BoundaryTiming, StageTiming
    from geopipe.engine import OpKind, PipeOp
    from geopipe.schedule import Schedule
    rep = G.load("sim_reports.json")
    tims = []
    for d in rep["timings"]:
        st = tuple(StageTiming(f, b, w, sy, sy, op, 1.0) for f, b, w, sy, op in d["stages"])
        bd = tuple(BoundaryTiming(f"{i}-{i + 1}", lat, bw, act, grad)
                   for i, (lat, bw, act, grad) in enumerate(d["boundaries"]))
        tims.append(gp.PlanTiming(st, bd, d["batch"], d["microbatch"]))
    kinds = {k.value: k for k in OpKind}
    out = {"digests": {}, "violations": {}, "actions": {}}
    t0 = time.time()
    for ad in (0, 1):
        for asy in (0, 1):
            for pol in gp.Policy:
                key = f"{ad}:{asy}:{pol.value}:3"
                rows, viols, acts = [], [], []
                for i, t in enumerate(tims):
                    tr = gp.NetworkTrace(breakpoints={k: tuple(tuple(p) for p in v)
                                                      for k, v in rep["traces"][i].items()})
                    try:
                        r = gp.simulate_timing(t, pol, tr, adapter_enabled=bool(ad),
                                               config=gp.SimConfig(iterations=3,
                                                                   async_iterations=bool(asy)))
                    except gp.SchedulingBugError:
                        rows.append(None)
                        viols.append(None)
                        acts.append(None)
                        continue
                    rows.append(SC.digest(r.schedule.ops, r.transfers))
                    acts.append(SC.action_digest(r.adapter_actions))
                    pert = SC.perturb(r.schedule.ops, 1000 * i + 7)
                    sched = Schedule(
                        ops=tuple(tuple(PipeOp(kinds[k], s_, a, b, z, it, mb)
                                        for k, s_, a, b, z, it, mb in stage) for stage in pert),
                        makespan=r.makespan, policy=pol, num_stages=t.num_stages,
                        micro_count=t.batch // t.microbatch)
                    msgs = gp.validate_schedule(sched, t)
                    viols.append([len(msgs), SC.text_digest(msgs), msgs[:3]])
                out["digests"][key] = rows
                out["violations"][key] = viols
                out["actions"][key] = acts
    G.save("schedules.json", out)
    print(f"schedules: {time.time() - t0:.1f}s", flush=True)


def _cli_inputs(d):
    """cluster / model / trace files for the CLI goldens (tests/golden/cli)."""
    import itertools as it
    os.makedirs(d, exist_ok=True)
    files = {}

    def cluster_doc(pcs_by_clique, intra=0.01, cross=1.0, memory=1e15, bandwidth=1e8,
                    latency=0.001):  # the reference's tests/test_cli.py fixture shape
        devices, links, clique_of = [], [], {}
        for c, pcs in enumerate(pcs_by_clique):
            for k, p_c in enumerate(pcs):
                did = f"c{c}d{k}"
                clique_of[did] = c
                devices.append({"id": did, "memory_bytes": memory,
                                "benchmarks": [{"task": "bench", "seconds": 1.0 / p_c}]})
        ids = [x["id"] for x in devices]
        for a, b in it.combinations(ids, 2):
            p_t = intra if clique_of[a] == clique_of[b] else cross
            links.append({"a": a, "b": b, "alpha_s": p_t, "beta_s": 1e-3, "payload_bytes": 1e6,
                          "latency_s": latency, "bandwidth_Bps": bandwidth})
        return {"schema": "cluster/v1", "devices": devices, "links": links}

    def model_doc(layers=6, batches=(8,), micros=(2, 4)):
        return {"schema": "model/v1",
                "layers": [{"fwd_flops": 8.0, "activation_out_bytes": 1e5, "param_bytes": 1e6}
                           for _ in range(layers)],
                "global_batch_candidates": list(batches), "microbatch_candidates": list(micros)}

    def inst_docs(name):
        spec = I.config(name, True)
        devices = [{"id": i, "memory_bytes": mem, "region": f"r{r}",
                    "benchmarks": [{"task": "bench", "seconds": 1.0 / p_c}]}
                   for i, r, _, p_c, mem in spec.devices()]
        links = [{"a": u, "b": v, "alpha_s": I.LINK_PAYLOAD_M / bw, "beta_s": lat,
                  "payload_bytes": I.LINK_PAYLOAD_M, "latency_s": lat, "bandwidth_Bps": bw}
                 for u, v, lat, bw in spec.links()]
        model = {"schema": "model/v1",
                 "layers": [{"fwd_flops": f, "bwd_input_flops": bi, "bwd_weight_flops": bw_,
                             "activation_out_bytes": a, "param_bytes": pb}
                            for f, bi, bw_, a, pb in spec.layers],
                 "global_batch_candidates": list(spec.batches),
                 "microbatch_candidates": list(spec.micros)}
        return {"schema": "cluster/v1", "devices": devices, "links": links}, model

    def put(name, doc):
        path = os.path.join(d, name)
        with open(path, "w") as fh:
            json.dump(doc, fh, indent=1)
        files[name] = path

    put("small_cluster.json", cluster_doc([[4.0, 4.0], [2.0, 2.0], [1.0, 1.0]], cross=0.5))
    put("small_model.json", model_doc())
    put("hetero_cluster.json", cluster_doc([[8.0, 3.0, 3.0], [2.0, 2.0], [5.0]], cross=0.3))
    put("hetero_model.json", model_doc(layers=9, batches=(8, 16), micros=(2, 4)))
    for name in ("c1", "c2"):
        c, m = inst_docs(name)
        put(f"{name}_cluster.json", c)
        put(f"{name}_model.json", m)
    put("trace.json", {"schema": "trace/v1", "events": [
        {"link": "0-1", "t_s": 0.5, "multiplier": 0.4},
        {"link": "0-1", "t_s": 3.0, "multiplier": 1.0},
        {"link": "1-2", "t_s": 1.0, "multiplier": 0.25}]})
    put("hetero_plan_edited.json", {"schema": "plan/v1", "batch": 16, "microbatch": 4, "stages": [
        {"fg": "fg2", "layers": [0, 3], "split": {"kind": "uniform", "parts": []}},
        {"fg": "fg0", "layers": [3, 7], "split": {"kind": "asymmetric_pp", "parts": [
            ["fg0.sg0", 3, 5], ["fg0.sg1", 5, 7]]}},
        {"fg": "fg1", "layers": [7, 9], "split": {"kind": "asymmetric_dp",
                                                  "parts": [["fg1.sg0", 1.0]]}}]})
    put("bad_cluster.json", {"schema": "cluster/v1", "devices": [
        {"id": "x", "benchmarks": [{"task": "b", "seconds": 1.0}]}], "links": []})
    return files


def dump_cli():
    """Outputs of the reference CLI (src/cli.py) on committed input files."""
    from cli_cases import cli_commands, run_cli
    geopipe()
    from geopipe.cli import main as ref_main
    d = os.path.join(G.GOLDEN, "cli")
    _cli_inputs(d)
    import tempfile
    out = {}
    t0 = time.time()
    with tempfile.TemporaryDirectory() as o:
        for case, argv in cli_commands():
            args = [a.replace("{d}", d).replace("{o}", o) for a in argv]
            rc, so, se = run_cli(ref_main, args)
            files = {}
            for a in args:
                if a.startswith(o) and os.path.exists(a) and "--out" in args and \
                        args[args.index("--out") + 1] == a:
                    files[os.path.basename(a)] = open(a).read()
            out[case] = {"rc": rc, "stdout": so.replace(d, "{d}").replace(o, "{o}"),
                         "stderr": se.replace(d, "{d}").replace(o, "{o}"), "files": files}
    G.save("cli_outputs.json", out)
    print(f"cli: {time.time() - t0:.1f}s", flush=True)


def ref_from_doc(doc):
    """Reference objects (model, topology, groups) from a golden instance doc."""
    gp = geopipe()
    from geopipe.profiling import ClusterTopology, CommMetric, ComputeMetric, LinkInfo
    from geopipe.timing import GroupIndex
    from geopipe.grouping import FirstLevelGroup, SecondLevelGroup
    layers = tuple(gp.LayerSpec(*row) for row in doc["layers"])
    model = gp.ModelSpec(layers=layers, global_batch_candidates=tuple(doc["batches"]),
                         microbatch_candidates=tuple(doc["micros"]))
    devices = tuple(gp.DeviceSpec(id=i, memory_bytes=mem, benchmark_times=(("b", 1.0),))
                    for i, mem, _ in doc["devices"])
    compute = {i: ComputeMetric(p_c=pc) for i, _, pc in doc["devices"]}
    links = {frozenset((u, v)): LinkInfo(metric=CommMetric(p_t=pt), latency_seconds=lat,
                                         bandwidth_bytes_per_s=bw)
             for u, v, pt, lat, bw in doc["links"]}
    topo = ClusterTopology(devices=devices, compute=compute, links=links)
    fgs = [FirstLevelGroup(id=i, member_device_ids=tuple(m), intra_metric=im,
                           aggregate_capacity=cap, min_intra_bandwidth=mb)
           for i, m, im, cap, mb in doc["fgs"]]
    sgs = {f: [SecondLevelGroup(id=i, parent_fg_id=f, member_device_ids=tuple(m),
                                aggregate_capacity=cap) for i, m, cap in v]
           for f, v in doc["sgs"].items()}
    return model, topo, GroupIndex.build(fgs, sgs)


PLAN_COST_CASES = ["small", "c1", "c1j", "c2j", "c4", "err_intra_bw", "err_gateway",
                   "single_fg"] + [f"rand{i}" for i in range(1, 16)]


def random_plan(rng, model, groups):
    """A random explicit plan: subset and order of groups, cuts, batch /
    micro-batch, split kinds with arbitrary pipeline parts."""
    gp = geopipe()
    n = len(model.layers)
    fg_ids = sorted(groups.fgs)
    k = rng.randint(1, min(len(fg_ids), n))
    order = rng.sample(fg_ids, k)
    cuts = sorted(rng.sample(range(1, n), k - 1)) if k > 1 else []
    bounds = [0] + cuts + [n]
    b = rng.choice(model.global_batch_candidates)
    m = rng.choice([x for x in (1, 2, 4, 8, 16, b) if b % x == 0])
    stages = []
    for s, f in enumerate(order):
        a, e = bounds[s], bounds[s + 1]
        kind = rng.choice(list(gp.SplitKind))
        sgs = [sg.id for sg in groups.sgs_by_fg[f]]
        if kind is gp.SplitKind.ASYMMETRIC_PP:
            parts = []
            for _ in range(rng.randint(0, min(4, len(sgs) + 1))):
                x, y = sorted(rng.sample(range(a, e + 1), 2)) if e - a >= 1 else (a, a)
                parts.append((rng.choice(sgs), x, y))
            parts = tuple(parts)
        elif kind is gp.SplitKind.ASYMMETRIC_DP:
            parts = tuple((sg, 1.0 / len(sgs)) for sg in sgs)
        elif kind is gp.SplitKind.ASYMMETRIC_TP_DP:
            parts = tuple((d, 0.5, 0.5) for d in groups.fgs[f].member_device_ids)
        else:
            parts = ()
        stages.append(gp.StageAssignment(fg_id=f, layer_start=a, layer_end=e,
                                         intra_split=gp.IntraSplit(kind, parts)))
    return gp.ParallelPlan(stages=tuple(stages), batch_b=b, microbatch_m=m)


def dump_plan_costs():
    """plan_cost + build_plan_timing of the reference for random explicit
    plans (arbitrary splits) on the golden instances."""
    gp = geopipe()
    from geopipe.fileio import plan_to_dict
    from geopipe.timing import build_plan_timing
    out = {}
    t0 = time.time()
    for name in PLAN_COST_CASES:
        doc = G.load(f"{name}.json")["instance"]
        model, topo, groups = ref_from_doc(doc)
        rng = random.Random(sum(map(ord, name)) * 7 + 1)
        rows = []
        for _ in range(40):
            plan = random_plan(rng, model, groups)
            opt = rng.choice([0.0, 0.25])
            rec = {"plan": plan_to_dict(plan), "opt_seconds": opt}
            try:
                bd = gp.plan_cost(plan, topo, model, groups, opt_seconds=opt)
                rec["cost"] = G.breakdown_to_dict(bd)
                t = build_plan_timing(plan, topo, model, groups, opt_seconds=opt)
                rec["timing"] = timing_to_dict(t)
            except Exception as e:
                rec["error"] = type(e).__name__
            rows.append(rec)
        out[name] = rows
    G.save("plan_costs.json", out)
    print(f"plan costs: {time.time() - t0:.1f}s", flush=True)


def dump_search_seeds():
    """search_plan of the reference for seeds 0-20 on C1-C4 (integer and
    jittered), the SURVEY §8(c) parity protocol (3)."""
    gp = geopipe()
    out = {}
    t0 = time.time()
    for name in ("c1", "c1j", "c2", "c2j", "c4", "c4j"):
        model, topo, groups = build_reference(I.config(name[:2], name.endswith("j")))
        out[name] = {str(s): run_or_error(lambda: gp.search_plan(model, topo, groups,
                                                                 gp.SearchConfig(seed=s)))
                     for s in range(21)}
        print(f"search seeds {name}: {time.time() - t0:.1f}s", flush=True)
    G.save("search_seeds.json", out)


def dump_search_warnings():
    """The warnings search_plan logs (src/planner.py:321, :367), in order,
    and the exception it raises, for golden cases x seeds (logging enabled,
    records captured from the `geopipe.planner` logger)."""
    import logging as lg
    gp = geopipe()
    lg.disable(lg.NOTSET)
    out = {}

    class Cap(lg.Handler):
        def __init__(self):
            super().__init__()
            self.msgs = []

        def emit(self, rec):
            self.msgs.append(rec.getMessage())
    logger = lg.getLogger("geopipe.planner")
    for name in ("c1", "c2j", "small", "rand10", "err_memory", "err_gateway", "err_intra_bw",
                 "k5n9", "c4"):
        doc = G.load(f"{name}.json")
        model, topo, groups = G.instance_from_dict(doc["instance"])
        out[name] = {}
        for seed in ((0,) if name == "c4" else (0, 1, 2)):
            h = Cap()
            logger.addHandler(h)
            logger.propagate = False
            try:
                gp.search_plan(model, topo, groups, gp.SearchConfig(seed=seed))
                err = None
            except Exception as e:
                err = type(e).__name__
            logger.removeHandler(h)
            out[name][str(seed)] = {"warnings": h.msgs, "error": err}
    lg.disable(lg.CRITICAL)
    G.save("search_warnings.json", out)


def dump_region_sweep():
    """C2 region-grouping sweep with the reference: groups built
    as group_first_level would for each set partition of the regions, then
    group_second_level and exhaustive_plan."""
    gp = geopipe()
    from geopipe.grouping import FirstLevelGroup, _mean_intra_pt, _min_intra_bw
    from geopipe.timing import GroupIndex
    from paper_2505_15536_b200.replan import set_partitions
    spec = I.config("c2")
    model, topo, _ = build_reference(spec)
    regions = {}
    for i, r, _, _, _ in spec.devices():
        regions.setdefault(r, []).append(i)
    regs = [regions[r] for r in sorted(regions)]
    out = {"regions": regs, "groupings": []}
    t0 = time.time()
    for rgs in set_partitions(len(regs)):
        blocks = [sorted(d for rr, b in zip(regs, rgs) if b == v for d in rr)
                  for v in range(max(rgs) + 1)]
        tuples = sorted(tuple(sorted(b)) for b in blocks)
        fgs = [FirstLevelGroup(id=f"fg{idx}", member_device_ids=m,
                               intra_metric=_mean_intra_pt(m, topo),
                               aggregate_capacity=sum(topo.p_c(x) for x in m),
                               min_intra_bandwidth=_min_intra_bw(m, topo))
               for idx, m in enumerate(tuples)]
        sgs = {fg.id: gp.group_second_level(fg, topo, 0.3) for fg in fgs}
        groups = GroupIndex.build(fgs, sgs)
        rec = {"rgs": rgs, "blocks": blocks,
               "fgs": [[fg.id, list(fg.member_device_ids), fg.intra_metric, fg.aggregate_capacity,
                        fg.min_intra_bandwidth] for fg in fgs],
               "sgs": {f: [[sg.id, list(sg.member_device_ids), sg.aggregate_capacity] for sg in v]
                       for f, v in sgs.items()}}
        rec.update(run_or_error(lambda: gp.exhaustive_plan(model, topo, groups,
                                                           gp.SearchConfig(seed=0))))
        out["groupings"].append(rec)
    G.save("region_sweep.json", out)
    print(f"region sweep: {time.time() - t0:.1f}s", flush=True)


def dump_regroup_replan():
    """exhaustive_plan of the reference on C2 with per-snapshot p_t
    (tests/grouping_cases.py c2snap*), regrouped by the reference."""
    gp = geopipe()
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import grouping_cases as GC
    from geopipe.profiling import ClusterTopology, CommMetric, LinkInfo
    from geopipe.timing import GroupIndex
    spec = I.config("c2")
    model, topo, _ = build_reference(spec)
    ids = sorted(d.id for d in topo.devices)
    pos = {d: i for i, d in enumerate(ids)}
    out = {}
    t0 = time.time()
    for s in range(4):
        pt, _, _, tn, tc = GC.build(f"c2snap{s}")
        links = {}
        for key, info in topo.links.items():
            u, v = tuple(key)
            links[key] = LinkInfo(metric=CommMetric(p_t=float(pt[pos[u], pos[v]])),
                                  latency_seconds=info.latency_seconds,
                                  bandwidth_bytes_per_s=info.bandwidth_bytes_per_s)
        t2 = ClusterTopology(devices=topo.devices, compute=topo.compute, links=links)
        fgs = gp.group_first_level(t2, tn)
        groups = GroupIndex.build(fgs, {fg.id: gp.group_second_level(fg, t2, tc) for fg in fgs})
        r = run_or_error(lambda: gp.exhaustive_plan(model, t2, groups, gp.SearchConfig(seed=0)))
        out[f"c2snap{s}"] = r
    G.save("regroup_replan.json", out)
    print(f"regroup re-plan: {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
