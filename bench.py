#!/usr/bin/env python3
"""Benchmark: candidate plans evaluated/s and full re-plan latency on B200.

Workload (BASELINE.json configs[3], App. D "c4"): the 80-layer Llama-2-70B
cost table on 64 heterogeneous devices in 4 tiers.  One STEP = one exact
exhaustive re-plan of that instance = the arg-min over all 11,387,376
(b, m, stage order, layer cuts) candidates, each fully evaluated as the
reference's `_evaluate` does (split choice + memory feasibility + Eq. 1).
Under torchrun every rank re-plans its own bandwidth snapshot of C4 (C3
recipe, snapshot = rank), so per-GPU work is fixed ("scaling": "weak"); the
per-snapshot winners are all-gathered once at the end (16 B per rank).

  value      candidates/s over all ranks, tables resident in HBM, device time
             of the K3 launches (CUDA events on the engine stream, L2 flushed
             between steps, max over ranks)
  e2e        the same metric through the C-ABI with host buffers: per step
             gp_ctx_load (H2D of the packed instance + K1 tables) +
             gp_argmin_range (K3 + D2H of the winner) + gp_plan_detail
  roofline   K3 is FP64-issue-bound (no HBM traffic per candidate): achieved
             FP64 ops/s = (ops per candidate) x candidates/s against the
             FP64 add rate measured live on this GPU
  cpu_baseline  the C oracle port (oracle/, test infrastructure) on all host
             threads over the same full range, rank 0 at N=1 only

`--impl reference` times that CPU implementation alone (the reference arm).
"""

from __future__ import annotations

import argparse
import json

import numpy as np
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Algorithmic FP64 ops per candidate in the reference's operation order
# (11k - 5 = 39 for k = 4 stages): 6 per stage (C1*m, M*c,
# three adds, max) + 5 per boundary (c+x, fill+, x-c', max0, res+).
ALG_OPS_PER_CAND_C4 = 39
# FP64 instructions the K3 sweep actually issues per candidate (SASS of the
# paired-q inner loop: 56 DADD/DMUL/DSETP per 2 q steps x 2 batch sizes).
K3_ISSUED_FP64_PER_CAND = 14
# dram__bytes_read.sum + write of one K3 launch after an L2 flush (ncu launch
# list of this bench, profiles/r1e_launches_bench.csv: 704,256 B read, 0 written)
K3_DRAM_BYTES = 704256


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.2)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            p = [x.strip() for x in l.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": mx or None, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(total, threads, target_s=10.0):
    """Oracle port on host cores over a bounded prefix of the range."""
    from oracle import oracle as O
    from paper_2505_15536_b200 import instances
    from paper_2505_15536_b200.layout import PackedInstance
    model, topo, groups = instances.load("c4")
    packed = PackedInstance(model, topo, groups, 1.25)
    # calibrate on a short prefix, then run ~target_s of work
    n0 = 200_000
    t = time.perf_counter()
    O.argmin_range(packed, 0, n0, threads=threads)
    dt = time.perf_counter() - t
    n = int(min(total, max(n0, n0 * target_s / max(dt, 1e-6))))
    t = time.perf_counter()
    st, best = O.argmin_range(packed, 0, n, threads=threads)
    dt = time.perf_counter() - t
    return n / dt, n, dt


def extra_sections(eng, packed, total, local, args, world):
    """Secondary measurements of the other kernels (each self-timed on the
    engine stream with CUDA events; inputs device-resident unless noted)."""
    import torch
    from paper_2505_15536_b200 import instances, replan, simulate
    from paper_2505_15536_b200.engine import Engine
    from paper_2505_15536_b200.enumeration import decode_indices, composition_table
    from paper_2505_15536_b200.layout import PackedInstance
    out = {}
    dev = torch.device("cuda", local)
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)

    def timed(fn, reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        fn()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            ev[0].record(stream)
        for _ in range(reps):
            fn()
        with torch.cuda.stream(stream):
            ev[1].record(stream)
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / reps

    # ---- K2: explicit batch of 2x10^7 random C4 candidates (> L2: HBM-bound)
    N = N_K2 = 20_000_000
    rng = np.random.default_rng(4)
    idx = rng.integers(0, total, size=N)
    order, counts, bm = decode_indices(80, 4, idx, composition_table(80, 4))
    d_o = torch.from_numpy(np.ascontiguousarray(order)).to(dev)
    d_c = torch.from_numpy(np.ascontiguousarray(counts)).to(dev)
    d_b = torch.from_numpy(np.ascontiguousarray(bm)).to(dev)
    d_cost = torch.empty(N, dtype=torch.float64, device=dev)
    d_st = torch.empty(N, dtype=torch.uint8, device=dev)
    ms = timed(lambda: eng.eval_batch_device(4, N, d_o.data_ptr(), d_c.data_ptr(), d_b.data_ptr(),
                                             d_cost.data_ptr(), d_st.data_ptr()), 20)
    bytes_per = 2 * 4 + 1 + 8 + 1
    hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6536.0
    out["k2_explicit_batch"] = {
        "candidates": N, "ms_per_launch": ms, "candidates_per_s": N / (ms * 1e-3),
        "roofline": {"bound": "hbm", "bytes_per_candidate": bytes_per,
                     "achieved_gbs": N * bytes_per / (ms * 1e-3) / 1e9, "peak_gbs": hbm,
                     "frac": N * bytes_per / (ms * 1e-3) / 1e9 / hbm},
        "note": "360 MB of candidates + results per launch (> 126 MB L2); order/counts/bm u8 "
                "in, cost f64 + status u8 out. k2_eval_batch_q4: stage codes in shared memory "
                "decide the 85 % memory-infeasible candidates without table gathers; the "
                "feasible ones are queued per warp and evaluated 32 at a time (stage-table and "
                "boundary gathers from L2). ncu (profiles/r1e_k2_eval_batch_q4_ncu_raw.csv): "
                "ALU pipe 57 %, long-scoreboard stalls dominant, DRAM 1.8 TB/s"}

    # ---- K5: 1F1B makespans of 10^5 of those C4 candidates
    # feasible candidates only (infeasible ones are rejected before simulating)
    cost_h = d_cost.cpu().numpy()
    feas = np.nonzero(np.isfinite(cost_h[:5_000_000]))[0][:200_000]
    NS = int(feas.size)
    eng.sim_candidates(order[feas], counts[feas], bm[feas], 1, 0.0)  # warm-up at full size
    t0 = time.perf_counter()
    msk, stk = eng.sim_candidates(order[feas], counts[feas], bm[feas], 1, 0.0)
    el = time.perf_counter() - t0
    out["k5_sim_1f1b"] = {"simulations": NS, "host_call_s": el, "simulations_per_s": NS / el,
                          "ok": int((stk == 0).sum()),
                          "note": "memory-feasible C4 plans, 1F1B, iterations=1; one thread per "
                                  "simulation; includes H2D/D2H of the batch"}

    # ---- K6: C3 - 10^4 bandwidth snapshots of C2, exact re-plan each
    spec = instances.config("c2")
    m2, t2, g2 = instances.build(spec)
    p2 = PackedInstance(m2, t2, g2, 1.25)
    nsnap = 10_000
    bws = replan.bandwidth_matrices(p2, [instances.snapshot_multipliers(spec, j)
                                         for j in range(nsnap)])
    e2 = Engine(local).load(p2)
    e2.replan_snapshots(bws)  # warm-up at full size (allocations outside the timed call)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b2, s2 = e2.replan_snapshots(bws)
    el = time.perf_counter() - t0
    lat = []
    for j in range(20):
        t1 = time.perf_counter()
        e2.replan_snapshots(bws[j:j + 1])
        lat.append(time.perf_counter() - t1)
    c2_total = e2.space_size()
    out["k6_snapshot_replan"] = {
        "snapshots": nsnap, "candidates_per_snapshot": c2_total, "host_call_s": el,
        "snapshots_per_s": nsnap / el, "candidates_per_s": nsnap * c2_total / el,
        "single_snapshot_latency_ms_p50": statistics.median(lat) * 1e3,
        "ok": int((s2 == 0).sum()),
        "note": "C3 recipe (App. D) on C2; bandwidth matrices H2D inside the call"}
    if world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        t0 = time.perf_counter()
        for j in range(5):
            m3, t3, g3 = instances.build(spec, instances.snapshot_multipliers(spec, j))
            p3 = PackedInstance(m3, t3, g3, 1.25)
            O.argmin_range(p3, 0, c2_total, threads=args.cpu_threads or os.cpu_count())
        out["k6_snapshot_replan"]["cpu_port_ms_per_snapshot"] = (time.perf_counter() - t0) / 5 * 1e3
    e2.close()

    # ---- C5: throughput vs batch size N
    eng.load(packed)
    sweep = {}
    for N in (10**3, 10**4, 10**5, 10**6, total):
        ms3 = timed(lambda: eng.argmin_range_async(0, N), 20)
        sweep[str(N)] = {"k3_range_ms": ms3, "k3_candidates_per_s": N / (ms3 * 1e-3)}
        if N <= N_K2:
            ms2 = timed(lambda: eng.eval_batch_device(4, N, d_o.data_ptr(), d_c.data_ptr(),
                                                      d_b.data_ptr(), d_cost.data_ptr(),
                                                      d_st.data_ptr()), 20)
            sweep[str(N)].update({"k2_explicit_ms": ms2, "k2_candidates_per_s": N / (ms2 * 1e-3)})
    eng.argmin_fetch()
    # N = 10^8: C4 under 9 bandwidth snapshots in one K6 launch
    spec4s = instances.config("c4")
    bw9 = replan.bandwidth_matrices(packed, [instances.snapshot_multipliers(spec4s, j)
                                             for j in range(9)])
    eng.replan_snapshots(bw9)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        eng.replan_snapshots(bw9)
    el9 = (time.perf_counter() - t0) / 5
    sweep[str(9 * total)] = {"k6_9_snapshots_host_call_ms": el9 * 1e3,
                             "candidates_per_s": 9 * total / el9}
    eng.load(packed)
    out["c5_batch_sweep"] = {
        "rows": sweep,
        "note": "K3 over the first N ranks of C4 (device time per call, L2 warm), K2 over the "
                "first N of the 2x10^7 random explicit C4 candidates, and N = 9 x C4 through "
                "K6 (host call incl. H2D of the bandwidth matrices)"}

    # ---- C2 region-grouping sweep (BASELINE config 2)
    from paper_2505_15536_b200.replan import region_grouping_sweep
    from paper_2505_15536_b200 import SearchConfig as _SC
    m2s, t2s, _ = instances.load("c2")
    regs = {}
    for i_, r_, _, _, _ in instances.config("c2").devices():
        regs.setdefault(r_, []).append(i_)
    regs = [regs[r_] for r_ in sorted(regs)]
    region_grouping_sweep(m2s, t2s, regs, _SC(seed=0), engine=eng)
    lat = []
    for _ in range(5):
        t0 = time.perf_counter()
        res_s, best_s = region_grouping_sweep(m2s, t2s, regs, _SC(seed=0), engine=eng)
        lat.append(time.perf_counter() - t0)
    n_eval = sum(r.evaluated for _, r in res_s if hasattr(r, "evaluated"))
    out["c2_region_grouping_sweep"] = {
        "groupings": len(res_s), "candidates": n_eval,
        "sweep_ms_p50": statistics.median(lat) * 1e3,
        "best_cost": res_s[best_s][1].breakdown.plan_cost,
        "note": "5 set partitions of the 3 regions: device grouping (K7 fixed partition), "
                "exhaustive re-plan each (K1 + K3/K2 + detail); the unmodified Python reference "
                "takes ~3 s for the same sweep on this container's CPU"}
    eng.load(packed)

    # ---- K7: regroup C4 (64 devices) per p_t snapshot
    from paper_2505_15536_b200 import grouping as GR
    _, t4, _ = instances.load("c4")
    ids4, pt4, bw4, pc4 = GR.topology_arrays(t4)
    spec4 = instances.config("c4")
    reg = np.array([{i: r for i, r, _, _, _ in spec4.devices()}[d] for d in ids4])
    nreg = int(reg.max()) + 1
    rng7 = np.random.default_rng(7)
    n7 = 1000
    fac = np.where(rng7.random((n7, nreg, nreg)) < 0.5, rng7.uniform(1.0, 3.0, (n7, nreg, nreg)), 1.0)
    fac = np.triu(fac) + np.triu(fac, 1).transpose(0, 2, 1)
    pts = pt4[None] * fac[:, reg][:, :, reg]
    GR.group_hierarchies(pts, bw4, pc4, engine=eng)  # warm-up at full size
    t0 = time.perf_counter()
    hs = GR.group_hierarchies(pts, bw4, pc4, engine=eng)
    el = time.perf_counter() - t0
    lat = []
    for j in range(20):
        t1 = time.perf_counter()
        GR.group_hierarchies(pts[j:j + 1], bw4, pc4, engine=eng)
        lat.append(time.perf_counter() - t1)
    out["k7_regroup"] = {
        "snapshots": n7, "devices": int(len(ids4)), "host_call_s": el,
        "snapshots_per_s": n7 / el, "single_snapshot_latency_ms_p50": statistics.median(lat) * 1e3,
        "groups_seen": sorted({len(h.fg_capacity) for h in hs}),
        "note": "group_first_level + group_second_level per C4 p_t snapshot, one CTA each; "
                "p_t matrices H2D inside the call; the Python reference takes ~50 ms per "
                "grouping at 64 devices (SURVEY §8(f))"}
    if world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        t0 = time.perf_counter()
        for j in range(20):
            O.group_hierarchy(pts[j], bw4, pc4)
        out["k7_regroup"]["cpu_port_ms_per_snapshot"] = (time.perf_counter() - t0) / 20 * 1e3

    # ---- K5 full: adapter + asynchronous iterations under degrading traces
    rng5 = np.random.default_rng(5)
    n5 = 100_000
    S5 = rng5.integers(2, 6, n5)
    tims = []
    for i in range(n5):
        S = int(S5[i])
        tims.append(simulate.make_timing(
            fwd=list(rng5.uniform(0.2, 2.0, S)), bwd=list(rng5.uniform(0.2, 2.0, S)),
            wgt=list(rng5.uniform(0.05, 1.0, S)), transfer=list(rng5.uniform(0.05, 2.5, S - 1)),
            microbatch=int(rng5.choice([2, 4, 8])), micro_count=int(rng5.integers(4, 17)),
            sync=list(rng5.uniform(0.0, 0.5, S)), opt=list(rng5.uniform(0.0, 0.3, S)),
            latency=float(rng5.uniform(0.0, 0.2))))
    traces = [{f"{b}-{b + 1}": [[float(t), float(m)] for t, m in
                                zip(np.sort(rng5.uniform(0, 60, 4)), rng5.choice([0.25, 0.5, 1.0], 4))]
               for b in range(4)} for _ in range(64)]
    arr5 = simulate.pack_timings(tims)
    tr5 = simulate.pack_traces(traces)
    ti5 = np.arange(n5) % 64
    # warm-up at full size (queue-scratch allocation outside the timed call)
    eng.simulate_report(arr5, n5, 3, 3, tr5, 64, ti5, adapter=True, async_iterations=True)
    t0 = time.perf_counter()
    reps5, _, st5 = eng.simulate_report(arr5, n5, 3, 3, tr5, 64, ti5, adapter=True,
                                        async_iterations=True)
    el = time.perf_counter() - t0
    out["k5_full_adapter"] = {
        "simulations": n5, "host_call_s": el, "simulations_per_s": n5 / el,
        "ok": int((st5 == 0).sum()),
        "adapter_actions": int(sum(r.adapter_actions for r in reps5)),
        "note": "ZB_COMPACT, 3 iterations, DynamicBatchAdapter on, asynchronous iterations, "
                "64 breakpoint traces; one thread per simulation; includes H2D/D2H"}
    if world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        t0 = time.perf_counter()
        O.sim_reports(arr5, 5000, 3, 3, tr5, ti5[:5000], adapter=True, async_iterations=True)
        out["k5_full_adapter"]["cpu_port_simulations_per_s_1thread"] = 5000 / (time.perf_counter() - t0)

    # ---- K4: exact re-plan of spaces far beyond enumeration (k = 8 groups)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_bnb import _many_group_instance
    for (k, n, seed) in ((6, 80, 6), (8, 80, 8)):
        mk, tk, gk = _many_group_instance(k, n, seed)
        pk = PackedInstance(mk, tk, gk, 1.25)
        ek = Engine(local).load(pk)
        ek.argmin_bnb()
        lat = []
        for _ in range(5):
            t0 = time.perf_counter()
            bb = ek.argmin_bnb()
            lat.append(time.perf_counter() - t0)
        out[f"k4_bnb_k{k}_n{n}"] = {
            "candidates_in_space": int(ek.space_size()), "replan_ms_p50": statistics.median(lat) * 1e3,
            "cost": bb.cost,
            "note": "exact arg-min by branch-and-bound with the exact-in-reals DP bound "
                    "(same winner as exhaustive enumeration; tests/test_bnb.py)"}
        ek.close()

    # ---- drop-in search_plan (beam, host RNG driver + K2 batches) on C4
    from paper_2505_15536_b200 import SearchConfig, search_plan
    model, topo, groups = instances.load("c4")
    search_plan(model, topo, groups, SearchConfig(seed=0), engine=eng)
    t0 = time.perf_counter()
    r = search_plan(model, topo, groups, SearchConfig(seed=0), engine=eng)
    out["search_plan_c4"] = {"seconds": time.perf_counter() - t0, "evaluated": r.evaluated,
                             "note": "reference Python driver (RNG, sort) on the host, one "
                                     "K2 batch per beam iteration across all (b, m) passes"}
    eng.load(packed)
    return out


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    threads = args.cpu_threads or os.cpu_count()
    from oracle import oracle as O
    from paper_2505_15536_b200 import instances
    from paper_2505_15536_b200.layout import PackedInstance
    model, topo, groups = instances.load("c4")
    packed = PackedInstance(model, topo, groups, 1.25)
    total = O.space_size(packed)
    # each step: a bounded sample (contiguous prefix) of the full re-plan
    n0 = 100_000
    t = time.perf_counter()
    O.argmin_range(packed, 0, n0, threads=threads)
    dt0 = time.perf_counter() - t
    per_step = int(min(total, max(n0, n0 * 4.0 / max(dt0, 1e-6))))
    for _ in range(args.warmup):
        O.argmin_range(packed, 0, min(per_step, n0), threads=threads)
    t = time.perf_counter()
    for _ in range(args.steps):
        O.argmin_range(packed, 0, per_step, threads=threads)
    el = time.perf_counter() - t
    rate = per_step * args.steps / el
    line = {
        "impl": "reference", "metric": "candidate plans evaluated/sec", "value": rate,
        "unit": "candidates/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "c4-exhaustive-replan", "candidates_per_replan": total,
                   "layers": 80, "devices": 64, "groups": 4},
        "cpu_baseline": {"value": rate, "unit": "candidates/s", "cores": threads,
                         "kind": "port",
                         "sample": f"first {per_step} candidates of the C4 exhaustive range "
                                   f"per step (oracle/oracle.c, {threads} threads)"},
        "e2e": {"value": rate, "unit": "candidates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    rank, world, local = dist_env()
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2505_15536_b200 import instances, abi
    from paper_2505_15536_b200.engine import Engine, fp64_peak
    from paper_2505_15536_b200.layout import PackedInstance

    model, topo, groups = instances.load("c4", snapshot=rank if world > 1 else None)
    packed = PackedInstance(model, topo, groups, 1.25)
    eng = Engine(local).load(packed)
    total = eng.space_size()
    stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", local))
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident throughput (value) --------------------------------
    for _ in range(max(3, args.warmup)):
        with torch.cuda.stream(stream):
            flush.zero_()
        eng.argmin_range_async(0, total)
    eng.argmin_fetch()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()               # evict L2 (outside the events)
                starts[i].record(stream)
            eng.argmin_range_async(0, total)
            with torch.cuda.stream(stream):
                ends[i].record(stream)
        torch.cuda.synchronize()
    barrier()
    kernel_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    best = eng.argmin_fetch()
    dev_ms = sum(kernel_ms)
    t = torch.tensor([dev_ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms_max = float(t.item())
    value = world * total * args.steps / (dev_ms_max * 1e-3)

    # ---- end-to-end through the C-ABI with host buffers (e2e) --------------
    h2d = sum(getattr(packed, a).nbytes for a in (
        "fwd", "bwd_in", "bwd_w", "act", "param", "batch", "micro", "p_c", "memory",
        "id_rank", "p_t", "lat", "bw", "fg_member_offset", "fg_members", "fg_capacity",
        "fg_min_bw", "fg_has_min_bw", "fg_sg_offset", "sg_member_offset", "sg_members",
        "sg_capacity"))
    import ctypes
    d2h = 24 + 8 + 4 * 4 + 32 + ctypes.sizeof(abi.GpPlanInfo)  # SolveOut record
    lat = []
    for i in range(args.warmup + args.steps):
        barrier()
        t0 = time.perf_counter()
        b, info = eng.replan(packed)     # graph: pinned H2D + K1 + K3 + detail + D2H
        el = time.perf_counter() - t0
        if i >= args.warmup:
            lat.append(el)
    e2e_s = torch.tensor([sum(lat)], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = world * total * args.steps / float(e2e_s.item())

    # ---- gather per-snapshot winners (tiny collective) -----------------------
    rec = torch.tensor([best.cost, float(best.index)], dtype=torch.float64,
                       device=f"cuda:{local}")
    if world > 1:
        out = [torch.empty_like(rec) for _ in range(world)]
        dist.all_gather(out, rec)
        winners = [(float(o[0]), int(o[1])) for o in out]
    else:
        winners = [(best.cost, best.index)]

    if rank == 0:
        peak = fp64_peak(local)
        per_launch_ms = dev_ms_max / args.steps
        cand_rate_1gpu = total / (per_launch_ms * 1e-3)
        achieved = ALG_OPS_PER_CAND_C4 * cand_rate_1gpu
        line = {
            "metric": "candidate plans evaluated/sec", "value": value,
            "unit": "candidates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_launch_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (App. D C4 recipe; snapshot = rank)",
            "config": {"workload": "c4-exhaustive-replan", "candidates_per_replan": total,
                       "layers": 80, "devices": 64, "groups": 4,
                       "batch_micro_pairs": len(packed.batches) * len(packed.micros),
                       "l2": "flushed between steps (256 MiB write)",
                       "parallelism": f"snapshot-per-gpu x{world}"},
            "replan_latency_ms": {"device_p50": statistics.median(kernel_ms),
                                  "device_min": min(kernel_ms),
                                  "c_abi_host_p50": statistics.median(lat) * 1e3},
            "e2e": {"value": e2e_value, "unit": "candidates/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "path": "gp_replan: one CUDA graph of pinned H2D + K1 + K3 + detail + D2H"},
            "roofline": {"bound": "fp64", "achieved": achieved / 1e12, "peak": peak / 1e12,
                         "unit": "TFLOP/s", "frac": achieved / peak, "traffic": K3_DRAM_BYTES,
                         "algorithmic_ops_per_candidate": ALG_OPS_PER_CAND_C4,
                         "issued_fp64_per_candidate": K3_ISSUED_FP64_PER_CAND,
                         "issued_frac": K3_ISSUED_FP64_PER_CAND * cand_rate_1gpu / peak,
                         "peak_source": "FP64 DADD issue rate measured live on this GPU "
                                        "(gp_diag_fp64_peak); not in MEASURED_PEAKS.json",
                         "kernel": "k3_sweep"},
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            "winners": winners[:8],
        }
        if not args.no_cpu_baseline and world == 1:
            threads = args.cpu_threads or os.cpu_count()
            rate, n, dt = cpu_baseline(total, threads)
            line["cpu_baseline"] = {
                "value": rate, "unit": "candidates/s", "cores": threads, "kind": "port",
                "sample": f"first {n} candidates of the C4 exhaustive range, "
                          f"{dt:.1f} s on {threads} host threads (oracle/oracle.c)"}
            line["cpu_replan_s_extrapolated"] = total / rate
        if not args.no_extra:
            line["extra"] = extra_sections(eng, packed, total, local, args, world)
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
