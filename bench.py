#!/usr/bin/env python3
"""Benchmark: candidate plans evaluated/s and exact re-plan latency on B200.

Workload (BASELINE.json configs[2]+[3]): the C4 instance - the
80-layer Llama-2-70B cost table on 64 heterogeneous devices in 4 tiers - under
the C3 bandwidth-fluctuation recipe.  One STEP = the exact exhaustive re-plan
of a fixed batch of S = 128 bandwidth snapshots (snapshot j = App. D recipe
with seed j), i.e. 128 x 11,387,376 candidates, each fully evaluated as the
reference's `_evaluate` does (split choice + memory feasibility + Eq. 1) and
reduced to that snapshot's arg-min under the reference key.  Under torchrun
the snapshots are partitioned by index over the N ranks (contiguous shards,
no data-path communication) and the per-snapshot winners (16 B each) are
all-gathered over NCCL inside the step, so every rank ends with all 128 plans
(fixed total work: "scaling": "strong").

  value      candidates/s over all ranks with the bandwidth matrices resident
             in HBM: CUDA events on the engine stream around each step (K6
             table patch + K3 sweep + NCCL all-gather), L2 flushed between
             steps, max over ranks
  e2e        the same step through the public API with host buffers:
             distributed.replan_snapshots_sharded (single GPU:
             replan.replan_snapshots) - pinned H2D of the matrices, K6,
             all-gather of the winners from device memory, one D2H - wall
             clock, max over ranks
  roofline   the sweep kernel is FP64-issue-bound (tables in shared memory,
             no per-candidate HBM traffic): the record sweep's 10.5
             algorithmic FP64 ops per C4 candidate (sweep_ops_per_candidate;
             the reference order's 11k - 5 = 39 is reported beside it) x
             candidates per launch over the launch's CUDA-event duration,
             against the FP64 add rate measured live on this GPU
  cpu_baseline  the C oracle port (oracle/, test infrastructure) on the host
             threads over a bounded prefix of one snapshot, rank 0 at N=1,
             plus the unmodified Python reference on a sample when it is
             importable (baseline/_ref)
  scaling_rows  the other sharded paths at the same N: one C4 re-plan
             item-sharded with the NCCL tuple arg-min, the BASELINE 10^6
             sampled C4 candidates in N K2 chunks + arg-min, C3 (C2 x 10^4
             snapshots) partitioned by index, and weak scaling

`--impl reference` times the CPU implementation alone (the reference arm).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# rank 0 prints exactly one JSON line on stdout: NCCL's version banner (the
# GPU boxes export NCCL_DEBUG=VERSION) and warnings go to stderr
if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
    os.environ["NCCL_DEBUG"] = "WARN"
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

# FP64 ops per candidate of independent evaluation in the reference's operation
# order (11k - 5 = 39 for k = 4 stages): 6 per stage (C1*m,
# M*c, three adds, max) + 5 per boundary (c+x, fill+, x-c', max0, res+).
REF_OPS_PER_CAND_C4 = 39
# FP64 ops per candidate the sweep's algorithm needs.  A run
# fixes stages 0..k-3, so only the last two stages vary along q, and the
# record sweep (k3_sweep_rec, the K6 batch kernel) tabulates per item the
# terms that depend on (a, q) or q alone (D2 = max0(x1 - c2), G2 = c2 + x2,
# D3 = max0(x2 - c3), M_b*c3).  Per q, shared by the NB batch sizes: res2,
# fill3, res3 = 3 adds; per (q, b): M_b*c2, 6 adds for t2 and t3 and the two
# compares against the arg-min bound (cost = max(mx1, t2, t3) <= T) = 9.
# NB = 2: (3 + 2 * 9) / 2 = 10.5 per candidate (the per-run and per-item
# work adds ~0.3).  39 x rate exceeds the FP64 pipe peak (the prefix work is
# shared), so the roofline uses this count; the reference-order equivalent
# rate is reported beside it.
def sweep_ops_per_candidate(nb):
    return (3 + 9 * nb) / nb


# Measured by ncu on the sweep kernel of this workload (not in-run):
# profiles/r2_k6_sweep_ncu_summary.json (issued FP64 per candidate from the
# FP64 pipe activity, and dram__bytes_read.sum + dram__bytes_write.sum of one
# launch; raw metrics in the .csv of the same name).
NCU_SOURCE = "profiles/r2_k6_sweep_ncu_summary.json"
SWEEP_ISSUED_FP64_PER_CAND = None
SWEEP_DRAM_BYTES = None
S_TOTAL = 128


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--snapshots", type=int, default=S_TOTAL)
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-rows", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def pct(xs, q):
    xs = sorted(xs)
    if not xs:
        return float("nan")
    return xs[min(len(xs) - 1, int(math.ceil(q / 100.0 * len(xs))) - 1)]


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def load_ncu_constants():
    """issued FP64 per candidate and DRAM bytes per launch of the sweep, from
    the committed ncu capture of this workload (None when absent)."""
    global SWEEP_ISSUED_FP64_PER_CAND, SWEEP_DRAM_BYTES
    path = os.path.join(ROOT, "profiles", "r2_k6_sweep_ncu_summary.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        SWEEP_ISSUED_FP64_PER_CAND = d.get("issued_fp64_per_candidate")
        SWEEP_DRAM_BYTES = d.get("dram_bytes_per_launch")


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
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        # nvidia-smi's NVML start-up takes driver locks for a few hundred ms;
        # let it reach its steady polling before the timed region starts
        time.sleep(1.0)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.05)
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


def cpu_baseline(packed, total, threads, target_s=10.0):
    """Oracle port on host cores over a bounded prefix of one snapshot's space."""
    from oracle import oracle as O
    n0 = 200_000
    t = time.perf_counter()
    O.argmin_range(packed, 0, n0, threads=threads)
    dt = time.perf_counter() - t
    n = int(min(total, max(n0, n0 * target_s / max(dt, 1e-6))))
    t = time.perf_counter()
    O.argmin_range(packed, 0, n, threads=threads)
    dt = time.perf_counter() - t
    return n / dt, n, dt


def python_reference_rate(spec_name="c4", n_cand=2000, procs=None):
    """The unmodified Python reference (`geopipe.planner._evaluate`, fresh cache
    per candidate, logging disabled) on a random sample of the C4 space: one
    process, and `procs` processes over contiguous shards.  None when the
    reference is not importable (baseline/_ref or /root/reference)."""
    import importlib
    import logging
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "geopipe")) and p not in sys.path:
            sys.path.insert(0, p)
    try:
        gp = importlib.import_module("geopipe")
    except ImportError:
        return None
    logging.disable(logging.CRITICAL)
    from concurrent.futures import ProcessPoolExecutor
    t0, t1 = _py_ref_worker((spec_name, 0, n_cand, 0.0))
    rate1 = n_cand / (t1 - t0)
    t0, t1 = _py_ref_worker((spec_name, 0, n_cand, 0.0, True))
    rate_log = n_cand / (t1 - t0)
    logging.disable(logging.CRITICAL)
    procs = procs or os.cpu_count() or 1
    start = time.time() + 6.0  # every worker has built its instance by then
    with ProcessPoolExecutor(procs) as ex:
        spans = list(ex.map(_py_ref_worker, [(spec_name, s + 1, n_cand, start)
                                             for s in range(procs)]))
    el = max(b for _, b in spans) - min(a for a, _ in spans)
    return {"value_1proc": rate1, "value_1proc_as_shipped_logging": rate_log,
            "value_all": procs * n_cand / el, "processes": procs,
            "unit": "candidates/s",
            "sample": f"{n_cand} random C4 candidates per process (fresh _evaluate cache each, "
                      "logging disabled); all processes start together",
            "source": "geopipe (unmodified reference) " + getattr(gp, "__version__", "")}


def _ref_import():
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "geopipe")) and p not in sys.path:
            sys.path.insert(0, p)
    import geopipe as gp
    return gp


def _ref_instance(gp, spec, multipliers=None):
    """(model, topology, groups) built with the reference's own constructors
    and grouping from an App. D spec (bandwidth x multiplier per pair)."""
    from geopipe.timing import GroupIndex
    devs = [gp.DeviceSpec(id=i, memory_bytes=mem, benchmark_times=(("bench", 1.0 / p_c),))
            for i, _, _, p_c, mem in spec.devices()]
    meas = []
    for u, v, lat, bw in spec.links():
        if multipliers is not None:
            bw = bw * multipliers[(min(u, v), max(u, v))]
        meas.append(gp.LinkMeasurement(endpoints=frozenset((u, v)), alpha_seconds=1e8 / bw,
                                       beta_seconds=lat, payload_bytes_m=1e8, latency_seconds=lat,
                                       bandwidth_bytes_per_s=bw))
    topo = gp.build_topology(devs, meas)
    fgs = gp.group_first_level(topo, 0.3)
    groups = GroupIndex.build(fgs, {f.id: gp.group_second_level(f, topo, 0.3) for f in fgs})
    model = gp.ModelSpec(layers=tuple(gp.LayerSpec(*r) for r in spec.layers),
                         global_batch_candidates=tuple(spec.batches),
                         microbatch_candidates=tuple(spec.micros))
    return model, topo, groups


def python_reference_replan(n_search=5, n_exhaustive=2):
    """The unmodified Python reference's re-plan per C3 bandwidth snapshot of
    C2: rebuild the topology from the scaled link
    measurements, regroup, then search_plan (p50 over ``n_search`` snapshots)
    and exhaustive_plan (p50 over ``n_exhaustive``); logging disabled.  None
    when the reference is not importable."""
    import logging
    try:
        gp = _ref_import()
    except ImportError:
        return None
    from paper_2505_15536_b200 import instances
    logging.disable(logging.CRITICAL)
    spec = instances.config("c2")
    ts, te = [], []
    for j in range(max(n_search, n_exhaustive)):
        mult = instances.snapshot_multipliers(spec, j)
        if j < n_search:
            t0 = time.perf_counter()
            m, t, g = _ref_instance(gp, spec, mult)
            gp.search_plan(m, t, g, gp.SearchConfig(seed=0))
            ts.append(time.perf_counter() - t0)
        if j < n_exhaustive:
            t0 = time.perf_counter()
            m, t, g = _ref_instance(gp, spec, mult)
            gp.exhaustive_plan(m, t, g, gp.SearchConfig(seed=0))
            te.append(time.perf_counter() - t0)
    logging.disable(logging.NOTSET)
    return {"c3_search_plan_s_p50": statistics.median(ts), "snapshots_search": len(ts),
            "c3_exhaustive_plan_s_p50": statistics.median(te), "snapshots_exhaustive": len(te),
            "note": "per C3 snapshot of C2: topology rebuilt from the scaled link measurements, "
                    "group_first_level / group_second_level, then the planner (one process)"}


def _py_ref_worker(args):
    spec_name, seed, n_cand, start = args[:4]
    as_shipped = len(args) > 4 and args[4]
    import logging
    import random
    root = logging.getLogger()
    saved = root.handlers[:]
    if as_shipped:  # the reference's per-plan warnings formatted and written (to /dev/null)
        logging.disable(logging.NOTSET)
        root.handlers[:] = [logging.StreamHandler(open(os.devnull, "w"))]
    else:
        logging.disable(logging.CRITICAL)
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "geopipe")) and p not in sys.path:
            sys.path.insert(0, p)
    from geopipe.planner import Candidate, _evaluate
    from geopipe.timing import GroupIndex
    import geopipe as gp
    from paper_2505_15536_b200 import instances
    from paper_2505_15536_b200.enumeration import decode_indices, composition_table
    # the instance built with the reference's own constructors and grouping
    spec = instances.config(spec_name)
    devs = [gp.DeviceSpec(id=i, memory_bytes=mem, benchmark_times=(("bench", 1.0 / p_c),))
            for i, _, _, p_c, mem in spec.devices()]
    meas = [gp.LinkMeasurement(endpoints=frozenset((u, v)), alpha_seconds=1e8 / bw,
                               beta_seconds=lat, payload_bytes_m=1e8, latency_seconds=lat,
                               bandwidth_bytes_per_s=bw) for u, v, lat, bw in spec.links()]
    topo = gp.build_topology(devs, meas)
    fgs = gp.group_first_level(topo, 0.3)
    groups = GroupIndex.build(fgs, {f.id: gp.group_second_level(f, topo, 0.3) for f in fgs})
    model = gp.ModelSpec(layers=tuple(gp.LayerSpec(*r) for r in spec.layers),
                         global_batch_candidates=tuple(spec.batches),
                         microbatch_candidates=tuple(spec.micros))
    fg = sorted(groups.fgs)
    n, k = model.num_layers, len(fg)
    total = 6 * math.factorial(k) * math.comb(n - 1, k - 1)
    idx = np.array(random.Random(seed).sample(range(total), n_cand))
    order, counts, bm = decode_indices(n, k, idx, composition_table(n, k))
    cfg = gp.SearchConfig(seed=0)
    nm = len(model.microbatch_candidates)
    cands = [(Candidate(tuple(fg[x] for x in order[i]), tuple(int(c) for c in counts[i])),
              model.global_batch_candidates[bm[i] // nm], model.microbatch_candidates[bm[i] % nm])
             for i in range(n_cand)]
    while time.time() < start:
        time.sleep(0.001)
    t = time.time()
    for c, b, m in cands:
        _evaluate(c, b, m, groups, topo, model, cfg, {})
    t1 = time.time()
    root.handlers[:] = saved
    logging.disable(logging.CRITICAL)
    return t, t1


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
                "in, cost f64 + status u8 out. k2_eval_batch_v4<16, true>: per-warp TMA rings "
                "of input chunks, four consecutive candidates per lane classified branch-free "
                "against infeasible-stage bit rows in shared memory (85 % are +inf without "
                "table reads), feasible ones queued and evaluated 32 at a time with the first- "
                "and last-stage and boundary tables in shared memory (two L2 gathers per "
                "candidate), vector stores. Diagnostic builds: streaming alone 78 us, "
                "classification 104 us per 2e7 (profiles/README.md)"}

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
        "single_snapshot_latency_ms_p99": pct(lat, 99) * 1e3,
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
    for (k, n, seed) in ((6, 80, 6), (8, 80, 8)):
        mk, tk, gk = instances.build(instances.many_group_config(k, n, seed))
        pk = PackedInstance(mk, tk, gk, 1.25)
        ek = Engine(local).load(pk)
        ek.argmin_bnb()
        lat = []
        for _ in range(9):
            t0 = time.perf_counter()
            bb = ek.argmin_bnb()
            lat.append(time.perf_counter() - t0)
        out[f"k4_bnb_k{k}_n{n}"] = {
            "candidates_in_space": int(ek.space_size()), "replan_ms_p50": statistics.median(lat) * 1e3,
            "replan_ms_p99": pct(lat, 99) * 1e3,
            "cost": bb.cost,
            "note": "exact arg-min by branch-and-bound with the exact-in-reals DP bound "
                    "(same winner as exhaustive enumeration; tests/test_bnb.py)"}
        ek.close()

    # ---- drop-in search_plan (beam, host RNG driver + K2 batches) on C4
    from paper_2505_15536_b200 import SearchConfig, search_plan
    import logging
    model, topo, groups = instances.load("c4")
    logging.disable(logging.WARNING)  # the 559 per-plan memory warnings (as the CPU baseline)
    search_plan(model, topo, groups, SearchConfig(seed=0), engine=eng)
    t0 = time.perf_counter()
    r = search_plan(model, topo, groups, SearchConfig(seed=0), engine=eng)
    logging.disable(logging.NOTSET)
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
    model, topo, groups = instances.load("c4", snapshot=0)
    packed = PackedInstance(model, topo, groups, 1.25)
    total = O.space_size(packed)
    # each step: a bounded sample (contiguous prefix) of snapshot 0's re-plan
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
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (App. D C4 recipe; C3 bandwidth snapshot 0)",
        "config": workload_config(args.snapshots, total, world),
        "cpu_baseline": {"value": rate, "unit": "candidates/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"first {per_step} candidates of snapshot 0's C4 exhaustive "
                                   f"range per step (oracle/oracle.c, {threads} threads)"},
        "e2e": {"value": rate, "unit": "candidates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    py = python_reference_rate()
    if py is not None:
        line["python_reference"] = py
    print(json.dumps(line), flush=True)
    return 0


def workload_config(S, total, world):
    return {"workload": "c4-snapshot-replan", "snapshots_per_step": S,
            "candidates_per_snapshot": total, "candidates_per_step": S * total,
            "layers": 80, "devices": 64, "groups": 4, "batch_micro_pairs": 6,
            "l2": "flushed between steps (256 MiB write)",
            "parallelism": f"snapshot shards x{world} (contiguous by index) + NCCL all-gather of "
                           "the 16-byte per-snapshot winners"}


class Ctx:
    """Per-rank handles shared by the sections."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.args = args
        self.rank, self.world, self.local = dist_env()
        self.dev = torch.device("cuda", self.local)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, x):
        t = self.torch.tensor([float(x)], dtype=self.torch.float64, device=self.dev)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def shard(self, n):
        from paper_2505_15536_b200.distributed import shard_items
        return shard_items(n, self.world, self.rank)


def event_loop(X, stream, step, steps, warmup, flush=None, sampler=None):
    """Device ms per step (CUDA events on `stream`), after `warmup` untimed steps."""
    torch = X.torch
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            if flush is not None:
                flush.zero_()
            step()
    X.barrier()
    st = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    en = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    with torch.cuda.stream(stream):
        for i in range(steps):
            if flush is not None:
                flush.zero_()
            st[i].record(stream)
            step()
            en[i].record(stream)
    torch.cuda.synchronize()
    X.barrier()
    return [a.elapsed_time(b) for a, b in zip(st, en)]


def scaling_rows(X, eng, packed, model, topo, groups, total):
    """The other sharded paths at this N (every rank takes part)."""
    torch, dist = X.torch, X.dist
    import random
    from paper_2505_15536_b200 import SearchConfig, instances, replan
    from paper_2505_15536_b200 import distributed as DI
    from paper_2505_15536_b200.engine import Engine
    from paper_2505_15536_b200.enumeration import composition_table, decode_indices
    from paper_2505_15536_b200.layout import PackedInstance
    rows = {}
    stream = torch.cuda.ExternalStream(eng.stream, device=X.dev)
    k = packed.n_fgs
    NC, NP, n_items = DI.space_dims(packed.n_layers, k, len(packed.batches), len(packed.micros))
    nbm = len(packed.batches) * len(packed.micros)

    # (a) ONE C4 exhaustive re-plan, items sharded over the ranks, NCCL tuple arg-min
    eng.load(packed)
    lo, hi = X.shard(n_items)
    dev_ms = event_loop(X, stream, lambda: DI_items(eng, lo, hi), 30, 3)
    cfg = SearchConfig(seed=0)
    lat = []
    for i in range(33):
        X.barrier()
        t0 = time.perf_counter()
        res = DI.exhaustive_plan_sharded(model, topo, groups, cfg, engine=eng)
        el = time.perf_counter() - t0
        if i >= 3:
            lat.append(el)
    lat_max = [X.max_over_ranks(v) for v in lat]
    dmax = [X.max_over_ranks(v) for v in dev_ms]
    rows["single_replan_item_sharded"] = {
        "candidates": total, "items": n_items, "items_this_rank": hi - lo,
        "device_ms_p50": statistics.median(dmax), "device_ms_p99": pct(dmax, 99),
        "api_ms_p50": statistics.median(lat_max) * 1e3, "api_ms_p99": pct(lat_max, 99) * 1e3,
        "candidates_per_s_device": total / (statistics.median(dmax) * 1e-3),
        "best_cost": res.breakdown.plan_cost,
        "note": "device: the rank's item-range sweep (K3), events on the engine stream, max over "
                "ranks; api: distributed.exhaustive_plan_sharded wall clock incl. the 24-byte "
                "NCCL all-gather of (first error, cost bits, tie), winner decode and plan detail"}

    # (b) BASELINE configs[3]: 10^6 sampled C4 candidates in N K2 chunks + arg-min
    idx = np.array(sorted(random.Random(4).sample(range(total), 10**6)), dtype=np.int64)
    order, counts, bm = decode_indices(80, 4, idx, composition_table(80, 4))
    lo, hi = X.shard(idx.size)
    nloc = hi - lo
    d_o = torch.from_numpy(np.ascontiguousarray(order[lo:hi])).to(X.dev)
    d_c = torch.from_numpy(np.ascontiguousarray(counts[lo:hi])).to(X.dev)
    d_b = torch.from_numpy(np.ascontiguousarray(bm[lo:hi])).to(X.dev)
    d_i = torch.from_numpy(idx[lo:hi]).to(X.dev)
    d_cost = torch.empty(max(1, nloc), dtype=torch.float64, device=X.dev)
    d_st = torch.empty(max(1, nloc), dtype=torch.uint8, device=X.dev)
    key = torch.empty(2, dtype=torch.int64, device=X.dev)
    gk = torch.empty(2 * X.world, dtype=torch.int64, device=X.dev)
    torch.cuda.synchronize()

    def k2_step():
        eng.eval_batch_device(4, nloc, d_o.data_ptr(), d_c.data_ptr(), d_b.data_ptr(),
                              d_cost.data_ptr(), d_st.data_ptr())
        eng.argmin_batch_device(nloc, d_cost.data_ptr(), d_st.data_ptr(), d_i.data_ptr(),
                                key.data_ptr())
        if X.world > 1:
            dist.all_gather_into_tensor(gk, key)
    dev_ms = event_loop(X, stream, k2_step, 30, 3)
    dmax = [X.max_over_ranks(v) for v in dev_ms]
    g = (gk if X.world > 1 else key).view(-1, 2).cpu().numpy()
    wi = min(range(g.shape[0]), key=lambda r: (int(g[r, 0]), int(g[r, 1])))
    rows["k2_sample_1e6_sharded"] = {
        "candidates": int(idx.size), "candidates_this_rank": nloc,
        "device_ms_p50": statistics.median(dmax), "device_ms_p99": pct(dmax, 99),
        "candidates_per_s": idx.size / (statistics.median(dmax) * 1e-3),
        "best_index": int(g[wi, 1]), "best_cost": float(np.int64(g[wi, 0]).view(np.float64)),
        "note": "random.Random(4).sample(range(11387376), 10**6) (BASELINE configs[3]); per "
                "rank: K2 on its contiguous chunk, gp_argmin_batch_device (cost, index), NCCL "
                "all-gather"}

    # (c) C3: C2 under 10^4 bandwidth snapshots, partitioned by index
    spec2 = instances.config("c2")
    m2, t2, g2 = instances.build(spec2)
    p2 = PackedInstance(m2, t2, g2, 1.25)
    e2 = Engine(X.local).load(p2)
    tot2 = e2.space_size()
    S2 = 10_000
    bws2 = replan.bandwidth_matrices(p2, [instances.snapshot_multipliers(spec2, j)
                                          for j in range(S2)])
    lo, hi = X.shard(S2)
    width = -(-S2 // X.world)
    d_bw2 = torch.from_numpy(np.ascontiguousarray(bws2[lo:hi])).to(X.dev)
    d_k2 = torch.zeros((width, 2), dtype=torch.int64, device=X.dev)
    d_f2 = torch.zeros(width, dtype=torch.int32, device=X.dev)
    gath2 = torch.empty((X.world * width, 2), dtype=torch.int64, device=X.dev)
    s2 = torch.cuda.ExternalStream(e2.stream, device=X.dev)
    torch.cuda.synchronize()

    def c3_step():
        e2.replan_snapshots_async(d_bw2.data_ptr(), hi - lo, d_k2.data_ptr(), d_f2.data_ptr())
        if X.world > 1:
            dist.all_gather_into_tensor(gath2, d_k2)
    dev_ms = event_loop(X, s2, c3_step, 10, 2)
    dmax = [X.max_over_ranks(v) for v in dev_ms]
    bws2p = torch.from_numpy(bws2).pin_memory().numpy()
    lat = []
    for i in range(6):
        X.barrier()
        t0 = time.perf_counter()
        if X.world > 1:
            res2 = DI.replan_snapshots_sharded(m2, t2, g2, SearchConfig(seed=0), bws2p, engine=e2)
        else:
            res2 = replan.replan_snapshots(m2, t2, g2, SearchConfig(seed=0), bws2p, engine=e2)
        el = time.perf_counter() - t0
        if i >= 1:
            lat.append(el)
    lmax = [X.max_over_ranks(v) for v in lat]
    rows["c3_snapshots_sharded"] = {
        "snapshots": S2, "candidates_per_snapshot": tot2, "snapshots_this_rank": hi - lo,
        "device_ms_p50": statistics.median(dmax), "device_ms_p99": pct(dmax, 99),
        "candidates_per_s": S2 * tot2 / (statistics.median(dmax) * 1e-3),
        "snapshots_per_s": S2 / (statistics.median(dmax) * 1e-3),
        "api_ms_p50": statistics.median(lmax) * 1e3, "api_ms_p99": pct(lmax, 99) * 1e3,
        "ok": int((res2.status == 0).sum()),
        "note": "BASELINE configs[2] (App. D C3 recipe on C2); device: K6 + NCCL all-gather of "
                "the winners; api: distributed.replan_snapshots_sharded with pinned host "
                "matrices (H2D, K6, D2H, all-gather)"}
    e2.close()

    # (e) BASELINE configs[4]: batch-size sweep at this N - the first N
    # enumeration ranks of C4 split into contiguous rank ranges (K3 range
    # kernel per rank), and N = 9 x C4 as 9 bandwidth snapshots split by index
    # (K6); device time per call, max over ranks (L2 warm)
    eng.load(packed)
    c5 = {}
    for N in (10**3, 10**4, 10**5, 10**6, total):
        lo_r, hi_r = X.shard(N)

        def c5_step(lo_r=lo_r, hi_r=hi_r):
            if hi_r > lo_r:
                eng.argmin_range_async(lo_r, hi_r)
        ms = event_loop(X, stream, c5_step, 20, 3)
        if hi_r > lo_r:
            eng.argmin_fetch()
        dmax = X.max_over_ranks(statistics.median(ms))
        c5[str(N)] = {"device_ms_p50": dmax, "candidates_per_s": N / (dmax * 1e-3),
                      "candidates_this_rank": hi_r - lo_r}
    spec4 = instances.config("c4")
    bw9 = replan.bandwidth_matrices(packed, [instances.snapshot_multipliers(spec4, j) for j in range(9)])
    lo9, hi9 = X.shard(9)
    d_bw9 = torch.from_numpy(np.ascontiguousarray(bw9[lo9:hi9])).to(X.dev)
    d_k9 = torch.zeros((max(1, hi9 - lo9), 2), dtype=torch.int64, device=X.dev)
    d_f9 = torch.zeros(max(1, hi9 - lo9), dtype=torch.int32, device=X.dev)
    torch.cuda.synchronize()

    def c5_k6():
        if hi9 > lo9:
            eng.replan_snapshots_async(d_bw9.data_ptr(), hi9 - lo9, d_k9.data_ptr(), d_f9.data_ptr())
    ms = event_loop(X, stream, c5_k6, 10, 2)
    dmax = X.max_over_ranks(statistics.median(ms))
    c5[str(9 * total)] = {"device_ms_p50": dmax, "candidates_per_s": 9 * total / (dmax * 1e-3),
                          "snapshots_this_rank": hi9 - lo9}
    rows["c5_batch_sweep_sharded"] = {
        "rows": c5,
        "note": "BASELINE configs[4]: the first N ranks of C4 in contiguous rank ranges per rank "
                "(K3 range kernel), N = 9 x C4 as 9 snapshots split by index (K6); device time "
                "per call, max over ranks; small N are launch-latency bound"}
    eng.load(packed)

    # (d) weak scaling: every rank re-plans its own C4 snapshot (K3), rank = snapshot
    m3, t3, g3 = instances.load("c4", snapshot=X.rank)
    p3 = PackedInstance(m3, t3, g3, 1.25)
    e3 = Engine(X.local).load(p3)
    s3 = torch.cuda.ExternalStream(e3.stream, device=X.dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=X.dev)
    dev_ms = event_loop(X, s3, lambda: e3.argmin_range_async(0, total), 20, 3, flush)
    e3.argmin_fetch()
    dmax = X.max_over_ranks(sum(dev_ms))
    rows["weak_snapshot_per_rank"] = {
        "candidates_per_s": X.world * total * len(dev_ms) / (dmax * 1e-3),
        "device_ms_per_replan": dmax / len(dev_ms), "scaling": "weak",
        "note": "round-1 headline: rank r re-plans C4 under snapshot r (K3 sweep), L2 flushed"}
    e3.close()
    del flush
    eng.load(packed)
    return rows


def DI_items(eng, lo, hi):
    from paper_2505_15536_b200.engine import lib, _check
    _check(lib().gp_argmin_items_async(eng.handle, int(lo), int(hi)))


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    load_ncu_constants()
    X = Ctx(args)
    torch, dist = X.torch, X.dist
    torch.cuda.set_device(X.local)
    if X.world > 1:
        dist.init_process_group("nccl", device_id=X.dev)
    from paper_2505_15536_b200 import SearchConfig, exhaustive_plan, instances, replan
    from paper_2505_15536_b200 import distributed as DI
    from paper_2505_15536_b200.engine import Engine, best_fields, fp64_peak
    from paper_2505_15536_b200.layout import packed_instance

    spec = instances.config("c4")
    model, topo, groups = instances.build(spec)
    packed = packed_instance(model, topo, groups, 1.25)
    eng = Engine(X.local).load(packed)
    total = eng.space_size()
    S = args.snapshots
    bws = replan.bandwidth_matrices(packed, [instances.snapshot_multipliers(spec, j)
                                             for j in range(S)])
    lo, hi = X.shard(S)
    nloc = hi - lo
    width = -(-S // X.world)
    d_bw = torch.from_numpy(np.ascontiguousarray(bws[lo:hi])).to(X.dev)
    d_keys = torch.zeros((width, 2), dtype=torch.int64, device=X.dev)
    d_flags = torch.zeros(width, dtype=torch.int32, device=X.dev)
    gathered = torch.empty((X.world * width, 2), dtype=torch.int64, device=X.dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=X.dev)
    stream = torch.cuda.ExternalStream(eng.stream, device=X.dev)
    torch.cuda.synchronize()

    # the winners' all-gather: NCCL by default; GP_PEER=1 = peer-memory stores
    # over NVLink (distributed.PeerGather; measured equal to NCCL at N=2 and
    # 4 - 0.483 vs 0.481 ms p50 steps at N=4 - the 16 B per snapshot gather is
    # latency-bound either way)
    peer = None
    if X.world > 1 and os.environ.get("GP_PEER", "0") == "1":
        peer = DI.PeerGather(eng, width * 16)
        if not peer.ok:
            peer.close(X.barrier)
            peer = None

    def step():
        eng.replan_snapshots_async(d_bw.data_ptr(), nloc, d_keys.data_ptr(), d_flags.data_ptr())
        if X.world > 1:
            if peer is not None:
                peer.gather(d_keys.data_ptr())
            else:
                dist.all_gather_into_tensor(gathered, d_keys)

    # ---- device-resident throughput (value) --------------------------------
    with torch.cuda.stream(stream):
        for _ in range(max(3, args.warmup)):
            flush.zero_()
            step()
    X.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    eng.kernel_timing(True)
    with ClockSampler(X.local) as clk:
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.zero_()               # evict L2 (outside the events)
                starts[i].record(stream)
                step()
                ends[i].record(stream)
        torch.cuda.synchronize()
    sweep_ms, sweep_n = eng.kernel_timing(False)
    X.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    dev_ms_max = X.max_over_ranks(sum(step_ms))
    value = S * total * args.steps / (dev_ms_max * 1e-3)
    if peer is not None:
        keys = np.frombuffer(peer.read(), dtype=np.int64).reshape(-1, 2)
    else:
        keys = (gathered if X.world > 1 else d_keys).cpu().numpy().reshape(-1, 2)
    flags_ok = int(d_flags[:nloc].sum().item()) == 0
    # rows of the gathered table in snapshot order
    rows_idx = np.concatenate([np.arange(r * width, r * width + (DI.shard_items(S, X.world, r)[1]
                                                                 - DI.shard_items(S, X.world, r)[0]))
                               for r in range(X.world)])
    win = keys[rows_idx]
    win_cost = win[:, 0].view(np.float64)

    # cross-check 4 snapshots through the other table path (K1 full build + K3)
    checked = 0
    if X.rank == 0:
        for j in (0, 1, S // 2, S - 1):
            eng.set_bandwidth(bws[j])
            b = eng.argmin_range(0, total)
            tie = DI.tie_of_index(b.index, *DI.space_dims(80, 4, 2, 3)[:2], 6)
            assert b.cost == win_cost[j] and tie == int(win[j, 1]), (j, b.cost, win_cost[j])
            checked += 1
        eng.reset_bandwidth()

    # ---- end to end through the public API with host buffers (e2e) ---------
    cfg = SearchConfig(seed=0)
    bws_pinned = torch.from_numpy(bws).pin_memory().numpy()
    lat = []
    for i in range(args.warmup + args.steps):
        X.barrier()
        t0 = time.perf_counter()
        if X.world > 1:
            res = DI.replan_snapshots_sharded(model, topo, groups, cfg, bws_pinned, engine=eng)
        else:
            res = replan.replan_snapshots(model, topo, groups, cfg, bws_pinned, engine=eng)
        el = time.perf_counter() - t0
        if i >= args.warmup:
            lat.append(el)
    e2e_s = X.max_over_ranks(sum(lat))
    e2e_value = S * total * args.steps / e2e_s
    assert (res.status == 0).all() and (res.cost.view(np.int64) == win[:, 0]).all()
    # whole job: the matrices in; out, per snapshot its 16-byte key + 4-byte
    # flags (one GPU) or under torchrun each rank's read of the gathered
    # [world x width x 3] int64 record table
    h2d = S * bws.shape[1] * bws.shape[2] * 8
    d2h = X.world * X.world * width * 3 * 8 if X.world > 1 else S * 20

    rows = None
    if not args.no_rows:
        rows = scaling_rows(X, eng, packed, model, topo, groups, total)

    # ---- single C4 re-plan latency (device K3, C-ABI graph, Python drop-in) -
    replan_lat = None
    if X.world == 1:
        eng.load(packed)
        k3_ms = event_loop(X, stream, lambda: eng.argmin_range_async(0, total), 50, 5, flush)
        eng.argmin_fetch()
        g_lat, p_lat = [], []
        for i in range(105):
            t0 = time.perf_counter()
            eng.replan(packed)
            if i >= 5:
                g_lat.append(time.perf_counter() - t0)
        for i in range(105):
            t0 = time.perf_counter()
            r_ = exhaustive_plan(model, topo, groups, cfg, engine=eng)
            if i >= 5:
                p_lat.append(time.perf_counter() - t0)
        replan_lat = {
            "device_k3_p50": statistics.median(k3_ms), "device_k3_p99": pct(k3_ms, 99),
            "c_abi_gp_replan_p50": statistics.median(g_lat) * 1e3,
            "c_abi_gp_replan_p99": pct(g_lat, 99) * 1e3,
            "dropin_exhaustive_plan_p50": statistics.median(p_lat) * 1e3,
            "dropin_exhaustive_plan_p99": pct(p_lat, 99) * 1e3,
            "note": "one exact C4 re-plan (11,387,376 candidates): device = K3 sweep (L2 "
                    "flushed); gp_replan = host call of the CUDA graph (arena pull + K1 + K3 + "
                    "detail, result in mapped memory); drop-in = exhaustive_plan(model, topology, "
                    "groups, config) of planner.py returning the SearchResult"}

    if X.rank == 0:
        peak = fp64_peak(X.local)
        per_step_ms = dev_ms_max / args.steps
        cand_per_launch = nloc * total
        launch_ms = sweep_ms / max(1, sweep_n)
        alg_ops = sweep_ops_per_candidate(len(packed.batches))
        achieved = alg_ops * cand_per_launch / (launch_ms * 1e-3)
        line = {
            "metric": "candidate plans evaluated/sec", "value": value,
            "unit": "candidates/s", "n_gpus": X.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (App. D C4 recipe; C3 bandwidth snapshots 0..%d)" % (S - 1),
            "config": workload_config(S, total, X.world),
            "e2e": {"value": e2e_value, "unit": "candidates/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_s / args.steps * 1e3,
                    "ms_p50": statistics.median(lat) * 1e3, "ms_p99": pct(lat, 99) * 1e3,
                    "path": ("distributed.replan_snapshots_sharded" if X.world > 1 else
                             "replan.replan_snapshots") +
                            (": pinned host bandwidth matrices -> per rank H2D of its shard, "
                             "gp_replan_snapshots_async (K6 table patch + K3 sweep) into device "
                             "keys, NCCL all-gather of the records from device memory, one D2H"
                             if X.world > 1 else
                             ": pinned host bandwidth matrices -> gp_replan_snapshots (the K6 "
                             "patch kernels read the member-pair and gateway entries of the "
                             "pinned matrices in place over PCIe - zero-copy - then the K3 "
                             "sweep, D2H of the winners)")},
            "roofline": {"bound": "fp64", "achieved": achieved / 1e12, "peak": peak / 1e12,
                         "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": SWEEP_DRAM_BYTES,
                         "traffic_source": NCU_SOURCE if SWEEP_DRAM_BYTES else None,
                         "kernel": "k3_sweep_rec<2,4> (K6 snapshot batch)",
                         "launch_ms": launch_ms, "launches_timed": sweep_n,
                         "candidates_per_launch": cand_per_launch,
                         "share_of_step": launch_ms / per_step_ms,
                         "algorithmic_ops_per_candidate": alg_ops,
                         "algorithm": "prefix-sharing record sweep with a bound-filtered arg-min "
                                      "(DESIGN.md §4): 10.5 FP64 ops per C4 candidate",
                         "reference_order_ops_per_candidate": REF_OPS_PER_CAND_C4,
                         "reference_equivalent_tflops": REF_OPS_PER_CAND_C4 * cand_per_launch
                         / (launch_ms * 1e-3) / 1e12,
                         "issued_fp64_per_candidate": SWEEP_ISSUED_FP64_PER_CAND,
                         "issued_source": NCU_SOURCE if SWEEP_ISSUED_FP64_PER_CAND else None,
                         "peak_source": "FP64 DADD issue rate measured live on this GPU "
                                        "(gp_diag_fp64_peak: 8 independent DADD chains per "
                                        "thread); MEASURED_PEAKS.json has no FP64 entry"},
            "gpu_launches": (3 + (2 if peer is not None else 0)) * X.world * args.steps,
            "gpu_launches_note": "per rank and step: k6_minbw, k6_patch, k3_sweep_rec" +
                                 (", k_peer_put, k_peer_wait (winners all-gathered through "
                                  "peer memory over NVLink)" if peer is not None else
                                  ("" if X.world == 1 else " (+ NCCL all-gather)")),
            "clocks": clk.summary(),
            "step_ms_p50": statistics.median(step_ms), "step_ms_p99": pct(step_ms, 99),
            "winners": {"flags_clear": flags_ok, "cross_checked_k1_k3": checked,
                        "first": [float(win_cost[0]), int(win[0, 1])]},
        }
        if replan_lat is not None:
            line["replan_latency_ms"] = replan_lat
        if rows is not None:
            line["scaling_rows"] = rows
        if not args.no_cpu_baseline and X.world == 1:
            threads = args.cpu_threads or os.cpu_count()
            rate, n, dt = cpu_baseline(packed, total, threads)
            line["cpu_baseline"] = {
                "value": rate, "unit": "candidates/s", "cores": threads, "kind": "port",
                "cpu_model": cpu_model(),
                "sample": f"first {n} candidates of the C4 exhaustive range, "
                          f"{dt:.1f} s on {threads} host threads (oracle/oracle.c)"}
            py = python_reference_rate()
            line["cpu_baseline"]["python_reference"] = py if py is not None else \
                "absent: geopipe not importable on this host (baseline/_ref missing)"
            rp = python_reference_replan()
            if rp is not None:
                line["cpu_baseline"]["python_reference_replan"] = rp
        if not args.no_extra and X.world == 1:
            line["extra"] = extra_sections(eng, packed, total, X.local, args, X.world)
        print(json.dumps(line), flush=True)
    if peer is not None:
        X.barrier()
        peer.close(X.barrier)
    eng.close()
    if X.world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
