"""1F1B makespan (K5) vs the reference's discrete-event engine.

Goldens: tests/golden/sim.json = simulate_timing(t, ONE_F_ONE_B,
SimConfig(iterations=1|2|3)).makespan of 1,500 random timings
(tests/test_schedule.py:random_timing) and of real plan timings
(build_plan_timing of search_plan winners, incl. C1/C2/C4).
"""

import math
import random

import numpy as np
import pytest

import golden_io as G
from paper_2505_15536_b200 import simulate as SM

SIM = G.load("sim.json")


def _timing(d):
    stages = tuple(SM.StageTiming(f, b, w, sy, sy, op, 1.0) for f, b, w, sy, op in d["stages"])
    bounds = tuple(SM.BoundaryTiming(f"{i}-{i + 1}", lat, bw, act, grad)
                   for i, (lat, bw, act, grad) in enumerate(d["boundaries"]))
    return SM.PlanTiming(stages, bounds, d["batch"], d["microbatch"])


TIMINGS = [_timing(d) for d in SIM["timings"]]


def _expected(it):
    ms = SIM["makespan"][str(it)]
    return np.array([m if not isinstance(m, str) else np.nan for m in ms]), \
        np.array([0 if not isinstance(m, str) else 8 for m in ms], np.uint8)


def _random_timings(n, seed):
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        S = rng.randint(1, 6)
        micro = rng.choice([1, 2, 4, 8])
        out.append(SM.make_timing(
            fwd=[rng.uniform(0.2, 2.0) for _ in range(S)],
            bwd=[rng.uniform(0.2, 2.0) for _ in range(S)],
            wgt=[rng.uniform(0.05, 1.0) for _ in range(S)],
            transfer=[rng.uniform(0.05, 2.5) for _ in range(S - 1)],
            microbatch=micro, micro_count=rng.randint(1, 12),
            sync=[rng.uniform(0.0, 0.5) for _ in range(S)],
            opt=[rng.uniform(0.0, 0.3) for _ in range(S)],
            latency=rng.uniform(0.0, 0.2)))
    return out


@pytest.mark.parametrize("it", [1, 2, 3])
def test_oracle_sim_matches_reference(oracle_lib, it):
    arr = SM.pack_timings(TIMINGS)
    ms, st = oracle_lib.sim_batch(arr, len(TIMINGS), it)
    exp, est = _expected(it)
    assert (st == est).all()
    assert (ms.view(np.uint64) == exp.view(np.uint64)).all()


def test_reference_schedule_kats(oracle_lib):
    # tests/test_schedule.py:97-104 (single stage, 1F1B): 2*(1+2+0.5)+0.25+0.75
    t = SM.make_timing(fwd=[1.0], bwd=[2.0], wgt=[0.5], transfer=[], microbatch=1,
                       micro_count=2, sync=[0.25], opt=[0.75])
    ms, st = oracle_lib.sim_batch(SM.pack_timings([t]), 1, 1)
    assert st[0] == 0 and ms[0] == pytest.approx(2 * (1 + 2 + 0.5) + 0.25 + 0.75)
    # tests/test_schedule.py:115-120: three iterations take three times as long
    t = SM.make_timing(fwd=[1.0, 1.0], bwd=[1.0, 1.0], wgt=[0.5, 0.5], transfer=[0.3],
                       microbatch=1, micro_count=3)
    one, _ = oracle_lib.sim_batch(SM.pack_timings([t]), 1, 1)
    three, _ = oracle_lib.sim_batch(SM.pack_timings([t]), 1, 3)
    assert three[0] == pytest.approx(3 * one[0])


def test_pack_rejects_inconsistent_timing():
    from paper_2505_15536_b200 import domain as D
    bad = SM.PlanTiming(TIMINGS[0].stages, TIMINGS[0].boundaries + TIMINGS[0].boundaries[:1]
                        if TIMINGS[0].boundaries else (SM.BoundaryTiming("x", 0, 1, 1, 1),),
                        4, 2)
    with pytest.raises(D.InvalidTimingError):
        SM.pack_timings([bad])


@pytest.mark.gpu
@pytest.mark.parametrize("it", [1, 2, 3])
def test_k5_matches_reference(engine, it):
    ms = SM.simulate_makespans(TIMINGS, it, engine=engine)
    exp, _ = _expected(it)
    assert (ms.view(np.uint64) == exp.view(np.uint64)).all()


@pytest.mark.gpu
def test_k5_matches_oracle_large(engine, oracle_lib):
    tims = _random_timings(20000, 11)
    arr = SM.pack_timings(tims)
    for it in (1, 2):
        ms, st = engine.sim_1f1b(arr, len(tims), it)
        oms, ost = oracle_lib.sim_batch(arr, len(tims), it)
        assert (st == ost).all()
        assert (ms.view(np.uint64) == oms.view(np.uint64)).all()


SIMC = G.load("sim_cands.json")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2j", "c4"])
def test_k5_candidates_match_reference_simulate(engine, oracle_lib, name):
    from cases import load_case
    from paper_2505_15536_b200.layout import PackedInstance
    doc, model, topo, groups = load_case(name)
    packed = PackedInstance(model, topo, groups, 1.25)
    engine.load(packed)
    rows = SIMC[name]
    dec = [oracle_lib.decode(packed, r[0]) for r in rows]
    order = np.stack([d[0] for d in dec]); counts = np.stack([d[1] for d in dec])
    bm = np.array([d[2] for d in dec], np.uint8)
    for col, (it, opt) in enumerate(((1, 0.0), (2, 0.5))):
        ms, st = engine.sim_candidates(order, counts, bm, it, opt)
        for r, m_, s_ in zip(rows, ms, st):
            if r[1 + col] == "infeasible":
                assert s_ == 3
            else:
                assert s_ == 0 and m_ == r[1 + col], (r, m_)


# ---------------------------------------------------------------- policies --
POL = G.load("sim_policies.json")
POL_TIMINGS = [_timing(d) for d in POL["timings"]]


def _pol_expected(key):
    ms = POL["makespan"][key]
    return np.array([m if not isinstance(m, str) else np.nan for m in ms])


@pytest.mark.parametrize("key", sorted(POL["makespan"]))
def test_oracle_policies_and_traces(oracle_lib, key):
    from paper_2505_15536_b200 import abi
    pol, it = key.split(":")
    arr = SM.pack_timings(POL_TIMINGS)
    tr = SM.pack_traces(POL["traces"])
    ms, st = oracle_lib.sim_policy_batch(arr, len(POL_TIMINGS), abi.POLICY_CODE[pol], int(it), tr,
                                         np.arange(len(POL_TIMINGS)))
    exp = _pol_expected(key)
    assert (st == 0).all()
    assert (ms.view(np.uint64) == exp.view(np.uint64)).all()


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(POL["makespan"]))
def test_k5_policies_and_traces(engine, key):
    pol, it = key.split(":")
    ms = SM.simulate_makespans_policy(POL_TIMINGS, pol, int(it), POL["traces"],
                                      np.arange(len(POL_TIMINGS)), engine=engine)
    exp = _pol_expected(key)
    assert (ms.view(np.uint64) == exp.view(np.uint64)).all()


@pytest.mark.gpu
def test_k5_constant_trace_policies_match_oracle(engine, oracle_lib):
    from paper_2505_15536_b200 import abi
    tims = _random_timings(5000, 21)
    arr = SM.pack_timings(tims)
    for pol, code in abi.POLICY_CODE.items():
        ms = SM.simulate_makespans_policy(tims, pol, 2, engine=engine)
        oms, ost = oracle_lib.sim_policy_batch(arr, len(tims), code, 2)
        assert (ms.view(np.uint64) == oms.view(np.uint64)).all(), pol


# ------------------------------------------------- adapter / async reports --
REP = G.load("sim_reports.json")
REP_TIMINGS = [_timing(d) for d in REP["timings"]]


def _rep_key(key):
    ad, asy, pol, it, deg, rec = key.split(":")
    return bool(int(ad)), bool(int(asy)), pol, int(it), float(deg), float(rec)


def _bits(x):
    return np.array(x, dtype=np.float64).view(np.uint64)


def test_report_golden_exercises_the_adapter():
    acts = sum(r[5] for k, rows in REP["reports"].items() if k.startswith("1:")
               for r in rows if not isinstance(r, str))
    stalls = sum(isinstance(r, str) for rows in REP["reports"].values() for r in rows)
    assert acts > 1000 and stalls > 0


@pytest.mark.parametrize("key", sorted(REP["reports"]))
def test_oracle_reports_match_reference(oracle_lib, key):
    from paper_2505_15536_b200 import abi
    ad, asy, pol, it, deg, rec = _rep_key(key)
    arr = SM.pack_timings(REP_TIMINGS)
    tr = SM.pack_traces(REP["traces"])
    reps, ends, st = oracle_lib.sim_reports(arr, len(REP_TIMINGS), abi.POLICY_CODE[pol], it, tr,
                                            np.arange(len(REP_TIMINGS)), adapter=ad,
                                            async_iterations=asy, degrade=deg, recover=rec)
    for i, row in enumerate(REP["reports"][key]):
        if isinstance(row, str):
            assert row == "SchedulingBugError" and st[i] == abi.GP_ERR_SCHEDULING
            continue
        r = reps[i]
        assert st[i] == 0
        assert _bits(r.makespan) == _bits(row[0])
        assert (_bits(ends[i]) == _bits(row[4])).all()
        S = len(row[3])
        bub = [(r.makespan - r.busy[s]) / r.makespan for s in range(S)]
        assert (_bits(bub) == _bits(row[3])).all()
        assert (r.adapter_actions, r.n_transfers, r.n_ops) == tuple(row[5:8])


def _check_summaries(out, rows):
    for o, row in zip(out, rows):
        assert _bits(o.makespan) == _bits(row[0])
        assert _bits(o.throughput) == _bits(row[1])
        assert _bits(o.steady_throughput) == _bits(row[2])
        assert (_bits(o.bubble_fractions) == _bits(row[3])).all()
        assert (_bits(o.iteration_ends) == _bits(row[4])).all()
        assert (o.adapter_action_count, o.transfer_count, o.op_count) == tuple(row[5:8])


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(REP["reports"]))
def test_k5_full_reports_match_reference(engine, key):
    ad, asy, pol, it, deg, rec = _rep_key(key)
    cfg = SM.SimConfig(iterations=it, async_iterations=asy,
                       adapter=SM.AdapterConfig(deg, rec))
    rows = REP["reports"][key]
    ok = [i for i, r in enumerate(rows) if not isinstance(r, str)]
    out = SM.simulate_timings([REP_TIMINGS[i] for i in ok], pol, [REP["traces"][i] for i in ok],
                              np.arange(len(ok)), adapter_enabled=ad, config=cfg, engine=engine)
    _check_summaries(out, [rows[i] for i in ok])
    for i, r in enumerate(rows):
        if isinstance(r, str):
            with pytest.raises(SM.D.SchedulingBugError):
                SM.simulate_timing(REP_TIMINGS[i], pol, REP["traces"][i], ad, cfg, engine=engine)


@pytest.mark.gpu
def test_k5_full_matches_oracle_large(engine, oracle_lib):
    """10^4 random timings x random degrading traces, adapter + async, 3
    iterations: device reports equal the oracle's bit for bit."""
    from paper_2505_15536_b200 import abi
    rng = random.Random(5)
    tims = _random_timings(10000, 33)
    traces = []
    for t in tims:
        bps = {}
        for b in range(len(t.stages) - 1):
            if rng.random() < 0.8:
                pts = sorted(set(round(rng.uniform(0.0, 60.0), 3) for _ in range(rng.randint(1, 6))))
                bps[f"{b}-{b + 1}"] = [[x, rng.choice([0.25, 0.5, 0.6, 1.0, 1.5])] for x in pts]
        traces.append(bps)
    arr = SM.pack_timings(tims)
    tr = SM.pack_traces(traces)
    idx = np.arange(len(tims))
    for pol, code in abi.POLICY_CODE.items():
        for ad, asy in ((True, False), (True, True), (False, True)):
            reps, ends, st = engine.simulate_report(arr, len(tims), code, 3, tr, len(traces), idx,
                                                    adapter=ad, async_iterations=asy)
            oreps, oends, ost = oracle_lib.sim_reports(arr, len(tims), code, 3, tr, idx,
                                                       adapter=ad, async_iterations=asy)
            assert (st == ost).all(), (pol, ad, asy)
            okm = st == 0
            a = np.frombuffer(reps, dtype=np.uint8).reshape(len(tims), -1)
            b = np.frombuffer(oreps, dtype=np.uint8).reshape(len(tims), -1)
            assert (a[okm] == b[okm]).all(), (pol, ad, asy)
            assert (ends.view(np.uint64)[okm] == oends.view(np.uint64)[okm]).all()


@pytest.mark.gpu
def test_k5_full_without_options_equals_fast_path(engine):
    tims = _random_timings(3000, 8)
    for pol in ("gpipe", "1f1b", "zb_original", "zb_compact"):
        fast = SM.simulate_makespans_policy(tims, pol, 2, engine=engine)
        full = SM.simulate_timings(tims, pol, config=SM.SimConfig(iterations=2), engine=engine)
        assert (np.array([o.makespan for o in full]).view(np.uint64) == fast.view(np.uint64)).all()


@pytest.mark.gpu
def test_k5_full_long_traces_match_oracle(engine, oracle_lib):
    """Traces with up to 200 breakpoints per link (the reference has no
    limit; the ABI holds GP_MAX_BREAKPOINTS = 256): device reports equal the
    oracle's bit for bit."""
    from paper_2505_15536_b200 import abi
    assert abi.GP_MAX_BREAKPOINTS >= 200
    rng = random.Random(9)
    tims = _random_timings(2000, 44)
    traces = []
    for t in tims:
        bps = {}
        for b in range(len(t.stages) - 1):
            pts = sorted(set(round(rng.uniform(0.0, 200.0), 4) for _ in range(rng.randint(50, 200))))
            bps[f"{b}-{b + 1}"] = [[x, rng.choice([0.25, 0.5, 0.75, 1.0, 1.25])] for x in pts]
        traces.append(bps)
    arr = SM.pack_timings(tims)
    tr = SM.pack_traces(traces)
    idx = np.arange(len(tims))
    for ad, asy in ((False, False), (True, True)):
        reps, ends, st = engine.simulate_report(arr, len(tims), abi.POLICY_CODE["1f1b"], 3, tr,
                                                len(traces), idx, adapter=ad, async_iterations=asy)
        oreps, oends, ost = oracle_lib.sim_reports(arr, len(tims), abi.POLICY_CODE["1f1b"], 3, tr,
                                                   idx, adapter=ad, async_iterations=asy)
        assert (st == ost).all()
        okm = st == 0
        a = np.frombuffer(reps, dtype=np.uint8).reshape(len(tims), -1)
        b = np.frombuffer(oreps, dtype=np.uint8).reshape(len(tims), -1)
        assert okm.mean() > 0.9
        assert (a[okm] == b[okm]).all()
        assert (ends.view(np.uint64)[okm] == oends.view(np.uint64)[okm]).all()
