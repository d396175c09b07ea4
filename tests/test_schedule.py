"""Schedules (K5 op / transfer records) and their validation (K8) vs the
reference's simulate_timing(...).schedule / .transfers, validate_schedule
and bubble_fraction (src/schedule.py:77-182).

Golden: tests/golden/schedules.json (scripts/make_golden.py dump_schedules):
per timing of sim_reports.json and per (adapter, async, policy) at 3
iterations, a digest of the reference's ops + transfers, and the count /
digest of validate_schedule's messages on a seeded perturbation
(tests/schedule_cases.py).
"""

import numpy as np
import pytest

import golden_io as G
import schedule_cases as SC
from paper_2505_15536_b200 import abi
from paper_2505_15536_b200 import schedule as SCH
from paper_2505_15536_b200 import simulate as SM
from test_sim import REP, REP_TIMINGS

GOLD = G.load("schedules.json")
KEYS = sorted(GOLD["digests"])


def _opts(key):
    ad, asy, pol, it = key.split(":")
    return bool(int(ad)), bool(int(asy)), pol, int(it)


def _perturbed(sched, seed):
    pert = SC.perturb(sched.ops, seed)
    ops = tuple(tuple(SCH.PipeOp(SCH.OpKind(k), s, a, b, z, it, mb) for k, s, a, b, z, it, mb in st)
                for st in pert)
    return SCH.Schedule(ops, sched.makespan, sched.policy, sched.num_stages, sched.micro_count)


def test_golden_has_violations_and_stalls():
    v = [r for rows in GOLD["violations"].values() for r in rows if r]
    assert sum(1 for r in v if r[0] > 0) > 500 and sum(1 for r in v if r[0] == 0) > 100
    assert any(r is None for rows in GOLD["digests"].values() for r in rows)


@pytest.mark.parametrize("key", KEYS)
def test_oracle_schedules_and_validation(oracle_lib, key):
    ad, asy, pol, it = _opts(key)
    arr = SM.pack_timings(REP_TIMINGS)
    tr = SM.pack_traces(REP["traces"])
    reps, ooff, ops, xoff, xfs, st, aoff, acts = oracle_lib.sim_schedules(
        arr, len(REP_TIMINGS), abi.POLICY_CODE[pol], it, tr, np.arange(len(REP_TIMINGS)),
        adapter=ad, async_iterations=asy)
    for i, t in enumerate(REP_TIMINGS):
        exp = GOLD["digests"][key][i]
        if exp is None:
            assert st[i] == abi.GP_ERR_SCHEDULING
            continue
        sched, xf = SCH.records_to_schedule(t, ops, int(ooff[i]), int(ooff[i + 1]), xfs,
                                            int(xoff[i]), int(xoff[i + 1]), reps[i].makespan, pol)
        assert SC.digest(sched.ops, xf) == exp, i
        a = [SCH.AdapterAction(x.t, x.stage, x.old_size, x.new_size, abi.ACTION_SIGNALS[x.signal])
             for x in (acts[j] for j in range(int(aoff[i]), int(aoff[i + 1])))]
        assert SC.action_digest(a) == GOLD["actions"][key][i], i
        p = _perturbed(sched, 1000 * i + 7)
        off, parr, _ = SCH.pack_schedules([p])
        recs, nv, _ = oracle_lib.validate_schedule(arr[i], parr, int(off[1]), p.makespan)
        msgs = [SCH.format_violation(v) for v in recs]
        cnt, dig, head = GOLD["violations"][key][i]
        assert (nv, SC.text_digest(msgs)) == (cnt, dig), (i, msgs[:3], head)


@pytest.mark.gpu
@pytest.mark.parametrize("key", KEYS)
def test_k5_schedules_and_k8_validation(engine, key):
    ad, asy, pol, it = _opts(key)
    rows = GOLD["digests"][key]
    ok = [i for i, r in enumerate(rows) if r is not None]
    cfg = SM.SimConfig(iterations=it, async_iterations=asy)
    out = SCH.generate_schedules([REP_TIMINGS[i] for i in ok], pol,
                                 [REP["traces"][i] for i in ok], np.arange(len(ok)),
                                 adapter_enabled=ad, config=cfg, engine=engine, with_actions=True)
    for i, (sched, xf, acts) in zip(ok, out):
        assert SC.digest(sched.ops, xf) == rows[i], i
        assert SC.action_digest(acts) == GOLD["actions"][key][i], i
    out = [(s_, x_) for s_, x_, _ in out]
    pert = [_perturbed(sched, 1000 * i + 7) for i, (sched, _) in zip(ok, out)]
    msgs = SCH.validate_schedules(pert, [REP_TIMINGS[i] for i in ok], engine=engine,
                                  max_violations=8)
    for i, m in zip(ok, msgs):
        cnt, dig, head = GOLD["violations"][key][i]
        assert (len(m), SC.text_digest(m)) == (cnt, dig), (i, m[:3], head)
    # bubble_fraction from the device busy sums equals the report's
    bub = SCH.bubble_fractions([s for s, _ in out], [REP_TIMINGS[i] for i in ok], engine=engine)
    summ = SM.simulate_timings([REP_TIMINGS[i] for i in ok], pol, [REP["traces"][i] for i in ok],
                               np.arange(len(ok)), adapter_enabled=ad, config=cfg, engine=engine)
    for b, s in zip(bub, summ):
        assert tuple(b) == s.bubble_fractions


@pytest.mark.gpu
def test_k8_rejects_non_dense_ids(engine):
    (sched, _), = SCH.generate_schedules([REP_TIMINGS[0]], "1f1b",
                                         config=SM.SimConfig(iterations=1), engine=engine)
    ops = list(sched.ops)
    st0 = list(ops[0])
    f = [j for j, o in enumerate(st0) if o.kind is SCH.OpKind.FORWARD]
    st0[f[0]], st0[f[1]] = st0[f[1]], st0[f[0]]
    ops[0] = tuple(st0)
    bad = SCH.Schedule(tuple(ops), sched.makespan, sched.policy, sched.num_stages,
                       sched.micro_count)
    with pytest.raises(SM.D.InputFileError):
        SCH.validate_schedules([bad], [REP_TIMINGS[0]], engine=engine)
