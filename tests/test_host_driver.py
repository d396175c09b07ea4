"""Host-side beam driver pieces (RNG + integer logic, no cost arithmetic)
match the reference draw for draw."""

import random

import pytest

import refbridge
from paper_2505_15536_b200 import domain as D
from paper_2505_15536_b200 import planner as P
from paper_2505_15536_b200 import instances as I


def test_expansion_kats():
    # reference tests/test_planner.py:95-137
    rng = random.Random(0)
    cand = D.Candidate(order=("a", "b"), counts=(2, 2))
    got = P.expand_candidates([cand], rng)
    assert cand in got and len(got) == 4
    got = P.expand_candidates([D.Candidate(("a", "b"), (1, 3))], random.Random(0))
    assert all(min(c.counts) >= 1 for c in got)
    single = D.Candidate(order=("a",), counts=(4,))
    assert P.expand_candidates([single], random.Random(0)) == [single]


def test_initial_candidates_capacity_proportional():
    m, t, g = I.load("c2")
    fgs = sorted(g.fgs.values(), key=lambda f: f.id)
    a = P.initial_candidates(m, fgs, 4, seed=7)
    b = P.initial_candidates(m, fgs, 4, seed=7)
    assert a == b and len(a) == 4
    assert all(sum(c.counts) == m.num_layers for c in a)


@pytest.mark.skipif(not refbridge.AVAILABLE, reason="reference not present")
@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_driver_matches_reference(name):
    gp = refbridge.geopipe()
    from geopipe import planner as RP
    spec = I.config(name, True)
    rm, rt, rg = refbridge.build_reference(spec)
    fgs = sorted(rg.fgs.values(), key=lambda f: f.id)
    for seed in range(20):
        ours = P.initial_candidates(rm, fgs, 8, seed)
        ref = RP.initial_candidates(rm, fgs, 8, seed)
        assert [(c.order, c.counts) for c in ours] == [(c.order, c.counts) for c in ref]
        r1, r2 = random.Random(seed), random.Random(seed)
        beam_o, beam_r = ours, ref
        for _ in range(5):
            eo = P.expand_candidates(beam_o, r1)
            er = RP.expand_candidates(beam_r, r2)
            assert [(c.order, c.counts) for c in eo] == [(c.order, c.counts) for c in er]
            beam_o, beam_r = eo[:8], er[:8]
    for total, w in [(7, [1.0, 2.0, 4.0]), (80, [3.3, 1.1, 7.7, 0.5]), (5, [2.0, 3.0])]:
        assert P.proportional_split(total, w, 1) == RP.proportional_split(total, w, 1)


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_tuple_expansion_matches_candidate_expansion(name):
    """The beam driver's tuple form (_expand_keys) yields the variants of
    expand_candidates in the same order and leaves the RNG in the same state."""
    m, t, g = I.load(name, jitter=True)
    fgs = sorted(g.fgs.values(), key=lambda f: f.id)
    for seed in range(10):
        beam = P.initial_candidates(m, fgs, 8, seed)
        keys = [(c.order, c.counts) for c in beam]
        r1, r2 = random.Random(seed), random.Random(seed)
        for _ in range(6):
            ec = P.expand_candidates(beam, r1)
            ek = P._expand_keys(keys, r2)
            assert [(c.order, c.counts) for c in ec] == ek
            assert r1.getstate() == r2.getstate()
            beam, keys = ec[3:11], ek[3:11]
