"""App. D instance generator (no reference needed) == the reference's own
constructors + group_first_level / group_second_level, field by field."""

import pytest

import refbridge
from paper_2505_15536_b200 import instances as I


@pytest.mark.skipif(not refbridge.AVAILABLE, reason="reference not present")
@pytest.mark.parametrize("name,jit", [("c1", False), ("c1", True), ("c2", False),
                                      ("c2", True), ("c4", False), ("c4", True)])
@pytest.mark.parametrize("snapshot", [None, 3])
def test_mirror_instance_equals_reference(name, jit, snapshot):
    spec = I.config(name, jit)
    mult = I.snapshot_multipliers(spec, snapshot) if snapshot is not None else None
    rm, rt, rg = refbridge.build_reference(spec, mult)
    mm, mt, mg = I.build(spec, mult)
    assert [tuple(vars(l).values()) for l in rm.layers] == \
        [tuple(vars(l).values()) for l in mm.layers]
    assert rm.global_batch_candidates == mm.global_batch_candidates
    assert rm.microbatch_candidates == mm.microbatch_candidates
    assert rt.device_ids == mt.device_ids
    for d in rt.device_ids:
        assert rt.p_c(d) == mt.p_c(d)
        assert rt.device(d).memory_bytes == mt.device(d).memory_bytes
    assert set(rt.links) == set(mt.links)
    for k, v in rt.links.items():
        w = mt.links[k]
        assert (v.metric.p_t, v.latency_seconds, v.bandwidth_bytes_per_s) == \
            (w.metric.p_t, w.latency_seconds, w.bandwidth_bytes_per_s)
    assert sorted(rg.fgs) == sorted(mg.fgs)
    for f in rg.fgs:
        a, b = rg.fgs[f], mg.fgs[f]
        assert (a.member_device_ids, a.intra_metric, a.aggregate_capacity,
                a.min_intra_bandwidth) == (b.member_device_ids, b.intra_metric,
                                           b.aggregate_capacity, b.min_intra_bandwidth)
        assert [(s.id, s.member_device_ids, s.aggregate_capacity) for s in rg.sgs_by_fg[f]] == \
            [(s.id, s.member_device_ids, s.aggregate_capacity) for s in mg.sgs_by_fg[f]]


def test_generator_shapes():
    m, t, g = I.load("c4")
    assert m.num_layers == 80 and len(t.devices) == 64
    assert [len(g.fgs[f].member_device_ids) for f in sorted(g.fgs)] == [16] * 4
    assert [len(g.sgs_by_fg[f]) for f in sorted(g.fgs)] == [2] * 4
