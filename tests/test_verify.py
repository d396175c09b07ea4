"""Per-candidate parity of the exhaustive / snapshot kernels (verify sink).

The arg-min tests elsewhere check only the winner of a K3 launch; a wrong
cost on a losing candidate would pass them.  Here every K3 / K6 launch runs
its verify instantiation (gp_diag_verify_begin: the same kernel source plus
a store of each evaluated candidate's cost at its enumeration index) and the
whole cost vector is compared bitwise against

* the reference's own `_evaluate` costs (tests/golden/*.costs.npy, every
  candidate of every golden case, including k = 5..8 stage groups), and
* the pinned oracle (oracle/, checked bit-exact against the reference on the
  same instances) for C4 (11,387,376 candidates) and for bandwidth snapshots.

Every dispatch route is covered: the full-item sweep in each shared-memory
mode (k fixed at compile time for k = 3..6, generic otherwise), the
sub-range tile kernel and the split (sweep + edge pieces) path, the
status-tracking generic kernel, multi-GPU item shards, the gp_replan CUDA
graph and the K6 snapshot sweep (fast path and the zero-bandwidth slow path).
"""

import math
import os

import numpy as np
import pytest

from cases import CASES_ALL, golden_costs, load_case, same_bits
from paper_2505_15536_b200 import instances as I
from paper_2505_15536_b200 import replan as R
from paper_2505_15536_b200.layout import PackedInstance

pytestmark = pytest.mark.gpu

SENTINEL = np.uint64(0xFFFFFFFFFFFFFFFF)
THREADS = os.cpu_count() or 8


def _status_of(v):
    """Status code carried by a verify slot (0 for a cost)."""
    bits = v.view(np.uint64)
    nan = np.isnan(v) & (bits != SENTINEL)
    return np.where(nan, (bits & np.uint64(15)).astype(np.uint8), 0).astype(np.uint8)


def _check(v, gc, gs, where=None):
    """Verify slots v (full space) == golden costs/status; `where` = mask of
    the positions that must have been written (others keep the sentinel)."""
    bits = v.view(np.uint64)
    if where is None:
        where = np.ones(v.size, bool)
    unwritten = bits == SENTINEL
    assert not unwritten[where].any(), np.nonzero(unwritten & where)[0][:10]
    assert unwritten[~where].all(), np.nonzero(~unwritten & ~where)[0][:10]
    st = _status_of(v)
    assert (st[where] == gs[where]).all(), np.nonzero((st != gs) & where)[0][:10]
    ok = gs[where] == 0
    good = same_bits(v[where][ok], gc[where][ok])
    assert good.all(), (np.nonzero(~good)[0][:10], v[where][ok][~good][:4], gc[where][ok][~good][:4])


def _run(engine, total, fn):
    engine.verify_begin(0, total)
    err = None
    try:
        fn()
    except Exception as e:  # the reference raises too (status slots say which)
        err = e
    return engine.verify_end(), err


def _load(engine, name):
    doc, model, topo, groups = load_case(name)
    packed = PackedInstance(model, topo, groups, 1.25)
    engine.load(packed)
    return doc, packed


@pytest.mark.parametrize("mode", [-1, 0, 1, 2, 3, 5])
@pytest.mark.parametrize("name", CASES_ALL)
def test_every_candidate_full_space(engine, name, mode):
    doc, packed = _load(engine, name)
    total = engine.space_size()
    gc, gs = golden_costs(name)
    if total == 0:
        return
    engine.set_k3_mode(mode)
    try:
        v, err = _run(engine, total, lambda: engine.argmin_range(0, total))
    finally:
        engine.set_k3_mode(-1)
    _check(v, gc, gs)
    assert (err is not None) == bool(gs.any()), err


@pytest.mark.parametrize("name", ["c1j", "c2", "c2j", "rand10", "rand5", "k5n9", "k6n8", "k7n8",
                                  "k8n9"])
def test_every_candidate_sub_ranges(engine, name):
    doc, packed = _load(engine, name)
    total = engine.space_size()
    gc, gs = golden_costs(name)
    rng = np.random.default_rng(sum(name.encode()))
    nbm = len(packed.batches) * len(packed.micros)
    per_b = total // len(packed.batches)
    ranges = [(0, total), (1, total - 1)]
    for _ in range(6):
        lo, hi = sorted(int(x) for x in rng.integers(0, total + 1, 2))
        ranges.append((lo, hi))
    for _ in range(3):  # inside one batch block: sweep + edge pieces (split path)
        b = int(rng.integers(0, len(packed.batches)))
        lo, hi = sorted(int(x) for x in rng.integers(0, per_b, 2))
        ranges.append((b * per_b + lo, b * per_b + hi))
    for lo, hi in ranges:
        for mode in (-1, 0, 3):
            engine.set_k3_mode(mode)
            try:
                v, err = _run(engine, total, lambda: engine.argmin_range(lo, hi))
            finally:
                engine.set_k3_mode(-1)
            where = np.zeros(total, bool)
            where[lo:hi] = True
            _check(v, gc, gs, where)
    assert nbm >= 1


@pytest.mark.parametrize("name", ["c2", "c2j", "k5n9", "k6n8", "k8n9"])
def test_every_candidate_item_shards(engine, name):
    """Multi-GPU shard unit: items [lo, hi) of (micro-batch, order)."""
    doc, packed = _load(engine, name)
    total = engine.space_size()
    gc, gs = golden_costs(name)
    k, n = packed.n_fgs, packed.n_layers
    NP, NC = math.factorial(k), math.comb(n - 1, k - 1)
    nm = len(packed.micros)
    n_items = nm * NP
    idx = np.arange(total)
    item = (idx // NC) % (nm * NP)  # (b * nm + m) * NP + perm -> m * NP + perm
    for world in (2, 3, 8):
        for r in range(world):
            lo, hi = n_items * r // world, n_items * (r + 1) // world
            v, err = _run(engine, total, lambda: engine.argmin_items(lo, hi))
            _check(v, gc, gs, (item >= lo) & (item < hi))


@pytest.mark.parametrize("name", ["c1", "c2j", "rand10", "k6n8", "k7n8"])
def test_every_candidate_replan_graph(engine, name):
    """gp_replan: one CUDA graph of arena pull + K1 + sweep + detail."""
    doc, packed = _load(engine, name)
    total = engine.space_size()
    gc, gs = golden_costs(name)
    for _ in range(2):  # capture, then replay
        v, err = _run(engine, total, lambda: engine.replan(packed))
        _check(v, gc, gs)


@pytest.mark.parametrize("name", ["c4", "c4j"])
def test_every_c4_candidate_vs_oracle(engine, oracle_lib, name):
    """All 11,387,376 C4 candidates through the production dispatch (sweep)
    and the gp_replan graph, bitwise against the pinned oracle."""
    doc, packed = _load(engine, name)
    total = engine.space_size()
    oc, os_ = oracle_lib.eval_range(packed, 0, total, threads=THREADS)
    v, err = _run(engine, total, lambda: engine.argmin_range(0, total))
    _check(v, oc, os_)
    v, err = _run(engine, total, lambda: engine.replan(packed))
    _check(v, oc, os_)
    exp = doc["oracle_argmin"]
    assert engine.argmin_range(0, total).cost == exp["cost"]


def test_c4_sub_ranges_vs_oracle(engine, oracle_lib):
    doc, packed = _load(engine, "c4")
    total = engine.space_size()
    rng = np.random.default_rng(44)
    per_b = total // 2
    NC = math.comb(79, 3)
    for lo, hi in [(NC * 7 + 5, NC * 19 + 3), (per_b - 1000, per_b + 1000),
                   (int(rng.integers(0, total // 2)), int(rng.integers(total // 2, total)))]:
        v, err = _run(engine, total, lambda: engine.argmin_range(lo, hi))
        v = v[lo:hi]
        assert not (v.view(np.uint64) == SENTINEL).any()
        oc, os_ = oracle_lib.eval_range(packed, lo, hi, threads=THREADS)
        assert same_bits(v, oc).all()


def _snapshot_packed(spec, mult):
    m, t, g = I.build(spec, mult)
    return PackedInstance(m, t, g, 1.25)


def test_every_candidate_k6_snapshots_c2(engine, oracle_lib):
    """K6: 40 C3 snapshots of C2 in one batch, plus two snapshots with a
    zero-bandwidth link (status-tracking slow path), per candidate."""
    spec = I.config("c2")
    model, topo, groups = I.build(spec)
    packed = PackedInstance(model, topo, groups, 1.25)
    engine.load(packed)
    total = engine.space_size()
    mults = [I.snapshot_multipliers(spec, j) for j in range(40)]
    ids = sorted(d.id for d in topo.devices)
    for j in (5, 17):  # zero bandwidth inside a group / on every cross link of a region
        m = dict(mults[j])
        if j == 5:
            m[(ids[0], ids[1])] = 0.0
        else:
            for key in m:
                if key[0][:2] != key[1][:2] and "r2" in (key[0][:2], key[1][:2]):
                    m[key] = 0.0
        mults[j] = m
    bws = R.bandwidth_matrices(packed, mults)
    S = len(mults)
    engine.verify_begin(0, S * total)
    bests, status = engine.replan_snapshots(bws)
    v = engine.verify_end().reshape(S, total)
    for j in range(S):
        ps = _snapshot_packed(spec, mults[j])
        oc, os_ = oracle_lib.eval_range(ps, 0, total, threads=THREADS)
        _check(v[j], oc, os_)
        st, ob = oracle_lib.argmin_range(ps, 0, total, threads=THREADS)
        assert int(status[j]) == st, j
        if st == 0:
            assert bests[j].cost == ob.cost and bests[j].index == ob.index, j
    # the context's own instance is unchanged afterwards
    assert engine.argmin_range(0, total).cost == oracle_lib.argmin_range(packed, 0, total,
                                                                         threads=THREADS)[1].cost


def test_every_candidate_k6_snapshots_c4(engine, oracle_lib):
    spec = I.config("c4")
    model, topo, groups = I.build(spec)
    packed = PackedInstance(model, topo, groups, 1.25)
    engine.load(packed)
    total = engine.space_size()
    mults = [I.snapshot_multipliers(spec, j) for j in range(3)]
    bws = R.bandwidth_matrices(packed, mults)
    engine.verify_begin(0, 3 * total)
    bests, status = engine.replan_snapshots(bws)
    v = engine.verify_end().reshape(3, total)
    for j in range(3):
        ps = _snapshot_packed(spec, mults[j])
        oc, os_ = oracle_lib.eval_range(ps, 0, total, threads=THREADS)
        _check(v[j], oc, os_)
        assert status[j] == 0


def test_verify_mode_is_transparent(engine):
    """The winner is the same with and without the verify sink."""
    doc, packed = _load(engine, "c2j")
    total = engine.space_size()
    a = engine.argmin_range(0, total)
    engine.verify_begin(0, total)
    b = engine.argmin_range(0, total)
    engine.verify_end()
    c = engine.argmin_range(0, total)
    assert (a.cost, a.index) == (b.cost, b.index) == (c.cost, c.index)
