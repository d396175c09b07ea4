"""GPU parity: the CUDA engine (through the C-ABI) vs the reference's answers.

Bar: bit-exact fp64 costs (including +inf for memory-infeasible plans and
the reference's exception for erroring ones), identical chosen plans,
splits, CostBreakdowns, traces and `evaluated` counts.  Reference answers
come from tests/golden/ (scripts/make_golden.py) and, at C4 scale, from the
oracle pinned there.
"""

import random

import numpy as np
import pytest

import golden_io as G
from cases import CASES_ALL, enumerate_encoded, golden_costs, load_case, same_bits
import paper_2505_15536_b200 as P
from paper_2505_15536_b200.layout import PackedInstance

pytestmark = pytest.mark.gpu

ERRORS = {"NoFeasiblePlanError": P.NoFeasiblePlanError,
          "InvalidTopologyError": P.InvalidTopologyError,
          "DegenerateGroupError": P.DegenerateGroupError,
          "InfeasibleSplitError": P.InfeasibleSplitError,
          "InputFileError": P.InputFileError}


def _load(engine, name):
    doc, model, topo, groups = load_case(name)
    packed = PackedInstance(model, topo, groups, 1.25)
    engine.load(packed)
    return doc, model, topo, groups, packed


# ---------------------------------------------------------------- K2 -------
@pytest.mark.parametrize("name", CASES_ALL)
def test_k2_every_candidate_bitwise(engine, name):
    doc, model, topo, groups, packed = _load(engine, name)
    order, counts, bm = enumerate_encoded(packed)
    gc, gs = golden_costs(name)
    if gc.size == 0:
        return
    cost, status = engine.eval_batch(order, counts, bm)
    assert (status == gs).all(), np.nonzero(status != gs)[0][:10]
    ok = same_bits(cost, gc)
    assert ok.all(), (np.nonzero(~ok)[0][:10], cost[~ok][:5], gc[~ok][:5])


@pytest.mark.parametrize("name", ["c4", "c4j"])
def test_k2_c4_sample_bitwise(engine, oracle_lib, name):
    doc, model, topo, groups, packed = _load(engine, name)
    idx = np.load(f"{G.GOLDEN}/{name}.sample_idx.npy")
    gc = np.load(f"{G.GOLDEN}/{name}.sample_costs.npy")
    k = packed.n_fgs
    order = np.zeros((idx.size, k), np.uint8)
    counts = np.zeros((idx.size, k), np.uint8)
    bm = np.zeros(idx.size, np.uint8)
    for r, i in enumerate(idx):
        order[r], counts[r], bm[r] = oracle_lib.decode(packed, int(i))
    cost, status = engine.eval_batch(order, counts, bm)
    assert (status == 0).all()
    assert same_bits(cost, gc).all()


@pytest.mark.parametrize("name", ["c4", "c4j"])
def test_k2_c4_random_1e5_vs_oracle(engine, oracle_lib, name):
    # SURVEY §8(c) protocol item (2): 10^5 random C4 candidates bitwise against
    # the pinned C oracle, through the large-batch path (>= 2^16) and the
    # small-batch path (the first 1,000)
    from paper_2505_15536_b200.enumeration import composition_table, decode_indices
    doc, model, topo, groups, packed = _load(engine, name)
    total = engine.space_size()
    idx = np.random.default_rng(2505).integers(0, total, size=100_000)
    order, counts, bm = decode_indices(80, 4, idx, composition_table(80, 4))
    ec, es = oracle_lib.eval_batch(packed, order, counts, bm, threads=8)
    cost, status = engine.eval_batch(order, counts, bm)
    assert (status == es).all()
    assert same_bits(cost, ec).all()
    c1, s1 = engine.eval_batch(order[:1000], counts[:1000], bm[:1000])
    assert (s1 == es[:1000]).all() and same_bits(c1, ec[:1000]).all()


def _tile(a, reps):
    return np.concatenate([a] * reps)


@pytest.mark.parametrize("name", CASES_ALL)
def test_k2_large_batch_path_bitwise(engine, name):
    # >= 2^16 candidates take the persistent kernel with the stage codes in
    # shared memory (k2_eval_batch_sc); tile every golden case past that and
    # mix in malformed candidates (status 1, cost NaN)
    doc, model, topo, groups, packed = _load(engine, name)
    order, counts, bm = enumerate_encoded(packed)
    gc, gs = golden_costs(name)
    if gc.size == 0:
        return
    reps = (1 << 16) // gc.size + 1
    order, counts, bm = _tile(order, reps), _tile(counts, reps), _tile(bm, reps)
    gc, gs = _tile(gc, reps), _tile(gs, reps).copy()
    bad = np.arange(7, order.shape[0], 9973)
    counts = counts.copy()
    counts[bad, 0] = 0
    gs[bad] = 1
    cost, status = engine.eval_batch(order, counts, bm)
    assert (status == gs).all(), np.nonzero(status != gs)[0][:10]
    good = gs == 0
    assert np.isnan(cost[~good]).all()
    ok = same_bits(cost[good], gc[good])
    assert ok.all(), (np.nonzero(~ok)[0][:10], cost[good][~ok][:5], gc[good][~ok][:5])


@pytest.mark.parametrize("name", ["c4", "c4j"])
def test_k2_c4_large_batch_path_bitwise(engine, oracle_lib, name):
    doc, model, topo, groups, packed = _load(engine, name)
    idx = np.load(f"{G.GOLDEN}/{name}.sample_idx.npy")
    gc = np.load(f"{G.GOLDEN}/{name}.sample_costs.npy")
    k = packed.n_fgs
    order = np.zeros((idx.size, k), np.uint8)
    counts = np.zeros((idx.size, k), np.uint8)
    bm = np.zeros(idx.size, np.uint8)
    for r, i in enumerate(idx):
        order[r], counts[r], bm[r] = oracle_lib.decode(packed, int(i))
    reps = 4
    cost, status = engine.eval_batch(_tile(order, reps), _tile(counts, reps), _tile(bm, reps))
    assert (status == 0).all()
    assert same_bits(cost, _tile(gc, reps)).all()


def test_k2_c4_malformed_large_batch_vs_oracle(engine, oracle_lib):
    # the k = 4 vector-lane kernel's packed-word input checks (byte-SIMD group
    # range / distinctness, zero counts, count sums, (b, m) range) and the
    # slow path (sums < n) against the oracle's or_evaluate, candidate by
    # candidate, on a batch past 2^16
    doc, model, topo, groups, packed = _load(engine, "c4")
    from paper_2505_15536_b200.enumeration import composition_table, decode_indices
    rng = np.random.default_rng(17)
    N = 140_000
    total = engine.space_size()
    order, counts, bm = decode_indices(packed.n_layers, 4, rng.integers(0, total, size=N),
                                       composition_table(packed.n_layers, 4))
    order, counts, bm = order.copy(), counts.copy(), bm.copy()
    kind = rng.integers(0, 12, size=N)
    col = rng.integers(0, 4, size=N)
    rows = np.arange(N)
    m = kind == 1  # duplicate group
    order[m, col[m]] = order[m, (col[m] + 1) % 4]
    for j, g in ((2, 4), (3, 15), (4, 16), (5, 31), (6, 200)):  # group out of range
        m = kind == j
        order[m, col[m]] = g
    m = kind == 7  # zero count
    counts[m, col[m]] = 0
    m = (kind == 8) & (counts[rows, col] > 1)  # sum < n (slow path)
    counts[m, col[m]] -= 1
    m = (kind == 9) & (counts[rows, col] < 250)  # sum > n
    counts[m, col[m]] += 1
    m = kind == 10  # (b, m) index out of range
    bm[m] = rng.integers(len(packed.batches) * len(packed.micros), 256, size=int(m.sum()))
    cost, status = engine.eval_batch(order, counts, bm)
    ocost, ostatus = oracle_lib.eval_batch(packed, order, counts, bm)
    assert (status == ostatus).all(), np.nonzero(status != ostatus)[0][:10]
    good = ostatus == 0
    assert np.isnan(cost[~good]).all()
    ok = same_bits(cost[good], ocost[good])
    assert ok.all(), np.nonzero(~ok)[0][:10]
    assert (~good).sum() > N // 2 and good.sum() > N // 10


def test_k2_image_follows_table_changes(engine, oracle_lib):
    """The k = 4 large-batch kernel bulk-copies a shared-memory image of the
    tables built once per table generation: a bandwidth snapshot
    (gp_set_bandwidth), a gp_replan graph replay and a reload must each give
    a fresh image (results equal to the oracle on the instance then loaded)."""
    from paper_2505_15536_b200 import instances as I
    from paper_2505_15536_b200.enumeration import composition_table, decode_indices
    spec = I.config("c4")
    base = PackedInstance(*I.build(spec), 1.25)
    snaps = [PackedInstance(*I.build(spec, I.snapshot_multipliers(spec, j)), 1.25) for j in (1, 2)]
    engine.load(base)
    total = engine.space_size()
    idx = np.random.default_rng(23).integers(0, total, size=70_000)
    order, counts, bm = decode_indices(base.n_layers, 4, idx, composition_table(base.n_layers, 4))

    def check(packed):
        cost, status = engine.eval_batch(order, counts, bm)
        ocost, ostatus = oracle_lib.eval_batch(packed, order, counts, bm)
        assert (status == ostatus).all()
        assert same_bits(cost, ocost).all()
        return cost

    c0 = check(base)
    engine.set_bandwidth(snaps[0].bw)
    c1 = check(snaps[0])
    assert not same_bits(c0, c1).all()  # the snapshot changes costs
    engine.reset_bandwidth()
    check(base)
    engine.replan(snaps[1])  # graph path: K1 inside the replayed graph
    check(snaps[1])
    engine.load(base)
    check(base)


def test_k2_batch_argmin_device(engine, oracle_lib):
    """gp_argmin_batch_device: least (cost, key) over the status-0 candidates
    of an evaluated batch - against numpy on a K2-evaluated C4 sample (keys =
    enumeration indices, malformed candidates mixed in) and on synthetic
    batches full of cost ties, +inf, errors, no keys, empty and all-invalid."""
    import torch
    from paper_2505_15536_b200.enumeration import composition_table, decode_indices
    doc, model, topo, groups, packed = _load(engine, "c4")
    dev = torch.device("cuda", engine.device)
    out = torch.zeros(2, dtype=torch.int64, device=dev)

    def run(cost, status, keys):
        n = cost.size
        dc = torch.from_numpy(cost).to(dev) if n else torch.zeros(1, dtype=torch.float64, device=dev)
        ds = torch.from_numpy(status).to(dev) if n else torch.zeros(1, dtype=torch.uint8, device=dev)
        dk = torch.from_numpy(keys.view(np.int64)).to(dev) if keys is not None and n else None
        torch.cuda.synchronize()
        engine.argmin_batch_device(n, dc.data_ptr(), ds.data_ptr(), dk.data_ptr() if dk is not None else 0,
                                   out.data_ptr())
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        return o[0], np.uint64(o[1])

    def expect(cost, status, keys):
        k = keys if keys is not None else np.arange(cost.size, dtype=np.uint64)
        ok = np.nonzero(status == 0)[0]
        if ok.size == 0:
            return np.float64(np.inf).view(np.int64), np.uint64(0xFFFFFFFFFFFFFFFF)
        j = ok[np.lexsort((k[ok], cost[ok]))[0]]
        return cost[j].view(np.int64), k[j]

    total = engine.space_size()
    rng = np.random.default_rng(31)
    idx = rng.integers(0, total, size=300_000).astype(np.uint64)
    order, counts, bm = decode_indices(packed.n_layers, 4, idx.astype(np.int64),
                                       composition_table(packed.n_layers, 4))
    counts = counts.copy()
    counts[::97, 0] = 0
    cost, status = engine.eval_batch(order, counts, bm)
    assert run(cost, status, idx) == expect(cost, status, idx)
    assert run(cost, status, None) == expect(cost, status, None)
    for n in (0, 1, 7, 1000, 70_001):
        c = rng.integers(0, 5, size=n).astype(np.float64)
        c[rng.random(n) < 0.2] = np.inf
        st = (rng.random(n) < 0.3).astype(np.uint8)
        keys = rng.permutation(n).astype(np.uint64) * np.uint64(3)
        assert run(c, st, keys) == expect(c, st, keys), n
        assert run(c, st, None) == expect(c, st, None), n
        assert run(c, np.ones(n, np.uint8), keys) == expect(c, np.ones(n, np.uint8), keys), n


def test_k2_rejects_bad_candidates(engine):
    doc, model, topo, groups, packed = _load(engine, "c2")
    order = np.array([[0, 0, 1], [0, 1, 7], [0, 1, 2], [0, 1, 2]], np.uint8)
    counts = np.array([[10, 10, 12], [10, 10, 12], [10, 0, 22], [10, 10, 12]], np.uint8)
    bm = np.array([0, 0, 0, 200], np.uint8)
    cost, status = engine.eval_batch(order, counts, bm)
    assert list(status) == [1, 1, 1, 1]
    assert np.isnan(cost).all()


# ---------------------------------------------------------------- K3 -------
def _key_argmin(packed, gc, gs, lo, hi, order, counts, bm):
    best = None
    for i in range(lo, hi):
        if gs[i]:
            return ("error", int(gs[i]))
        key = (gc[i], tuple(order[i]), tuple(counts[i]), int(bm[i]))
        if best is None or key < best[0]:
            best = (key, i)
    return best


@pytest.mark.parametrize("name", ["c1", "c1j", "c2", "c2j", "rand5", "rand10", "small"])
def test_k3_random_subranges(engine, name):
    doc, model, topo, groups, packed = _load(engine, name)
    gc, gs = golden_costs(name)
    order, counts, bm = enumerate_encoded(packed)
    N = gc.size
    rng = random.Random(7)
    ranges = [(0, N), (0, 1), (N - 1, N)] + \
        [tuple(sorted(rng.sample(range(N + 1), 2))) for _ in range(12)]
    for lo, hi in ranges:
        if hi <= lo:
            continue
        exp = _key_argmin(packed, gc, gs, lo, hi, order, counts, bm)
        got = engine.argmin_range(lo, hi)
        assert got.index == exp[1], (lo, hi)
        assert same_bits(got.cost, gc[exp[1]])
        assert got.evaluated == hi - lo


def test_k3_interleaved_calls_rearm_state(engine):
    # the sweep and the sub-range kernel re-arm their work counters and leave
    # err_idx clean, and the engine skips the resets while it knows the device
    # state: interleave every entry point that touches that state and check
    # each answer
    doc, model, topo, groups, packed = _load(engine, "c2j")
    gc, gs = golden_costs("c2j")
    order, counts, bm = enumerate_encoded(packed)
    N = gc.size
    rng = random.Random(11)
    full = _key_argmin(packed, gc, gs, 0, N, order, counts, bm)[1]
    for rep in range(3):
        assert engine.argmin_range(0, N).index == full
        lo, hi = sorted(rng.sample(range(N + 1), 2))
        if hi > lo:
            assert engine.argmin_range(lo, hi).index == _key_argmin(
                packed, gc, gs, lo, hi, order, counts, bm)[1]
        assert engine.argmin_range(0, N).index == full
        b, _ = engine.replan(packed)
        assert b.index == full
        assert engine.argmin_range(0, N).index == full
        cost, status = engine.eval_batch(order[:100], counts[:100], bm[:100])
        assert same_bits(cost, gc[:100]).all()
        engine.load(packed)
        assert engine.argmin_range(0, N).index == full


@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4, 5])
@pytest.mark.parametrize("name", ["c1j", "c2", "c2j", "rand5", "rand10", "rand6", "small"])
def test_k3_all_kernel_variants_agree(engine, name, mode):
    doc, model, topo, groups, packed = _load(engine, name)
    gc, gs = golden_costs(name)
    order, counts, bm = enumerate_encoded(packed)
    N = gc.size
    rng = random.Random(mode)
    ranges = [(0, N)] + [tuple(sorted(rng.sample(range(N + 1), 2))) for _ in range(6)]
    try:
        engine.set_k3_mode(mode)
        for lo, hi in ranges:
            if hi <= lo:
                continue
            exp = _key_argmin(packed, gc, gs, lo, hi, order, counts, bm)
            got = engine.argmin_range(lo, hi)
            assert got.index == exp[1], (mode, lo, hi)
    finally:
        engine.set_k3_mode(-1)


@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4, 5])
def test_k3_c4_variants(engine, mode):
    doc, model, topo, groups, packed = _load(engine, "c4j")
    try:
        engine.set_k3_mode(mode)
        got = engine.argmin_range(0, engine.space_size())
    finally:
        engine.set_k3_mode(-1)
    assert got.index == doc["oracle_argmin"]["index"]
    assert got.cost == doc["oracle_argmin"]["cost"]


@pytest.mark.parametrize("name", ["c4", "c4j"])
def test_k3_c4_split_subranges_vs_oracle(engine, oracle_lib, name):
    # sub-ranges inside one batch block with whole (micro, order) blocks take
    # the sweep (single batch index) + tile-kernel edges + combine; b = 1
    # exercises the batch offset.  The pinned C oracle is the checker.
    doc, model, topo, groups, packed = _load(engine, name)
    NC = 79079
    bblk = 3 * 24 * NC
    ranges = [(0, 1_000_000), (17, 5 * NC + 3), (bblk + 12_345, bblk + 9 * NC - 1),
              (2 * bblk - 4 * NC - 5, 2 * bblk), (bblk, bblk + 2 * NC)]
    for lo, hi in ranges:
        st, exp = oracle_lib.argmin_range(packed, lo, hi, threads=8)
        assert st == 0
        got = engine.argmin_range(lo, hi)
        assert got.index == exp.index, (lo, hi)
        assert same_bits(got.cost, exp.cost)
        assert got.evaluated == hi - lo


@pytest.mark.parametrize("name", CASES_ALL)
def test_exhaustive_plan_matches_reference(engine, name):
    doc, model, topo, groups = load_case(name)
    ex = doc["exhaustive"]
    cfg = P.SearchConfig(seed=0, beam_width=doc["search_config"]["beam_width"],
                         max_iter=doc["search_config"]["max_iter"])
    if "error" in ex:
        with pytest.raises(ERRORS[ex["error"]]):
            P.exhaustive_plan(model, topo, groups, cfg, engine=engine)
        return
    res = P.exhaustive_plan(model, topo, groups, cfg, engine=engine)
    assert G.normalize_result(res) == ex["result"]


@pytest.mark.parametrize("name", ["c4", "c4j"])
def test_k3_c4_full_argmin(engine, name):
    doc, model, topo, groups, packed = _load(engine, name)
    total = engine.space_size()
    assert total == 11_387_376
    got = engine.argmin_range(0, total)
    exp = doc["oracle_argmin"]
    assert got.index == exp["index"]
    assert got.cost == exp["cost"]
    assert list(got.order[:got.k]) == exp["order"]
    assert list(got.counts[:got.k]) == exp["counts"]


# ---------------------------------------------------------- search_plan ----
SEARCH_CASES = [(n, s) for n in CASES_ALL + ["c4", "c4j"]
                for s in G.load(f"{n}.json")["search"]]


@pytest.mark.parametrize("name,seed", SEARCH_CASES)
def test_search_plan_matches_reference(engine, name, seed):
    doc, model, topo, groups = load_case(name)
    exp = doc["search"][seed]
    cfg = P.SearchConfig(seed=int(seed), beam_width=doc["search_config"]["beam_width"],
                         max_iter=doc["search_config"]["max_iter"])
    if "error" in exp:
        with pytest.raises(ERRORS[exp["error"]]):
            P.search_plan(model, topo, groups, cfg, engine=engine)
        return
    res = P.search_plan(model, topo, groups, cfg, engine=engine)
    assert G.normalize_result(res) == exp["result"]


def test_space_overflow_is_an_error(engine):
    """16 groups x 255 layers: the space exceeds 2^64 -> InputFileError, not wraparound."""
    from paper_2505_15536_b200 import instances as I
    import paper_2505_15536_b200 as P
    regions = [[[(1e14 * (1 + r), 80e9)]] for r in range(16)]
    layers = I.transformer_layers(255, 1024, 4096, 512, 32000, d_kv=1024)
    spec = I.InstanceSpec("huge", layers, (64,), (8,), regions, intra_bw=[1e9] * 16,
                          intra_lat=[1e-4] * 16, cross_bw=1e8, cross_lat=0.01)
    model, topo, groups = I.build(spec)
    engine.load(PackedInstance(model, topo, groups, 1.25))
    with pytest.raises(P.InputFileError):
        engine.space_size()


# search_plan for seeds 0-20 on C1-C4 (SURVEY §8(c) parity protocol (3))
SEEDS = G.load("search_seeds.json")


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(SEEDS))
def test_search_plan_seeds_0_to_20(engine, name):
    from paper_2505_15536_b200 import instances as I
    model, topo, groups = I.load(name[:2], name.endswith("j"))
    for seed, exp in SEEDS[name].items():
        res = P.search_plan(model, topo, groups, P.SearchConfig(seed=int(seed)), engine=engine)
        assert G.normalize_result(res) == exp["result"], (name, seed)


def test_replan_graph_after_loads_of_other_shapes(engine):
    """gp_replan replays its captured graph only while the context holds an
    instance of the graph's shape: replan(A), then loads / searches / K4 on
    smaller instances B, then replan(A') must still give A's golden answer
    (stale run groups, prefixes and host geometry otherwise)."""
    from paper_2505_15536_b200 import instances as I
    docA, mA, tA, gA = load_case("c2j")
    pA = PackedInstance(mA, tA, gA, 1.25)
    expA = docA["exhaustive"]["result"]["breakdown"]["plan_cost"]
    gc, gs = golden_costs("c2j")
    for other in ["rand10", "small", "k5n9", "c1", "rand12"]:
        b, _ = engine.replan(pA)
        assert b.cost == expA
        docB, mB, tB, gB = load_case(other)
        pB = PackedInstance(mB, tB, gB, 1.25)
        engine.load(pB)
        if pB.n_fgs >= 2:
            engine.argmin_bnb()
        P.search_plan(mB, tB, gB, P.SearchConfig(seed=1), engine=engine)
        pA2 = PackedInstance(mA, tA, gA, 1.25)  # a different object of A's shape
        b, info = engine.replan(pA2)
        assert b.cost == expA, other
        assert info.plan_cost == expA
        total = engine.space_size()
        assert total == gc.size
        assert engine.argmin_range(0, total).cost == expA
    # and K6 snapshots in between
    spec = I.config("c2")
    m2, t2, g2 = I.build(spec)
    p2 = PackedInstance(m2, t2, g2, 1.25)
    engine.load(p2)
    from paper_2505_15536_b200 import replan as R
    engine.replan_snapshots(R.bandwidth_matrices(p2, [I.snapshot_multipliers(spec, 3)]))
    b, _ = engine.replan(pA)
    assert b.cost == expA


def test_reset_bandwidth_restores_groupindex_min_bw(engine):
    """After snapshots, the loaded GroupIndex min_intra_bandwidth values come
    back (not min(bw) re-derived from the matrix): use a hierarchy whose
    stored min bandwidth differs from the matrix minimum."""
    import dataclasses
    doc, model, topo, groups = load_case("c2j")
    fg = sorted(groups.fgs)[0]
    g0 = groups.fgs[fg]
    fgs = dict(groups.fgs)
    fgs[fg] = dataclasses.replace(g0, min_intra_bandwidth=g0.min_intra_bandwidth * 0.5)
    groups2 = dataclasses.replace(groups, fgs=fgs)
    packed = PackedInstance(model, topo, groups2, 1.25)
    engine.load(packed)
    total = engine.space_size()

    def costs():
        engine.verify_begin(0, total)
        engine.argmin_range(0, total)
        return engine.verify_end()

    before = costs()
    engine.set_bandwidth(packed.bw)  # snapshot = same matrix: min bw re-derived from it
    derived = costs()
    assert not same_bits(derived, before).all()  # the stored value really differs
    engine.reset_bandwidth()
    assert same_bits(costs(), before).all()


WARN = G.load("search_warnings.json")


@pytest.mark.parametrize("name", sorted(WARN))
def test_search_plan_warnings_and_errors_in_reference_order(engine, name):
    """search_plan logs one warning per memory-infeasible plan when it is first
    evaluated (src/planner.py:321) and one per infeasible (b, m) pass (:367),
    in the reference's sequential pass order, and raises the first error in
    that order - although the passes run in lock-step on the GPU."""
    import logging
    doc, model, topo, groups = load_case(name)
    logger = logging.getLogger("paper_2505_15536_b200.planner")
    for seed, exp in WARN[name].items():
        msgs = []

        class Cap(logging.Handler):
            def emit(self, rec):
                msgs.append(rec.getMessage())
        h = Cap()
        logger.addHandler(h)
        old = logger.propagate
        logger.propagate = False
        try:
            P.search_plan(model, topo, groups, P.SearchConfig(seed=int(seed)), engine=engine)
            err = None
        except P.GeopipeError as e:
            err = type(e).__name__
        finally:
            logger.removeHandler(h)
            logger.propagate = old
        assert err == exp["error"], (name, seed)
        assert msgs == exp["warnings"], (name, seed)
