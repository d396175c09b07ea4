"""Shared helpers for the schedule tests: a canonical digest of a schedule
(ops + transfers) and a seeded perturbation recipe for validate_schedule.
Works on the reference's objects and on the mirrors alike."""

from __future__ import annotations

import hashlib
import random


def _kind(k):
    return getattr(k, "value", k)


def canonical(schedule_ops, transfers):
    ops = [[(s, _kind(o.kind), o.start, o.end, o.size, o.iteration, o.microbatch_id)
            for o in stage] for s, stage in enumerate(schedule_ops)]
    xf = [(x.link_id, x.direction, x.boundary, x.start, x.end, x.size, x.iteration,
           x.microbatch_id) for x in transfers]
    return repr((ops, xf))


def digest(schedule_ops, transfers):
    return hashlib.sha1(canonical(schedule_ops, transfers).encode()).hexdigest()[:20]


def action_digest(actions):
    return hashlib.sha1(repr([(a.t, a.stage, a.old_size, a.new_size, a.signal)
                              for a in actions]).encode()).hexdigest()[:20]


def text_digest(messages):
    return hashlib.sha1("\n".join(messages).encode()).hexdigest()[:20]


def perturb(schedule_ops, seed):
    """Per-stage lists of (kind, stage, start, end, size, iteration, mb)
    with 0-4 seeded corruptions: ops moved earlier, ends before starts,
    sync / optimizer ops dropped or duplicated, syncs pulled before their
    weight updates, adjacent ops of different kinds swapped."""
    r = random.Random(seed)
    st = [[[_kind(o.kind), o.stage, o.start, o.end, o.size, o.iteration, o.microbatch_id]
           for o in stage] for stage in schedule_ops]
    for _ in range(r.randint(0, 4)):
        s = r.randrange(len(st))
        ops = st[s]
        if not ops:
            continue
        mode = r.randrange(6)
        j = r.randrange(len(ops))
        o = ops[j]
        if mode == 0:
            d = r.uniform(0.1, 2.0) * (o[3] - o[2] + 0.1)
            o[2] -= d
            o[3] -= d * r.choice([0.0, 0.5, 1.0])
        elif mode == 1:
            o[3] = o[2] - r.uniform(0.01, 1.0)
        elif mode == 2:
            closes = [q for q, x in enumerate(ops) if x[0] in "SO"]
            if closes:
                del ops[r.choice(closes)]
        elif mode == 3:
            closes = [q for q, x in enumerate(ops) if x[0] in "SO"]
            if closes:
                q = r.choice(closes)
                ops.insert(q + 1, list(ops[q]))
        elif mode == 4:
            syncs = [q for q, x in enumerate(ops) if x[0] == "S"]
            if syncs:
                x = ops[r.choice(syncs)]
                x[2] -= r.uniform(0.05, 3.0)
        else:
            if j + 1 < len(ops) and (ops[j][0] != ops[j + 1][0] or ops[j][6] is None):
                ops[j], ops[j + 1] = ops[j + 1], ops[j]
    return st
