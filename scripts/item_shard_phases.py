"""Phases of distributed.exhaustive_plan_sharded under torchrun (C4): the
rank's item-range arg-min, the key all-gather, the winner decode and the
plan assembly (winner detail).  Usage: torchrun --nproc-per-node N
scripts/item_shard_phases.py"""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_15536_b200 import SearchConfig, instances  # noqa: E402
from paper_2505_15536_b200 import distributed as DI  # noqa: E402
from paper_2505_15536_b200.engine import Engine  # noqa: E402
from paper_2505_15536_b200.layout import packed_instance  # noqa: E402
from paper_2505_15536_b200.planner import assemble  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
spec = instances.config("c4")
model, topo, groups = instances.build(spec)
cfg = SearchConfig(seed=0)
eng = Engine(rank)
ph = {k: [] for k in ("load", "local", "reduce", "decode", "assemble", "api")}
for it in range(40):
    dist.barrier()
    t0 = time.perf_counter()
    packed = packed_instance(model, topo, groups, 1.25)
    eng.load(packed)
    k = packed.n_fgs
    NC, NP, n_items = DI.space_dims(packed.n_layers, k, len(packed.batches), len(packed.micros))
    nbm = len(packed.batches) * len(packed.micros)
    t1 = time.perf_counter()
    lo, hi = DI.shard_items(n_items, world, rank)
    st, b, msg = eng.argmin_items_status(lo, hi)
    key = (b.cost, DI.tie_of_index(b.index, NC, NP, nbm))
    t2 = time.perf_counter()
    cost, tie = DI.reduce_key(key, None, torch.device("cuda"), None)
    t3 = time.perf_counter()
    order, counts, bm = DI.decode_candidate(tie, NC, NP, nbm, packed.n_layers, k)
    t4 = time.perf_counter()
    assemble(packed, eng, np.array(order, np.uint8), np.array(counts, np.uint8), bm)
    t5 = time.perf_counter()
    dist.barrier()
    t6 = time.perf_counter()
    DI.exhaustive_plan_sharded(model, topo, groups, cfg, engine=eng)
    t7 = time.perf_counter()
    if it >= 10:
        for kk, v in zip(("load", "local", "reduce", "decode", "assemble", "api"),
                         (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t7 - t6)):
            ph[kk].append(v)
out = {kk: round(float(np.median(v)) * 1e3, 4) for kk, v in ph.items()}
allo = [None] * world
dist.all_gather_object(allo, out)
if rank == 0:
    for r, o in enumerate(allo):
        print(world, r, o)
dist.destroy_process_group()
