"""Phases of the sharded snapshot re-plan through the public API under
torchrun: the host-staged form (gp_replan_snapshots + a host-record
all-gather) vs distributed.replan_snapshots_sharded (device-resident keys
gathered straight from HBM).  Usage: torchrun --nproc-per-node N
scripts/e2e_phases.py"""
import os, sys, time
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
from paper_2505_15536_b200 import instances, replan, SearchConfig
from paper_2505_15536_b200 import distributed as DI
from paper_2505_15536_b200.engine import Engine, best_fields
from paper_2505_15536_b200.layout import packed_instance
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
spec = instances.config("c4"); model, topo, groups = instances.build(spec)
packed = packed_instance(model, topo, groups, 1.25)
eng = Engine(rank).load(packed)
S = 128
bws = replan.bandwidth_matrices(packed, [instances.snapshot_multipliers(spec, j) for j in range(S)])
bws = torch.from_numpy(bws).pin_memory().numpy()
lo, hi = DI.shard_items(S, world, rank)
ph = {k: [] for k in ("replan", "gather", "decode", "total", "api_total")}
cfg = SearchConfig(seed=0)
for it in range(25):
    dist.barrier(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    bests, status = eng.replan_snapshots(bws[lo:hi])
    t1 = time.perf_counter()
    cost, index = best_fields(bests, hi - lo)
    rec = np.zeros((hi - lo, 3), dtype=np.int64)
    rec[:, 0] = cost.view(np.int64); rec[:, 1] = index.view(np.int64); rec[:, 2] = status
    allrec = DI.gather_snapshot_records(rec, S, None, torch.device("cuda"))
    t2 = time.perf_counter()
    res = DI.decode_snapshot_records(packed, allrec)
    t3 = time.perf_counter()
    dist.barrier(); torch.cuda.synchronize()
    t4 = time.perf_counter()
    res2 = DI.replan_snapshots_sharded(model, topo, groups, cfg, bws, engine=eng)
    t5 = time.perf_counter()
    assert (res2.cost == res.cost).all() and (res2.index == res.index).all() and (res2.status == res.status).all()
    if it >= 5:
        ph["api_total"].append(t5 - t4)
        ph["replan"].append(t1 - t0); ph["gather"].append(t2 - t1); ph["decode"].append(t3 - t2); ph["total"].append(t3 - t0)
out = {k: float(np.median(v)) * 1e3 for k, v in ph.items()}
allo = [None] * world
dist.all_gather_object(allo, out)
if rank == 0:
    for r, o in enumerate(allo): print(world, r, {k: round(v, 3) for k, v in o.items()})
dist.destroy_process_group()
