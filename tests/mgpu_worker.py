"""torchrun worker for tests/test_multigpu.py (one rank per GPU, NCCL).

Runs the sharded product paths on every rank and writes rank 0's answers to
the JSON file named by argv[1]:
  exhaustive  distributed.exhaustive_plan_sharded on golden cases
  errors      the exception class every rank raised for erroring instances
  snapshots   distributed.replan_snapshots_sharded over C3 snapshots of C2
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def main():
    import torch
    import torch.distributed as dist
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import golden_io as G
    from cases import load_case
    import paper_2505_15536_b200 as P
    from paper_2505_15536_b200 import distributed as DI
    from paper_2505_15536_b200 import instances as I
    from paper_2505_15536_b200 import replan as R
    from paper_2505_15536_b200.engine import Engine
    from paper_2505_15536_b200.layout import PackedInstance
    eng = Engine(local)
    out = {"world": dist.get_world_size(), "exhaustive": {}, "errors": {}}
    for name in ["c1j", "c2", "c2j", "rand10", "k5n9", "k6n8", "k8n9", "c4", "c4j"]:
        doc, model, topo, groups = load_case(name)
        res = DI.exhaustive_plan_sharded(model, topo, groups, P.SearchConfig(seed=0), engine=eng)
        out["exhaustive"][name] = G.normalize_result(res)
    for name in ["err_gateway", "err_intra_bw"]:
        doc, model, topo, groups = load_case(name)
        try:
            DI.exhaustive_plan_sharded(model, topo, groups, P.SearchConfig(seed=0), engine=eng)
            out["errors"][name] = None
        except Exception as e:
            out["errors"][name] = type(e).__name__
    spec = I.config("c2")
    model, topo, groups = I.build(spec)
    packed = PackedInstance(model, topo, groups, 1.25)
    bws = R.bandwidth_matrices(packed, [I.snapshot_multipliers(spec, j) for j in range(37)])
    res = DI.replan_snapshots_sharded(model, topo, groups, P.SearchConfig(seed=0), bws, engine=eng)
    out["snapshots"] = [r if isinstance(r, tuple) else type(r).__name__ for r in res]
    # snapshots whose tables raise (a device cut off from every link): the
    # device-resident sharded path hands them to their owners' status path;
    # the answers must equal the single-engine re-plan's
    import numpy as np
    bws2 = bws.copy()
    for j in (3, 11, 20, 36):
        d = 1 + j % 5
        bws2[j][d, :] = 0.0
        bws2[j][:, d] = 0.0
    fix = lambda rr: [r if isinstance(r, tuple) else type(r).__name__ for r in rr]  # noqa: E731
    got = fix(DI.replan_snapshots_sharded(model, topo, groups, P.SearchConfig(seed=0), bws2, engine=eng))
    exp = fix(R.replan_snapshots(model, topo, groups, P.SearchConfig(seed=0), bws2, engine=eng))
    out["flagged_equal"] = got == exp
    # pinned host matrices (the bench's e2e input)
    pinned = torch.from_numpy(np.ascontiguousarray(bws2)).pin_memory().numpy()
    out["pinned_equal"] = fix(DI.replan_snapshots_sharded(model, topo, groups, P.SearchConfig(seed=0),
                                                          pinned, engine=eng)) == exp
    # an instance whose own tables raise: the asynchronous path is refused on
    # every rank, all ranks take the host-staged path together
    docE, mE, tE, gE = load_case("err_gateway")
    pE = PackedInstance(mE, tE, gE, 1.25)
    bwE = np.stack([pE.bw] * 5)
    gotE = fix(DI.replan_snapshots_sharded(mE, tE, gE, P.SearchConfig(seed=0), bwE, engine=eng))
    expE = fix(R.replan_snapshots(mE, tE, gE, P.SearchConfig(seed=0), bwE, engine=eng))
    out["refused_equal"] = gotE == expE
    out["refused_kinds"] = sorted(set(gotE))
    out["flagged_errors"] = sum(not isinstance(r, (tuple, list)) for r in got)
    # peer-memory all-gather (NVLink stores + arrival counter) vs NCCL's, for
    # the K6 winners of C3 snapshot shards, over several epochs
    import numpy as np
    world, rank = dist.get_world_size(), dist.get_rank()
    eng.load(packed)
    S = 37
    width = -(-S // world)
    lo, hi = DI.shard_items(S, world, rank)
    d_bw = torch.from_numpy(np.ascontiguousarray(bws[lo:hi])).cuda()
    d_keys = torch.zeros((width, 2), dtype=torch.int64, device="cuda")
    d_flags = torch.zeros(width, dtype=torch.int32, device="cuda")
    ref = torch.empty((world * width, 2), dtype=torch.int64, device="cuda")
    pg = DI.PeerGather(eng, width * 16)
    out["peer_ok"] = pg.ok
    out["peer_equal"] = []
    for epoch in range(3):
        if hi > lo:
            eng.replan_snapshots_async(d_bw.data_ptr(), hi - lo, d_keys.data_ptr(), d_flags.data_ptr())
        torch.cuda.synchronize()
        d_keys[0, 1] += epoch  # a different payload per epoch
        torch.cuda.synchronize()
        dist.all_gather_into_tensor(ref, d_keys)
        if pg.ok:
            pg.gather(d_keys.data_ptr())
            got = np.frombuffer(pg.read(), dtype=np.int64).reshape(-1, 2)
            out["peer_equal"].append(bool((got == ref.cpu().numpy()).all()))
    # back-to-back epochs in stream order (no host sync between gathers) with
    # rank 0 delayed before it consumes each table: the alternating tables
    # keep epoch e's table intact until its owner has copied it out
    out["peer_pipelined_equal"] = []
    if pg.ok:
        class _Cai:  # a torch view of a raw device address
            def __init__(self, ptr, n):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8",
                                                 "data": (ptr, False), "version": 3}
        n = world * width * 2
        E = 6
        pay = [d_keys.clone() for _ in range(E)]
        for e in range(E):
            pay[e][:, 1] += 1000 * (e + 1) + rank
        outs = [torch.empty(n, dtype=torch.int64, device="cuda") for _ in range(E)]
        torch.cuda.synchronize()
        dist.barrier()
        est = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", torch.cuda.current_device()))
        with torch.cuda.stream(est):
            for e in range(E):
                pg.gather(pay[e].data_ptr())
                if rank == 0:
                    torch.cuda._sleep(2_000_000)
                outs[e].copy_(torch.as_tensor(_Cai(pg.records, n), device="cuda"))
        torch.cuda.synchronize()
        for e in range(E):
            dist.all_gather_into_tensor(ref, pay[e])
            out["peer_pipelined_equal"].append(bool((outs[e].cpu().numpy() ==
                                                     ref.cpu().numpy().reshape(-1)).all()))
    dist.barrier()
    pg.close(dist.barrier)
    gathered = [None] * dist.get_world_size()
    dist.all_gather_object(gathered, out)
    if dist.get_rank() == 0:
        out["all_ranks_equal"] = all(g == gathered[0] for g in gathered)
        with open(sys.argv[1], "w") as f:
            json.dump(out, f)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
