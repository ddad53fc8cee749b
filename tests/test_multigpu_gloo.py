"""The multi-GPU path's host logic on CPU: two processes (gloo), each plans
its shard's arrival/departure replans in one launch and the plans are
gathered on rank 0 -- here through the test-only emulation build."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from helpers import ensure_emu


def _worker(rank, world, port, lib, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2105_13336_b200 import multigpu as MG
    from paper_2105_13336_b200.planner import Planner
    p = Planner(lib_path=lib)
    shards = MG.shards_of_rank(rank, world, 4)
    reqs = []
    for s in shards:
        reqs += MG.shard_requests(s, MG.initial_peaks(p, [s]))
    reqs = reqs[:5] + reqs[-3:]  # a bounded subset per shard set keeps the test fast
    outs = MG.plan_shards(p, reqs)
    got = MG.gather_plans(outs, [r[0] for r in reqs], rank, world)
    if rank == 0:
        q.put([[(n, h[:40], fp) for n, h, fp in part] for part in got])
    dist.destroy_process_group()


def test_two_rank_shard_and_gather():
    lib = ensure_emu()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, lib, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(res) == 2
    names = [n for part in res for n, _, _ in part]
    assert names[0].startswith("C5s0.") and any(n.startswith("C5s1.") for n in names)
    # every gathered plan matches the reference fixture for that replan
    from helpers import golden
    gold = {c["name"]: c["final_merged_peak"] for c in golden("configs") if c["ratio"] is None}
    for n, _, fp in (x for part in res for x in part):
        if n in gold:
            assert fp == gold[n], n
