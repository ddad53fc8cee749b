"""The multi-GPU path's host logic on CPU: 2 and 4 processes (gloo), each plans
its shards' arrival/departure replans in one launch and the plans are
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
    shards = MG.shards_of_rank(rank, world, 8)  # strong scaling: shard g on rank g % world
    assert shards == [g for g in range(8) if g % world == rank]
    reqs = []
    for s in shards:
        sreq = MG.shard_requests(s, MG.initial_peaks(p, [s]))
        reqs += sreq[:2] + sreq[-1:]  # a bounded subset per shard keeps the test fast
    outs = MG.plan_shards(p, reqs)
    got = MG.gather_plans(outs, [r[0] for r in reqs], rank, world)
    if rank == 0:
        q.put([[(n, h[:40], fp) for n, h, fp in part] for part in got])
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_shard_and_gather(world):
    """C5 strong scaling (bench.py --gpus N): the 8 shards round-robin over the
    ranks, each rank plans its shards' replans in one launch, rank 0 gathers
    every plan and each matches the reference fixture of that replan."""
    lib = ensure_emu()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, lib, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(res) == world
    names = [n for part in res for n, _, _ in part]
    assert sorted({n.split(".")[0] for n in names}) == [f"C5s{g}" for g in range(8)]
    for r, part in enumerate(res):  # rank r's part holds exactly its shards
        assert {int(n.split(".")[0][3:]) % world for n, _, _ in part} == {r}
    # every gathered plan matches the reference fixture for that replan
    from helpers import golden
    gold = {c["name"]: c["final_merged_peak"] for c in golden("configs") if c["ratio"] is None}
    for n, _, fp in (x for part in res for x in part):
        if n in gold:
            assert fp == gold[n], n
