"""C5: concurrent dynamic workloads sharded across GPUs, one process per GPU.

The reference plans every arrival/departure with a fresh memsched::build_plan
over the active job set (Orchestrator::rebuild, orchestrator.cpp:96-110,
called from run_scenario, scenario.cpp:200-262). Jobs
interact only through SwapBudget and the merged-peak budget of ONE build, so a
shard of workloads is the planning unit:

  * shard g = workloads w{8g}..w{8g+7} (configs.c5_job), 8 arrivals then 7
    departures, each a build_plan over the active set with
    memory_budget = 70% of that set's summed initial peaks;
  * rank r plans the shards assigned to it -- every replan of every shard in
    ONE kernel launch (one CTA per replan);
  * the only exchange is a gather of the serialised plans to rank 0
    (torch.distributed.gather_object over NCCL, or gloo on CPU).
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

from . import configs as CF

SHARD_SIZE = 8


def shard_requests(shard: int, initial_peaks: Dict[str, int]) -> List[Tuple[str, list, dict]]:
    """(name, jobs, planner_config) for every replan of one shard."""
    jobs = {k: CF.c5_job(k) for k in range(SHARD_SIZE * shard, SHARD_SIZE * shard + SHARD_SIZE)}
    out = []
    for i, active in enumerate(CF.c5_shard_events(shard)):
        js = [jobs[k] for k in active]
        budget = CF.budget_of([initial_peaks[g["job_id"]] for g, _ in js])
        out.append((f"C5s{shard}.{i}", js, CF.planner_config(budget)))
    return out


def shards_of_rank(rank: int, world: int, n_shards: int) -> List[int]:
    return [g for g in range(n_shards) if g % world == rank]


def initial_peaks(planner, shards: Sequence[int]) -> Dict[str, int]:
    """Initial per-job peaks (make_job_context's report) for the shards' jobs,
    from one planner launch (one single-job group per workload)."""
    ks = [k for s in shards for k in range(SHARD_SIZE * s, SHARD_SIZE * s + SHARD_SIZE)]
    groups = [[CF.c5_job(k)] for k in ks]
    outs = planner.build_plan_groups(groups, {"pcie_bandwidth": CF.BW, "transfer_setup": CF.SETUP,
                                              "memory_budget": 0}, with_views=False)
    return {"w%02d" % k: o["merged_peak_history"][0] for k, o in zip(ks, outs)}


def plan_shards(planner, reqs: Sequence[Tuple[str, list, dict]], with_views: bool = False) -> List[dict]:
    """Every replan of the given requests in ONE launch (per-group budgets)."""
    return planner.build_plan_groups([r[1] for r in reqs], [r[2] for r in reqs], with_views=with_views)


def gather_plans(results: Sequence[dict], names: Sequence[str], rank: int, world: int):
    """Serialised plans of every rank, gathered on rank 0 (None elsewhere)."""
    payload = [(n, r["plans_json"], r["final_merged_peak"]) for n, r in zip(names, results)]
    if world == 1:
        return [payload]
    import torch.distributed as dist
    out = [None] * world if rank == 0 else None
    dist.gather_object(payload, out, dst=0)
    return out
