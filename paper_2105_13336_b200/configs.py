"""The BASELINE.json workload configurations.

Every config is a list of *plan requests*: one build_plan call each, as
(jobs, planner_config) with jobs = [(graph, latencies), ...].

  C1  VGG-16 b32, single workload                                   1 request
  C2  ResNet-50 b64, single workload (wrapped Opt-phase pairs)       1 request
  C3  InceptionV3 -> +DenseNet -> +VGG-16 arriving in sequence       3 requests
  C5  64 workloads (w00..w63), 8 per shard; per shard 8 arrivals
      then 7 departures, each a replan of the active set            15 per shard
  C4  ~1M-access GPT-2-medium trace (paper_2105_13336_b200.gpt2)    1 request

Planner settings follow acceptance criterion 5 (test_acceptance.cpp:195-202):
pcie_bandwidth 256, transfer_setup 1, memory_budget = 70% of the set's
summed initial peak (integer: sum * 7 // 10), max_swap_ratio 1.0. The
"ratio 0.1" variants exercise the recomputation branch.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Tuple

from . import workload as W

BW = 256
SETUP = 1
C5_FAMILIES = [("vgg16", 32), ("resnet50", 64), ("inception_v3", 32), ("inception_v4", 32), ("densenet", 32)]

# Summed initial per-job peaks (make_job_context report, swap_planner.cpp:156-169)
# of every job, from the reference (tests/test_configs.py re-derives them).
INITIAL_PEAK = {
    "vgg16": 66336, "resnet50": 124192, "inception_v3": 71360, "densenet": 55840,
}

# C4: the GPT-2-medium trace (workload.gpt2_workload), 70 micro-batches =
# 990,518 accesses; the 1-micro-batch instance (16,445 accesses) is the
# bounded CPU sample the reference can still plan (~80 s). Initial peaks from
# the restated oracle's make_job_context (equal to the reference's on every
# C4-family instance the reference finishes).
C4_MICRO_BATCHES = 70
C4_INITIAL_PEAK = {70: 5548992512, 10: 5297088512, 1: 4654684160}


def c4_request(micro_batches: int = C4_MICRO_BATCHES):
    """(name, jobs, config) of C4 at the given micro-batch count (70 % budget)."""
    from paper_2105_13336_b200 import workload as W
    cfg = {"pcie_bandwidth": BW, "transfer_setup": SETUP,
           "memory_budget": C4_INITIAL_PEAK[micro_batches] * 7 // 10}
    return (f"C4.M{micro_batches}", [W.c4_job(micro_batches)], cfg)


def budget_of(initial_peaks: List[int]) -> int:
    return sum(initial_peaks) * 7 // 10


def planner_config(budget: int, ratio: Optional[float] = None, jobs=None) -> dict:
    cfg = {"pcie_bandwidth": BW, "transfer_setup": SETUP, "memory_budget": int(budget)}
    if ratio is not None and jobs is not None:
        cfg["max_swap_ratios"] = {g["job_id"]: ratio for g, _ in jobs}
    return cfg


def c5_job(k: int) -> Tuple[dict, dict]:
    fam, b = C5_FAMILIES[k % 5]
    g = W.generate_workload(fam, b, 0, 0, "w%02d" % k)
    return g, W.true_latency_table(g, 13 + k)


def c5_shard_events(shard: int) -> List[List[int]]:
    """Active job sets (job indices) of one shard: 8 arrivals then 7 departures."""
    ids = list(range(8 * shard, 8 * shard + 8))
    sets = [ids[: i + 1] for i in range(8)]
    sets += [ids[i + 1:] for i in range(7)]
    return sets


class Request:
    """One build_plan call: jobs + planner config (budget needs initial peaks)."""

    def __init__(self, jobs, ratio: Optional[float] = None, budget: Optional[int] = None, name: str = ""):
        self.jobs = jobs
        self.ratio = ratio
        self.budget = budget
        self.name = name

    def config(self, initial_peaks: Optional[Dict[str, int]] = None) -> dict:
        b = self.budget
        if b is None:
            if initial_peaks is None:
                raise ValueError("budget needs the jobs' initial peaks")
            b = budget_of([initial_peaks[g["job_id"]] for g, _ in self.jobs])
        return planner_config(b, self.ratio, self.jobs)

    @property
    def n_accesses(self) -> int:
        n = 0
        for g, _ in self.jobs:
            n += sum(len(o["inputs"]) + len(o["outputs"]) for o in g["ops"])
        return n


def requests(name: str, ratio: Optional[float] = None) -> List[Request]:
    """Plan requests of config `name` in {"C1","C2","C3","C5","C5s<g>"}."""
    if name == "C1":
        jobs = [W.job("vgg16", 32, "vgg16")]
        return [Request(jobs, ratio, None, "C1")]
    if name == "C2":
        jobs = [W.job("resnet50", 64, "resnet50")]
        return [Request(jobs, ratio, None, "C2")]
    if name == "C3":
        all_jobs = [W.job("inception_v3", 32, "inception_v3"), W.job("densenet", 32, "densenet"),
                    W.job("vgg16", 32, "vgg16")]
        return [Request(all_jobs[: i + 1], ratio, None, f"C3.{i + 1}") for i in range(3)]
    if name.startswith("C5s"):
        g = int(name[3:])
        jobs = {k: c5_job(k) for k in range(8 * g, 8 * g + 8)}
        return [Request([jobs[k] for k in s], ratio, None, f"C5s{g}.{i}") for i, s in enumerate(c5_shard_events(g))]
    if name == "C5":
        out = []
        for g in range(8):
            out.extend(requests(f"C5s{g}", ratio))
        return out
    raise ValueError(name)
