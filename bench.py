#!/usr/bin/env python3
"""Headline benchmark: TENSILE scheduling-plan generation on B200.

metric  tensor-access events/s = accesses of the planned trace(s) / plan-gen
        time of memsched::build_plan (BASELINE.json "metric"); also reported:
        plan-gen ms per workload set and peak-mem bytes saved.
step    N = 1 (default): one build_plan of C4, the ~1 M-access GPT-2-medium
        trace (990,518 accesses) -- BASELINE.json publishes no number on any
        config, so the headline is the largest single-GPU configuration.
        N > 1 (default): C5 strong scaling -- the 64 workloads' 8 shards
        (8 arrivals + 7 departures = 15 replans each, 120 replans in all) are
        split over the ranks, shard g on rank g % N, every replan of a rank in
        ONE launch; the plans are gathered on rank 0 (NCCL) and checked there.
        --workload C1|C2|C3|C4|C5 overrides.
value   device time of the planning kernel with inputs resident in HBM,
        CUDA events on the launching stream, L2 flushed between steps; whole
        job = all ranks' events / max-over-ranks time.
e2e     the same metric through the C-ABI call a user makes
        (tsl_build_plan_groups: host validation + topo order + one H2D +
        kernel + one D2H + results) from host buffers, wall clock.

--impl reference times the reference's CPU scheduler on this box's host on
the same workload: the unmodified reference sources compiled by
oracle/Makefile (oracle/_ref) where it can finish (C1-C3, C5: the 8 shards in
min(8, cores) processes), and the restated oracle port on C4 (the reference
needs days for 1 M accesses; its own 1-micro-batch sample is timed beside it).
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tensor-access events/s"
UNIT = "events/s"
C4_SAMPLE_MB = 10      # our arm's cpu_baseline: the port on C4's first 10 micro-batches (~5-15 s)
REF_ARM_BUDGET_S = 150  # the reference arm stops adding steps after this much host time


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["auto", "C1", "C2", "C3", "C4", "C5"], default="auto")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="bounded CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    a = ap.parse_args()
    return a


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def resolve(name: str, world: int) -> str:
    """auto: C4 on one GPU (the tier's N=1 config), C5 strong scaling on N > 1."""
    return name if name != "auto" else ("C4" if world == 1 else "C5")


def c5_peaks(shards, planner=None):
    """Initial per-job peaks of the shards' workloads (make_job_context):
    from the device planner on the GPU arm, from the reference on the CPU arm."""
    from paper_2105_13336_b200 import configs as CF
    from paper_2105_13336_b200 import multigpu as MG
    if planner is not None:
        return MG.initial_peaks(planner, shards)
    from oracle import ref
    return ref.initial_peaks([CF.c5_job(k) for s in shards for k in range(8 * s, 8 * s + 8)])


def workload(name: str, rank: int = 0, world: int = 1, planner=None):
    """[(request name, jobs, planner config)] this rank plans per step."""
    from paper_2105_13336_b200 import configs as CF
    if name in ("C1", "C2"):
        req = CF.requests(name)[0]
        return [(req.name, req.jobs, req.config(CF.INITIAL_PEAK))]
    if name == "C3":  # one replan per arrival: {inception_v3}, {+densenet}, {+vgg16}
        return [(r.name, r.jobs, r.config(CF.INITIAL_PEAK)) for r in CF.requests("C3")]
    if name == "C4":
        return [CF.c4_request()]
    if name.startswith("C4.M"):  # bounded CPU samples of the same generator
        return [CF.c4_request(int(name[4:]))]
    from paper_2105_13336_b200 import multigpu as MG
    shards = MG.shards_of_rank(rank, world, 8)  # C5: shard g on rank g % world
    peaks = c5_peaks(shards, planner)
    return [r for s in shards for r in MG.shard_requests(s, peaks)]


def n_accesses(jobs) -> int:
    return sum(len(o["inputs"]) + len(o["outputs"]) for g, _ in jobs for o in g["ops"])


WORKLOAD_DESC = {
    "C1": "C1 VGG-16 b32, single workload, one build_plan",
    "C2": "C2 ResNet-50 b64, single workload with across-iteration (Opt-phase) swap-ins, one build_plan",
    "C3": "C3 InceptionV3 + DenseNet + VGG-16 arriving in sequence, one replan per arrival (3 build_plans)",
    "C4": "C4 GPT-2-medium seq-1024 training trace, 70 micro-batches, 990,518 accesses, one build_plan",
    "C5": "C5 64 concurrent dynamic workloads in 8 shards, 8 arrivals + 7 departures per shard = 120 replans; "
          "strong scaling: shard g on GPU g % N",
}
def job_config(name: str, world: int, reqs_total: int, ev_total: int) -> dict:
    """The workload description both arms print (identical dicts)."""
    from paper_2105_13336_b200 import configs as CF
    return {"workload": WORKLOAD_DESC[name], "requests": reqs_total, "accesses_per_step": ev_total,
            "pcie_bandwidth": CF.BW, "transfer_setup": CF.SETUP,
            "memory_budget": "70% of each set's initial peak", "max_swap_ratio": 1.0,
            "parallelism": (f"{world} GPU(s), shards round-robin" if name == "C5" else
                            f"{world} GPU(s), replicas" if world > 1 else "1 GPU")}


def c5_totals():
    """(replans, accesses) of the whole C5 job (all 8 shards)."""
    from paper_2105_13336_b200 import configs as CF
    ev = 0
    for s in range(8):
        jobs = {k: CF.c5_job(k) for k in range(8 * s, 8 * s + 8)}
        for active in CF.c5_shard_events(s):
            ev += n_accesses([jobs[k] for k in active])
    return 120, ev


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)

    def stop(self) -> dict:
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        rows = []
        if self.path and os.path.exists(self.path):
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
            os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(float(r[1]) for r in rows), "sm_max_mhz": float(rows[0][2]),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit()),
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
def time_reference(reqs, kind: str):
    """One step of the CPU scheduler over reqs: ms (the reference library, or
    the restated oracle port)."""
    from oracle import ref, tslo
    ms = 0.0
    for _, jobs, cfg in reqs:
        if kind == "reference":
            ms += ref.build_plan(jobs, cfg, repeats=1)[1]["times_ms"][0]
        else:
            ms += tslo.build_plan(jobs, cfg)["ms"]
    return ms


def cpu_reference(reqs, seconds: float, kind: str, max_steps: int = 10 ** 9):
    """Repeated steps for about `seconds` of host time: (events/s, median ms, steps)."""
    ev = sum(n_accesses(j) for _, j, _ in reqs)
    times = []
    t_end = time.perf_counter() + seconds
    while (time.perf_counter() < t_end or not times) and len(times) < max_steps:
        times.append(time_reference(reqs, kind))
    ms = statistics.median(times)
    return ev / (ms / 1e3), ms, len(times)


def host_cpu() -> dict:
    """The GPU box's host CPU (state the model and core count)."""
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            model = next((l.split(":", 1)[1].strip() for l in f if l.startswith("model name")), "")
    except OSError:
        pass
    return {"model": model, "logical_cpus": os.cpu_count()}


def _shard_plan_ms(shard: int):
    """One C5 shard's 15 replans through the reference (a worker process)."""
    sys.path.insert(0, ROOT)
    from paper_2105_13336_b200 import multigpu as MG
    reqs = MG.shard_requests(shard, c5_peaks([shard]))
    return sum(n_accesses(j) for _, j, _ in reqs), time_reference(reqs, "reference")


def cpu_parallel_shards(shards=range(8)) -> dict:
    """C5 on the host: the shards in min(8, cores) processes (one build_plan
    per core: the reference has no threads); throughput = all events / the
    slowest process."""
    import multiprocessing as mp
    shards = list(shards)
    n = max(1, min(len(shards), os.cpu_count() or 1))
    with mp.get_context("spawn").Pool(n) as pool:
        res = pool.map(_shard_plan_ms, shards)
    # processes run their shards in turn: the wall time of one is its shards' sum
    per_proc = [0.0] * n
    for i, (_, ms) in enumerate(res):
        per_proc[i % n] += ms
    ev = sum(e for e, _ in res)
    slow = max(per_proc)
    return {"value": ev / (slow / 1e3), "ms_per_step": slow, "processes": n, "events": ev,
            "sample": f"all {len(shards)} shards x 15 replans, {n} processes (reference, -O3)"}


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(name: str):
    """DRAM bytes per launch of the planning kernel on this workload, from the
    newest committed ncu capture (profiles/r*/ncu_traffic_<workload>.json)."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", f"ncu_traffic_{name}.json")), reverse=True):
        d = json.load(open(p))
        return d.get("dram_bytes_per_launch"), os.path.relpath(p, ROOT)
    return None, None


def plan_digest(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def golden_parity(name: str, digests) -> str:
    """In-bench parity: [(request name, save_plans sha256)] vs the fixtures."""
    if name == "C4":  # digests of the restated oracle (the reference cannot plan C4)
        p = os.path.join(ROOT, "tests", "golden", "c4.json")
        d = json.load(open(p))["cases"].get("M70") if os.path.exists(p) else None
        if d is None:
            return "unchecked (no oracle digest)"
        ok = all(h == d["plans_sha256"] for _, h in digests)
        return "byte-identical save_plans vs the restated oracle (C4)" if ok else "MISMATCH vs oracle digest (C4)"
    p = os.path.join(ROOT, "tests", "golden", "configs.json")
    if not os.path.exists(p):
        return "unchecked"
    gold = {c["name"]: c for c in json.load(open(p)) if c["ratio"] is None}
    seen = 0
    for n, h in digests:
        g = gold.get(n)
        if g is None:
            continue
        if h != g["plans_sha256"]:
            return f"MISMATCH on {n}"
        seen += 1
    return f"byte-identical save_plans vs the reference on {seen} of {len(digests)} plan(s)"


# ---------------------------------------------------------------------------
def run_reference(a, rank, world):
    if rank != 0:
        return
    name = resolve(a.workload, world)
    from oracle import ref
    have_ref = ref.available()
    extra = {}
    if name == "C5":  # the whole job: 8 shards over the host's cores
        if not have_ref:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}), flush=True)
            return
        n_req, ev = c5_totals()
        runs = []
        t0 = time.perf_counter()
        for _ in range(max(1, a.steps)):
            runs.append(cpu_parallel_shards())
            if time.perf_counter() - t0 > REF_ARM_BUDGET_S:
                break
        ms = statistics.median(r["ms_per_step"] for r in runs)
        kind, cores = "reference", runs[0]["processes"]
        sample = f"{len(runs)} x " + runs[0]["sample"]
    else:
        reqs = workload(name)
        n_req, ev = len(reqs), sum(n_accesses(j) for _, j, _ in reqs)
        # C4: the reference cannot finish 1 M accesses; the
        # restated oracle port plans the same full trace, one step at a time
        kind = "port" if (name == "C4" or not have_ref) else "reference"
        cores = 1
        warm = 0 if name == "C4" else a.warmup
        for _ in range(warm):
            time_reference(reqs, kind)
        times = []
        t0 = time.perf_counter()
        for _ in range(max(1, a.steps)):
            times.append(time_reference(reqs, kind))
            if time.perf_counter() - t0 > REF_ARM_BUDGET_S:
                break
        ms = statistics.mean(times)
        sample = (f"{len(times)} x build_plan of the full {name} on 1 host thread "
                  f"({'restated oracle port, oracle/tensile_oracle.cpp' if kind == 'port' else 'oracle/_ref: reference sources compiled -O3'})")
        if name == "C4" and have_ref:
            # the reference's own code on the largest C4 sample it finishes in
            # about a minute, and the size-sweep extrapolation
            sreq = workload("C4.M1")
            sev = sum(n_accesses(j) for _, j, _ in sreq)
            sms = time_reference(sreq, "reference")
            expo = 2.15  # reference plan time ~ A^2.15
            extra["reference_sample"] = {
                "value": sev / (sms / 1e3), "unit": UNIT, "ms": sms, "accesses": sev, "kind": "reference",
                "sample": "C4 generator at 1 micro-batch (16,445 accesses), oracle/_ref, 1 thread",
                "extrapolated_full_c4_s": round(sms / 1e3 * (ev / sev) ** expo, 1),
                "extrapolation": f"plan time x (990,518 / {sev})^{expo} (SURVEY.md §6 size sweep)"}
        times_n = len(times)
    value = ev / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": len(runs) if name == "C5" else times_n, "steps_requested": a.steps,
            "warmup": 0 if name in ("C4", "C5") else a.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if name == "C5" else "weak", "vs_baseline": None, "dtype": "int64",
            "impl": "reference",
            "data": "synthetic traces from the reference generator (workload.cpp) and the C4 GPT-2 generator, "
                    "latency seed 13",
            "config": job_config(name, world, n_req, ev), "plan_gen_ms": ms,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "host": host_cpu(),
                             "sample": sample, **extra},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def device_timed(prep, stream, flush, steps):
    """Mean device ms of `steps` launches (CUDA events on the launching
    stream, L2 flushed before each)."""
    import torch
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for e0, e1 in evs:
        flush.zero_()  # on the same stream, outside the event pair
        e0.record(stream)
        prep.launch_async(stream.cuda_stream)
        e1.record(stream)
    torch.cuda.synchronize()
    return statistics.mean(e0.elapsed_time(e1) for e0, e1 in evs)


def run_ours(a, rank, world, local):
    import torch
    from paper_2105_13336_b200 import abi
    from paper_2105_13336_b200 import configs as CF
    from paper_2105_13336_b200.planner import Planner
    name = resolve(a.workload, world)
    # TSL_BENCH_BACKEND=gloo (test only): several ranks may share one GPU, so
    # the N>1 path (shards per rank, barriers, max over ranks, plan gather)
    # can be exercised on a one-GPU box; the driver's runs use NCCL
    backend = os.environ.get("TSL_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(backend)
    planner = Planner(local)
    reqs = workload(name, rank, world, planner)
    groups = [j for _, j, _ in reqs]
    cfgs = [c for _, _, c in reqs]
    ev = sum(n_accesses(j) for j in groups)
    prep = planner.prepare(groups, cfgs)
    # a real (non-default) stream: the kernel is launched on it and the CUDA
    # events are recorded on it
    stream = torch.cuda.Stream(device=f"cuda:{local}")
    torch.cuda.set_stream(stream)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=f"cuda:{local}")  # 256 MB > L2
    # e2e path: the caller's packed descriptors, one C-ABI call per step
    cfg_arr, ncfg, keep = planner._configs(cfgs, len(groups))
    descs, arr, offs = planner._pack_groups(groups)
    res = (C.c_void_p * len(groups))()
    L = planner.lib
    stats = abi.TslStats()

    def e2e_step():
        rc = L.tsl_build_plan_groups(planner._ctx, arr, offs, len(groups), cfg_arr, ncfg, res)
        if rc:
            raise RuntimeError(L.tsl_last_error().decode())
        peak = sum(L.tsl_result_final_merged_peak(res[g]) for g in range(len(groups)))
        L.tsl_result_stats(res[0], C.byref(stats))
        for g in range(len(groups)):
            L.tsl_result_destroy(res[g])
        return peak

    for _ in range(a.warmup):
        prep.launch_async(stream.cuda_stream)
        e2e_step()
    torch.cuda.synchronize()
    # ---- device-timed region: kernel only, inputs resident, L2 flushed between steps ----
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    wall0 = time.perf_counter()
    dev_ms = device_timed(prep, stream, flush, a.steps)
    wall_dev = time.perf_counter() - wall0
    clocks = sampler.stop()
    # ---- e2e region: host buffers -> C-ABI -> host results ----
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / a.steps
    # whole job: every rank's events over the slowest rank's time
    ev_all, n_req_all = ev, len(reqs)
    if dist:
        dev = f"cuda:{local}" if backend == "nccl" else "cpu"
        t = torch.tensor([dev_ms, e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, e2e_ms = t.tolist()
        n = torch.tensor([ev, len(reqs)], device=dev, dtype=torch.int64)
        dist.all_reduce(n, op=dist.ReduceOp.SUM)
        ev_all, n_req_all = (int(v) for v in n.tolist())
    outs = prep.collect(with_views=False)
    prep.close()
    alg_bytes = sum(o["stats"]["algorithmic_bytes"] for o in outs)
    digests = [(n, plan_digest(o["plans_json"])) for (n, _, _), o in zip(reqs, outs)]
    gather_ms = None
    if name == "C5":  # the only collective: every rank's plans to rank 0
        from paper_2105_13336_b200 import multigpu as MG
        g0 = time.perf_counter()
        parts = MG.gather_plans(outs, [n for n, _, _ in reqs], rank, world)
        gather_ms = (time.perf_counter() - g0) * 1e3
        if rank == 0:
            digests = [(n, plan_digest(text)) for part in parts for n, text, _ in part]
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    parity = golden_parity(name, digests)
    init_peak = (CF.C4_INITIAL_PEAK[CF.C4_MICRO_BATCHES] if name == "C4" else
                 sum(CF.INITIAL_PEAK.get(g["job_id"], 0) for g, _ in groups[-1]) if name != "C5" else None)
    saved = (init_peak - outs[-1]["final_merged_peak"]) if init_peak else None  # the full set (C3: last arrival)
    peak, how = hbm_peak()
    achieved = alg_bytes / (dev_ms / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(name)
    line = {
        "metric": METRIC, "value": ev_all / (dev_ms / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": dev_ms, "higher_is_better": True,
        "scaling": "strong" if name == "C5" else "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic traces from the reference generator (workload.cpp) and the C4 GPT-2 generator, "
                "latency seed 13",
        "config": job_config(name, world, n_req_all, ev_all),
        "timing": {"l2": "flushed between steps (256 MB write)", "per_gpu_requests": len(reqs),
                   "per_gpu_accesses": ev},
        "plan_gen_ms": dev_ms, "peak_bytes_saved": saved, "parity": parity,
        "e2e": {"value": ev_all / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(stats.h2d_bytes), "d2h_bytes_per_step": int(stats.d2h_bytes),
                "host_prep_ms": stats.prep_ms, "launches_per_step": 1},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src, "peak_source": how,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "note": "SURVEY.md 8(d) byte formula over the build / the device-timed launch"},
        "clocks": clocks, "gpu_launches": a.steps, "timed_wall_s": wall_dev,
    }
    if gather_ms is not None:
        line["plan_gather_ms"] = gather_ms
    if world == 1 and name == "C4":
        # the N=1 anchor of the C5 strong-scaling curve (N > 1 runs default to C5)
        c5 = workload("C5", 0, 1, planner)
        p5 = planner.prepare([j for _, j, _ in c5], [c for _, _, c in c5])
        for _ in range(2):
            p5.launch_async(stream.cuda_stream)
        ms5 = device_timed(p5, stream, flush, 5)
        o5 = p5.collect(with_views=False)
        p5.close()
        ev5 = sum(n_accesses(j) for _, j, _ in c5)
        line["c5_strong_scaling_n1"] = {
            "value": ev5 / (ms5 / 1e3), "unit": UNIT, "ms_per_step": ms5, "requests": len(c5), "accesses": ev5,
            "parity": golden_parity("C5", [(n, plan_digest(o["plans_json"])) for (n, _, _), o in zip(c5, o5)])}
    if world == 1 and not a.no_cpu_baseline:
        from oracle import ref
        if name == "C4":  # the port on a bounded sample of the same generator
            sreqs, kind = workload(f"C4.M{C4_SAMPLE_MB}"), "port"
            what = f"C4 generator at {C4_SAMPLE_MB} of 70 micro-batches (143,498 accesses), restated oracle port"
            rate, ms, n = cpu_reference(sreqs, 0.0, kind, 1)
        elif name == "C5":
            d = cpu_parallel_shards()
            rate, ms, n, kind, what = d["value"], d["ms_per_step"], 1, "reference", d["sample"]
        else:
            kind = "reference" if ref.available() else "port"
            rate, ms, n = cpu_reference(reqs, a.cpu_seconds, kind)
            what = f"{name} step, {'oracle/_ref (reference sources -O3)' if kind == 'reference' else 'restated oracle port'}"
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": 8 if name == "C5" else 1, "kind": kind,
                                "ms_per_step": ms, "host": host_cpu(), "sample": f"{n} x {what}"}
        if name == "C5":
            line["cpu_baseline"]["cores"] = d["processes"]
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    a = parse()
    rank, world, local = dist_env()
    if a.impl == "reference":
        run_reference(a, rank, world)
    else:
        run_ours(a, rank, world, local)


if __name__ == "__main__":
    main()
