#!/usr/bin/env python3
"""Headline benchmark: TENSILE scheduling-plan generation on B200.

metric  tensor-access events/s = accesses of the planned trace(s) / plan-gen
        time of memsched::build_plan (BASELINE.json "metric"); also reported:
        plan-gen ms per workload set and peak-mem bytes saved.
step    one build_plan of the workload (default C2: ResNet-50 b64, the
        configuration BASELINE.json's metric is quoted on; configs[1]).
        --workload C5: one GPU plans its 8-workload shard's 15 arrival /
        departure replans in ONE launch (weak scaling, 8 workloads per GPU).
value   device time of the planning kernel with inputs resident in HBM,
        CUDA events on the launching (torch current) stream, L2 flushed
        between steps; whole job = sum over ranks / max-over-ranks time.
e2e     the same metric through the C-ABI call a user makes
        (tsl_build_plan_groups: host validation + topo order + one H2D +
        kernel + one D2H + results) from host buffers, wall clock.

--impl reference times the reference's own CPU scheduler on this box's host
(oracle/_ref/libmemsched_ref.so, the unmodified reference sources compiled by
oracle/Makefile; the restated oracle port when that library is absent) on the
same workload; single-threaded, as the reference is.
"""
from __future__ import annotations

import argparse
import ctypes as C
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["C1", "C2", "C3", "C4", "C5"], default="C2")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="bounded CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(name: str, rank: int, planner=None):
    """[(request name, jobs, planner config)] for one rank's step."""
    from paper_2105_13336_b200 import configs as CF
    if name in ("C1", "C2"):
        req = CF.requests(name)[0]
        return [(req.name, req.jobs, req.config(CF.INITIAL_PEAK))]
    if name == "C3":  # one replan per arrival: {inception_v3}, {+densenet}, {+vgg16}
        return [(r.name, r.jobs, r.config(CF.INITIAL_PEAK)) for r in CF.requests("C3")]
    if name == "C4":
        return [CF.c4_request()]
    if name == "C4-sample":  # the reference cannot plan C4; its bounded CPU sample
        return [CF.c4_request(1)]
    from paper_2105_13336_b200 import multigpu as MG
    peaks = MG.initial_peaks(planner, [rank % 8]) if planner is not None else None
    if peaks is None:  # CPU arm: the reference's own initial peaks
        from oracle import ref
        peaks = ref.initial_peaks([CF.c5_job(k) for k in range(8 * (rank % 8), 8 * (rank % 8) + 8)])
    return MG.shard_requests(rank % 8, peaks)


def n_accesses(jobs) -> int:
    return sum(len(o["inputs"]) + len(o["outputs"]) for g, _ in jobs for o in g["ops"])


def workload_desc(name: str) -> str:
    return {"C1": "C1 VGG-16 b32, single workload, one build_plan",
            "C2": "C2 ResNet-50 b64, single workload with across-iteration (Opt-phase) swap-ins, one build_plan",
            "C3": "C3 InceptionV3 + DenseNet + VGG-16 arriving in sequence, one replan per arrival (3 build_plans, one launch)",
            "C4": "C4 GPT-2-medium seq-1024 training trace, 70 micro-batches, 990,518 accesses, one build_plan",
            "C5": "C5 shard: 8 concurrent dynamic workloads, 8 arrivals + 7 departures = 15 replans per GPU"}[name]


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
def cpu_reference(reqs, seconds: float, max_plans: int = 10 ** 9):
    """Time the reference scheduler (or the oracle port) on the host: returns
    (events/s, ms per step, steps, kind)."""
    from oracle import ref, tslo
    kind = "reference" if ref.available() else "port"
    ev = sum(n_accesses(j) for _, j, _ in reqs)
    times = []
    t_end = time.perf_counter() + seconds
    while (time.perf_counter() < t_end or not times) and len(times) < max_plans:
        step = 0.0
        for _, jobs, cfg in reqs:
            if kind == "reference":
                step += ref.build_plan(jobs, cfg, repeats=1)[1]["times_ms"][0]
            else:
                step += tslo.build_plan(jobs, cfg)["ms"]
        times.append(step)
    ms = statistics.median(times)
    return ev / (ms / 1e3), ms, len(times), kind


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
    from oracle import ref
    reqs = workload("C5", shard)
    return sum(n_accesses(j) for _, j, _ in reqs), sum(ref.build_plan(j, c, repeats=1)[1]["times_ms"][0]
                                                       for _, j, c in reqs)


def cpu_parallel_shards() -> dict:
    """C5 on the host: N = min(8, cores) processes, shard k in process k, one
    step each; throughput = all events / the slowest shard."""
    import multiprocessing as mp
    n = max(1, min(8, os.cpu_count() or 1))
    with mp.get_context("spawn").Pool(n) as pool:
        res = pool.map(_shard_plan_ms, range(n))
    ev = sum(e for e, _ in res)
    slow = max(ms for _, ms in res)
    return {"processes": n, "value": ev / (slow / 1e3), "unit": UNIT, "slowest_shard_ms": slow,
            "sample": f"shards 0..{n - 1}, one 15-replan step each, one process per shard (reference, -O3)"}


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(name: str):
    p = os.path.join(ROOT, "profiles", f"ncu_traffic_{name}.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("dram_bytes_per_launch")
    return None


def golden_parity(name: str, results) -> str:
    """Cheap in-bench parity: the plans of this run vs the reference fixtures."""
    import hashlib
    if name == "C4":  # digests of the restated oracle (the reference cannot plan C4)
        p = os.path.join(ROOT, "tests", "golden", "c4.json")
        d = json.load(open(p))["cases"].get("M70") if os.path.exists(p) else None
        if d is None:
            return "unchecked (no oracle digest)"
        ok = all(hashlib.sha256(r["plans_json"].encode()).hexdigest() == d["plans_sha256"] for _, r in results)
        return "byte-identical save_plans vs the restated oracle (C4)" if ok else "MISMATCH vs oracle digest (C4)"
    p = os.path.join(ROOT, "tests", "golden", "configs.json")
    if not os.path.exists(p):
        return "unchecked"
    gold = {c["name"]: c for c in json.load(open(p)) if c["ratio"] is None}
    seen = 0
    for n, r in results:
        g = gold.get(n)
        if g is None:
            continue
        if hashlib.sha256(r["plans_json"].encode()).hexdigest() != g["plans_sha256"]:
            return f"MISMATCH on {n}"
        seen += 1
    return f"byte-identical save_plans vs reference on {seen} plan(s)" if seen else "unchecked"


# ---------------------------------------------------------------------------
def run_reference(a, rank, world):
    if rank != 0:
        return
    # C4: the reference cannot plan 1 M accesses; its arm
    # runs the bounded 1-micro-batch sample of the same generator, 1 step
    sample = a.workload == "C4"
    reqs = workload("C4-sample" if sample else a.workload, 0)
    ev = sum(n_accesses(j) for _, j, _ in reqs)
    from oracle import ref, tslo
    kind = "reference" if ref.available() else "port"
    for _ in range(0 if sample else a.warmup):
        cpu_reference(reqs, 0.0, 1)
    times = []
    t0 = time.perf_counter()
    for _ in range(a.steps):
        times.append(cpu_reference(reqs, 0.0, 1)[1])
        if time.perf_counter() - t0 > 150:  # keep the reference arm within minutes
            break
    ms = statistics.mean(times)
    value = ev / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": len(times),
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "impl": "reference",
            "data": "synthetic traces from the reference generator (workload.cpp), latency seed 13",
            "config": {"workload": workload_desc(a.workload), "requests": len(reqs), "accesses_per_step": ev},
            "plan_gen_ms": ms,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": kind, "host": host_cpu(),
                             "threads_note": "the reference has no threads: one build_plan uses one core",
                             "sample": f"{len(times)} x build_plan of {'the C4 1-micro-batch sample (16,445 accesses)' if sample else a.workload}, single thread "
                                       f"({'oracle/_ref: reference sources compiled -O3' if kind == 'reference' else 'restated oracle port'})"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if a.workload == "C5" and kind == "reference":
        line["cpu_baseline"]["parallel_shards"] = cpu_parallel_shards()
    print(json.dumps(line), flush=True)


def run_ours(a, rank, world, local):
    import torch
    from paper_2105_13336_b200 import abi
    from paper_2105_13336_b200.planner import Planner
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
    reqs = workload(a.workload, rank, planner)
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
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    wall0 = time.perf_counter()
    for e0, e1 in evs:
        flush.zero_()  # on the same stream, outside the event pair
        e0.record(stream)
        prep.launch_async(stream.cuda_stream)
        e1.record(stream)
    torch.cuda.synchronize()
    wall_dev = time.perf_counter() - wall0
    clocks = sampler.stop()
    dev_ms = statistics.mean(e0.elapsed_time(e1) for e0, e1 in evs)
    # ---- e2e region: host buffers -> C-ABI -> host results ----
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / a.steps
    if dist:
        t = torch.tensor([dev_ms, e2e_ms], device=f"cuda:{local}" if backend == "nccl" else "cpu",
                         dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, e2e_ms = t.tolist()
    outs = prep.collect(with_views=False)
    prep.close()
    alg_bytes = sum(o["stats"]["algorithmic_bytes"] for o in outs)
    parity = golden_parity(a.workload, [(n, o) for (n, _, _), o in zip(reqs, outs)])
    # gather the serialised plans on rank 0 (the only collective, C5)
    gather_ms = None
    if a.workload == "C5":
        from paper_2105_13336_b200 import multigpu as MG
        g0 = time.perf_counter()
        MG.gather_plans(outs, [n for n, _, _ in reqs], rank, world)
        gather_ms = (time.perf_counter() - g0) * 1e3
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    from paper_2105_13336_b200 import configs as CF
    init_peak = (CF.C4_INITIAL_PEAK[CF.C4_MICRO_BATCHES] if a.workload == "C4" else
                 sum(CF.INITIAL_PEAK.get(g["job_id"], 0) for g, _ in groups[-1]) if a.workload not in ("C5",) else None)
    saved = (init_peak - outs[-1]["final_merged_peak"]) if init_peak else None  # the full set (C3: last arrival)
    peak, how = hbm_peak()
    achieved = alg_bytes / (dev_ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": world * ev / (dev_ms / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": dev_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic traces from the reference generator (workload.cpp), latency seed 13",
        "config": {"workload": workload_desc(a.workload), "requests_per_gpu": len(reqs),
                   "accesses_per_gpu_step": ev, "pcie_bandwidth": CF.BW, "transfer_setup": CF.SETUP,
                   "memory_budget": "70% of the set's initial peak", "l2": "flushed between steps (256 MB write)",
                   "parallelism": f"{world} GPU(s), one CTA per build_plan"},
        "plan_gen_ms": dev_ms, "peak_bytes_saved": saved, "parity": parity,
        "e2e": {"value": world * ev / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(stats.h2d_bytes), "d2h_bytes_per_step": int(stats.d2h_bytes),
                "host_prep_ms": stats.prep_ms, "launches_per_step": 1},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic(a.workload), "peak_source": how,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "note": "latency-bound single-CTA kernel; SURVEY.md 8(d) byte formula"},
        "clocks": clocks, "gpu_launches": a.steps, "timed_wall_s": wall_dev,
    }
    if gather_ms is not None:
        line["plan_gather_ms"] = gather_ms
    if world == 1 and not a.no_cpu_baseline:
        c4 = a.workload == "C4"
        rate, ms, n, kind = cpu_reference(workload("C4-sample", 0) if c4 else reqs, a.cpu_seconds, 1 if c4 else 10 ** 9)
        what = "C4 1-micro-batch sample (16,445 accesses; the reference cannot plan full C4)" if c4 else f"{a.workload} step"
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": 1, "kind": kind, "ms_per_step": ms,
                                "host": host_cpu(),
                                "sample": f"{n} x {what} on 1 host thread (~{a.cpu_seconds:.0f} s), "
                                          f"{'reference sources compiled -O3 (oracle/_ref)' if kind == 'reference' else 'restated oracle port'}"}
        if a.workload == "C5" and kind == "reference":
            line["cpu_baseline"]["parallel_shards"] = cpu_parallel_shards()
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
