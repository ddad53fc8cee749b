"""Tick-level executor model over the C-ABI (tsl_simulate, csrc/tsl_sim.cpp):
the reference's memsched::simulate (simulator.hpp:84-87) in vanilla /
scheduled / passive mode, its SimController hook, and compute_metrics
(simulator.cpp:598-632).

    trace = simulate([(graph, true_latencies, launch_tick)], plans, mode="scheduled",
                     iterations=3, pcie_bandwidth=..., transfer_setup=..., memory_budget=...,
                     controller=None)

`plans` is a save_plans document ({job_id: plan}); jobs without an entry run
an empty plan. `controller(job_id, iteration, observed)` (observed: {op:
ticks}) may return {job_id: plan} to install at those jobs' next iteration
boundary. The trace dict carries the SimulationTrace fields and "csv"
(SimulationTrace::to_csv).
"""
from __future__ import annotations

import ctypes as C
import json
import math
from typing import Callable, Dict, Optional, Sequence

from . import abi
from .planner import PlannerError, ValidationError, load_library

MODES = {"vanilla": 0, "scheduled": 1, "passive": 2}


class TslSimConfig(C.Structure):
    _fields_ = [("mode", C.c_int32), ("iterations", C.c_int32), ("ticks_per_iteration_limit", C.c_int64),
                ("memory_budget", C.c_int64), ("pcie_bandwidth", C.c_int64), ("transfer_setup", C.c_int64),
                ("n_slowdown", C.c_int32), ("slowdown_jobs", C.POINTER(C.c_int32)),
                ("slowdown_mult", C.POINTER(C.c_double))]


CTRL = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_int64))


def _lib(path: Optional[str] = None):
    L = load_library(path)
    if not getattr(L, "_sim_bound", False):
        vp = C.c_void_p
        L.tsl_simulate.argtypes = [C.POINTER(abi.TslJobDesc), C.POINTER(C.c_int64), C.c_int32,
                                   C.POINTER(abi.TslPlanDesc), C.POINTER(TslSimConfig), CTRL, vp, C.POINTER(vp)]
        L.tsl_sim_set_plan.argtypes = [vp, C.c_int32, C.POINTER(abi.TslPlanDesc)]
        L.tsl_sim_peak.argtypes = [vp]
        L.tsl_sim_peak.restype = C.c_int64
        L.tsl_sim_trace_json.argtypes = [vp]
        L.tsl_sim_trace_json.restype = vp
        L.tsl_sim_trace_csv.argtypes = [vp]
        L.tsl_sim_trace_csv.restype = vp
        L.tsl_sim_destroy.argtypes = [vp]
        L.tsl_base_release_flags.argtypes = [C.POINTER(abi.TslJobDesc), C.POINTER(C.c_int64), C.c_int32,
                                             C.POINTER(C.c_int32)]
        L._sim_bound = True
    return L


def _raise(L, rc):
    msg = L.tsl_last_error().decode()
    raise (ValidationError if rc == abi.TSL_ERR_VALIDATION else PlannerError)(rc, msg)


def _take(L, p) -> str:
    s = C.cast(p, C.c_char_p).value.decode()
    L.tsl_free(p)
    return s


def base_release_flags(graph: dict, lib_path: Optional[str] = None) -> list:
    """activity_analysis' flags of one job (the vanilla/passive baseline plan)."""
    L = _lib(lib_path)
    descs, arr = abi.pack_jobs([(graph, {o["id"]: 1 for o in graph["ops"]})])
    n = C.c_int32()
    rc = L.tsl_base_release_flags(arr, None, 0, C.byref(n))
    if rc:
        _raise(L, rc)
    buf = (C.c_int64 * max(1, n.value))()
    rc = L.tsl_base_release_flags(arr, buf, n.value, C.byref(n))
    if rc:
        _raise(L, rc)
    return list(buf[: n.value])


def baseline_plans(jobs: Sequence, lib_path: Optional[str] = None) -> dict:
    """baseline_plans (scenario.cpp:180-194): release at last use, no events."""
    return {g["job_id"]: {"version": 0, "swap_events": [], "recompute_events": [],
                          "release_flags": base_release_flags(g, lib_path)} for g, _, _ in jobs}


def simulate(jobs: Sequence, plans: Optional[dict] = None, mode: str = "vanilla", iterations: int = 1,
             memory_budget: int = 0, pcie_bandwidth: int = 1, transfer_setup: int = 0,
             slowdown: Optional[Dict[int, float]] = None, ticks_per_iteration_limit: int = 10_000_000,
             controller: Optional[Callable] = None, lib_path: Optional[str] = None) -> dict:
    L = _lib(lib_path)
    plans = plans or {}
    descs, arr = abi.pack_jobs([(g, lat) for g, lat, _ in jobs])
    launch = (C.c_int64 * max(1, len(jobs)))(*[int(t) for _, _, t in jobs])
    by_id = {d.graph["job_id"]: d for d in descs}
    order = [g["job_id"] for g, _, _ in jobs]
    pds = [abi.PlanDesc(plans.get(j, {}), by_id[j]) for j in order]
    parr = (abi.TslPlanDesc * max(1, len(pds)))(*[p.desc for p in pds])
    sl = sorted((slowdown or {}).items())
    sj = (C.c_int32 * max(1, len(sl)))(*[int(k) for k, _ in sl])
    sm = (C.c_double * max(1, len(sl)))(*[float(v) for _, v in sl])
    cfg = TslSimConfig(MODES[mode], int(iterations), int(ticks_per_iteration_limit), int(memory_budget),
                       int(pcie_bandwidth), int(transfer_setup), len(sl), sj, sm)
    keep = []
    err = []

    def _cb(_user, sim, job, iteration, observed):
        try:
            g = jobs[job][0]
            obs = {o["id"]: observed[k] for k, o in enumerate(g["ops"]) if observed[k] >= 0}
            new = controller(g["job_id"], iteration, obs)
            for jid, plan in (new or {}).items():
                if jid not in by_id:
                    continue
                pd = abi.PlanDesc(plan, by_id[jid])
                keep.append(pd)
                rc = L.tsl_sim_set_plan(sim, order.index(jid), C.byref(pd.desc))
                if rc:
                    return rc
            return 0
        except Exception as e:  # surfaces after the run
            err.append(e)
            return abi.TSL_ERR_INTERNAL

    cb = CTRL(_cb) if controller else CTRL()
    out = C.c_void_p()
    rc = L.tsl_simulate(arr, launch, len(jobs), parr, C.byref(cfg), cb, None, C.byref(out))
    if err:
        raise err[0]
    if rc:
        _raise(L, rc)
    try:
        trace = json.loads(_take(L, L.tsl_sim_trace_json(out)))
        trace["csv"] = _take(L, L.tsl_sim_trace_csv(out))
    finally:
        L.tsl_sim_destroy(out)
    return trace


def compute_metrics(vanilla: dict, experimental: dict) -> dict:
    """compute_metrics (simulator.cpp:598-632): MSR, EOR, CBR (inf when EOR == 0)."""
    def jobs_of(t):
        return {j["job_id"] for j in t["jobs"] if j["iteration_times"]}

    if jobs_of(vanilla) != jobs_of(experimental):
        raise ValidationError(abi.TSL_ERR_VALIDATION, "traces cover different job sets")

    def time_cost(t):
        return sum(sum(j["iteration_times"]) / len(j["iteration_times"]) for j in t["jobs"] if j["iteration_times"])

    vmp, emp = float(vanilla["peak"]), float(experimental["peak"])
    vtc, etc = time_cost(vanilla), time_cost(experimental)
    if vmp <= 0:
        raise ValidationError(abi.TSL_ERR_VALIDATION, "vanilla peak must be positive")
    if vtc <= 0:
        raise ValidationError(abi.TSL_ERR_VALIDATION, "vanilla time cost must be positive")
    msr = (vmp - emp) / vmp
    eor = (etc - vtc) / vtc
    return {"msr": msr, "eor": eor, "cbr": math.inf if eor == 0.0 else msr / eor}
