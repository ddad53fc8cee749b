"""The replan lifecycle around the device planner: memsched::Orchestrator
(orchestrator.hpp:30-60, orchestrator.cpp:89-159) over the C-ABI session
(tsl_session_*, csrc/tsl_session.cpp), and run_scenario (scenario.cpp:223-262)
driving the tick-level executor model (sim.py) with it.

    orch = Orchestrator(planner, config, graphs)
    orch.plan_with_latencies({job: {op: ticks}})    # -> BuildResult dict (versions bumped)
    orch.plan_cold_start(predictor)                  # latencies from a LatencyPredictor
    orch.replan_if_needed({job: {op: observed}})     # -> None or {job: plan}
    orch.add_job(graph, latencies) / orch.remove_job(job_id)   # arrival / departure
    orch.rebuild()                                   # replan the active set now

Every rebuild is one device launch over the active set; `rebuild_ms` lists
their wall times (validation, H2D, kernel, D2H and result assembly).
"""
from __future__ import annotations

import ctypes as C
import json
from typing import Dict, List, Optional, Sequence

from . import abi
from .planner import Planner, PlannerError, ValidationError, _collect


def _bind(L):
    if getattr(L, "_session_bound", False):
        return L
    vp = C.c_void_p
    L.tsl_session_create.argtypes = [vp, C.POINTER(abi.TslConfig), C.POINTER(vp)]
    L.tsl_session_destroy.argtypes = [vp]
    L.tsl_session_add_job.argtypes = [vp, C.POINTER(abi.TslJobDesc)]
    L.tsl_session_remove_job.argtypes = [vp, C.c_char_p]
    L.tsl_session_set_latencies.argtypes = [vp, C.c_char_p, C.POINTER(C.c_int64)]
    L.tsl_session_rebuild.argtypes = [vp, C.POINTER(vp)]
    L.tsl_session_replan_if_needed.argtypes = [vp, C.c_int32, C.POINTER(C.c_char_p), C.POINTER(C.POINTER(C.c_int64)),
                                               C.POINTER(vp)]
    L.tsl_session_replan_count.argtypes = [vp]
    L.tsl_session_rebuild_times.argtypes = [vp, C.POINTER(C.POINTER(C.c_double))]
    L.tsl_session_n_jobs.argtypes = [vp]
    L.tsl_session_latencies.argtypes = [vp, C.c_char_p, C.POINTER(C.c_int64)]
    L._session_bound = True
    return L


class Orchestrator:
    """memsched::Orchestrator on the B200 planner (plus arrival/departure)."""

    def __init__(self, planner: Planner, config: dict, graphs: Sequence[dict] = ()):
        self.planner = planner
        self.L = _bind(planner.lib)
        self._cfg = abi.make_config(**config)
        self._h = C.c_void_p()
        rc = self.L.tsl_session_create(planner._ctx, C.byref(self._cfg), C.byref(self._h))
        if rc:
            self._raise(rc)
        self._jobs: Dict[str, abi.JobDesc] = {}
        self._order: List[str] = []
        for g in graphs:
            self.add_job(g)

    def _raise(self, rc):
        msg = self.L.tsl_last_error().decode()
        raise (ValidationError if rc == abi.TSL_ERR_VALIDATION else PlannerError)(rc, msg)

    def close(self):
        if self._h:
            self.L.tsl_session_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- the active set ----------------------------------------------------
    def add_job(self, graph: dict, latencies: Optional[dict] = None):
        """A job arrives (latencies: its current estimates, or None until set)."""
        descs, arr = abi.pack_jobs([(graph, latencies if latencies is not None else {})])
        if latencies is None:
            arr[0].op_latencies = C.POINTER(C.c_int64)()
        rc = self.L.tsl_session_add_job(self._h, arr)
        if rc:
            self._raise(rc)
        self._jobs[graph["job_id"]] = descs[0]
        self._order.append(graph["job_id"])

    def remove_job(self, job_id: str):
        """A job departs; its plan version counter is kept."""
        rc = self.L.tsl_session_remove_job(self._h, job_id.encode())
        if rc:
            self._raise(rc)
        self._jobs.pop(job_id, None)
        self._order.remove(job_id)

    def set_latencies(self, job_id: str, latencies: dict):
        g = self._jobs[job_id].graph
        lat = (C.c_int64 * max(1, len(g["ops"])))(*[int(latencies[o["id"]]) for o in g["ops"]])
        rc = self.L.tsl_session_set_latencies(self._h, job_id.encode(), lat)
        if rc:
            self._raise(rc)

    def latencies(self, job_id: str) -> dict:
        g = self._jobs[job_id].graph
        buf = (C.c_int64 * max(1, len(g["ops"])))()
        rc = self.L.tsl_session_latencies(self._h, job_id.encode(), buf)
        if rc:
            self._raise(rc)
        return {o["id"]: int(buf[k]) for k, o in enumerate(g["ops"])}

    # -- Orchestrator ------------------------------------------------------
    def _result(self, res) -> dict:
        try:
            return _collect(self.L, res, list(self._jobs.values()), True)
        finally:
            self.L.tsl_result_destroy(res)

    def rebuild(self) -> dict:
        res = C.c_void_p()
        rc = self.L.tsl_session_rebuild(self._h, C.byref(res))
        if rc:
            self._raise(rc)
        return self._result(res)

    def plan_with_latencies(self, latencies: Dict[str, dict]) -> dict:
        """orchestrator.cpp:112-116: the table replaces every estimate."""
        for jid in self._order:
            if jid not in latencies:
                raise PlannerError(abi.TSL_ERR_VALIDATION, "map::at")
            self.set_latencies(jid, latencies[jid])
        return self.rebuild()

    def plan_cold_start(self, predictor) -> dict:
        """orchestrator.cpp:118-124: latencies from the fitted predictor at the
        configured cold-start GPU usage."""
        usage = self._cfg.cold_start_gpu_usage
        for jid in self._order:
            self.set_latencies(jid, predictor.predict_latencies(self._jobs[jid].graph, usage))
        return self.rebuild()

    def replan_if_needed(self, observed: Dict[str, dict]) -> Optional[dict]:
        """orchestrator.cpp:126-159 -> {job: plan dict} or None."""
        keep, ids, ptrs = [], [], []
        for jid, ops in observed.items():
            if jid not in self._jobs:
                continue
            g = self._jobs[jid].graph
            arr = (C.c_int64 * max(1, len(g["ops"])))(*[int(ops.get(o["id"], -1)) for o in g["ops"]])
            keep.append(arr)
            ids.append(jid.encode())
            ptrs.append(C.cast(arr, C.POINTER(C.c_int64)))
        idarr = (C.c_char_p * max(1, len(ids)))(*ids)
        parr = (C.POINTER(C.c_int64) * max(1, len(ptrs)))(*ptrs)
        res = C.c_void_p()
        rc = self.L.tsl_session_replan_if_needed(self._h, len(ids), idarr, parr, C.byref(res))
        if rc:
            self._raise(rc)
        if not res:
            return None
        out = self._result(res)
        return {jid: j["plan"] for jid, j in out["jobs"].items()}

    @property
    def replan_count(self) -> int:
        return int(self.L.tsl_session_replan_count(self._h))

    @property
    def rebuild_ms(self) -> List[float]:
        p = C.POINTER(C.c_double)()
        n = self.L.tsl_session_rebuild_times(self._h, C.byref(p))
        return [p[i] for i in range(n)]


# ---------------------------------------------------------------------------
def mode_stats(mode: str, trace: dict, replans: int) -> dict:
    """stats_from (scenario.cpp:152-168) -> the ModeStats fields."""
    times = {j["job_id"]: j["iteration_times"] for j in trace["jobs"] if j["iteration_times"]}
    total = sum(sum(t) / len(t) for t in times.values())
    return {"mode": mode, "peak": trace["peak"], "total_mean_iteration_time": total,
            "passive_swap_count": trace["passive_swap_count"], "blocked_ticks": trace["blocked_ticks"],
            "replan_count": replans, "iteration_times": dict(sorted(times.items()))}


def run_scenario(scn: dict, planner: Planner, modes=("vanilla", "scheduled", "passive")) -> dict:
    """run_scenario (scenario.cpp:223-262) over a cli.load_scenario document:
    {"stats": {mode: ModeStats fields}, "traces": {mode: trace}, "plans":
    {job: plan}, "replan_count", "diagnostic", "rebuild_ms"}."""
    from . import sim
    from . import workload as W
    for m in modes:
        if m not in ("vanilla", "scheduled", "passive"):
            raise ValidationError(abi.TSL_ERR_VALIDATION, "unknown mode: " + m)
    cfg = scn["config"]
    seed = scn.get("seed", 0)
    jobs = [(g, W.true_latency_table(g, seed), t) for g, t in zip(scn["jobs"], scn["launch_ticks"])]
    kw = dict(iterations=scn.get("iterations", 3), memory_budget=cfg["memory_budget"],
              pcie_bandwidth=cfg["pcie_bandwidth"], transfer_setup=cfg["transfer_setup"],
              slowdown=scn.get("gpu_slowdown_curve") or None, lib_path=planner.lib._name)
    out = {"stats": {}, "traces": {}, "plans": {}, "replan_count": 0, "diagnostic": "", "rebuild_ms": []}
    base = sim.baseline_plans(jobs, planner.lib._name) if ("vanilla" in modes or "passive" in modes) else {}
    for mode in ("vanilla", "passive"):
        if mode in modes:
            t = sim.simulate(jobs, base, mode=mode, **kw)
            out["traces"][mode], out["stats"][mode] = t, mode_stats(mode, t, 0)
    if "scheduled" in modes:
        orch = Orchestrator(planner, cfg, scn["jobs"])
        if scn.get("latency_file"):
            with open(scn["latency_file"]) as f:
                table = json.load(f)
            build = orch.plan_with_latencies({j: {o: int(t) for o, t in ops.items()} for j, ops in table.items()})
        elif scn.get("predictor_file"):
            from .latency import LatencyPredictor
            with open(scn["predictor_file"]) as f:
                build = orch.plan_cold_start(LatencyPredictor.from_json(f.read()))
        else:
            raise ValidationError(abi.TSL_ERR_VALIDATION, "scheduled mode needs a latency source: fit a predictor "
                                  "(predictor_file) or supply a latency table (latency_file)")
        out["plans"] = {j: v["plan"] for j, v in build["jobs"].items()}
        out["diagnostic"] = build["diagnostic"]

        def controller(job, iteration, observed):  # ReplanController (scenario.cpp:113-126)
            return orch.replan_if_needed({job: observed})

        t = sim.simulate(jobs, out["plans"], mode="scheduled", controller=controller, **kw)
        out["replan_count"] = orch.replan_count
        out["rebuild_ms"] = orch.rebuild_ms
        out["traces"]["scheduled"], out["stats"]["scheduled"] = t, mode_stats("scheduled", t, orch.replan_count)
    return out
