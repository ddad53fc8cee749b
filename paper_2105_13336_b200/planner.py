"""Python face of the B200 plan generator (ctypes over include/tensile_b200.h).

Mirrors the reference's entry points for the hot path:
  Planner.build_plan(jobs, config)    memsched::build_plan   (orchestrator.hpp:26-28)
  Planner.build_plan_groups(groups)   independent build_plan calls, one CTA each
  Planner.analyze_job(g, lat, plan)   memsched::analyze_job  (peak.hpp:77-78)
Results carry the reference's own serialisations (save_plans text,
PeakReport::to_json text) so callers and tests compare bytes.

Errors raise ValidationError (the reference's memsched::ValidationError) or
PlannerError. The library must be the in-tree CUDA build
(paper_2105_13336_b200/libtensile_b200.so); there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import time
from typing import Dict, List, Optional, Sequence

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtensile_b200.so")


class PlannerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class ValidationError(PlannerError):
    """memsched::ValidationError (types.hpp:41-44)."""


_libs: Dict[str, C.CDLL] = {}


def load_library(path: Optional[str] = None) -> C.CDLL:
    path = path or LIB_PATH
    if path in _libs:
        return _libs[path]
    if not os.path.exists(path):
        raise PlannerError(abi.TSL_ERR_CUDA, f"CUDA planner library not built: {path} "
                           "(run python -c 'import __graft_entry__ as g; g.build()')")
    L = C.CDLL(path)
    vp = C.c_void_p
    L.tsl_last_error.restype = C.c_char_p
    L.tsl_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.tsl_destroy.argtypes = [vp]
    L.tsl_build_plan.argtypes = [vp, C.POINTER(abi.TslJobDesc), C.c_int32, C.POINTER(abi.TslConfig), C.POINTER(vp)]
    L.tsl_build_plan_groups.argtypes = [vp, C.POINTER(abi.TslJobDesc), C.POINTER(C.c_int32), C.c_int32,
                                        C.POINTER(abi.TslConfig), C.c_int32, C.POINTER(vp)]
    L.tsl_plan_prepare.argtypes = [vp, C.POINTER(abi.TslJobDesc), C.POINTER(C.c_int32), C.c_int32,
                                   C.POINTER(abi.TslConfig), C.c_int32, C.POINTER(vp)]
    L.tsl_plan_run.argtypes = [vp, C.c_int32, C.POINTER(C.c_double)]
    L.tsl_plan_launch_async.argtypes = [vp, vp]
    L.tsl_plan_collect.argtypes = [vp, C.POINTER(vp)]
    L.tsl_plan_destroy.argtypes = [vp]
    L.tsl_analyze_job.argtypes = [vp, C.POINTER(abi.TslJobDesc), C.POINTER(abi.TslPlanDesc), C.POINTER(vp)]
    L.tsl_result_n_jobs.argtypes = [vp]
    L.tsl_result_job.argtypes = [vp, C.c_int32, C.POINTER(abi.TslJobView)]
    L.tsl_result_history.argtypes = [vp, C.POINTER(C.POINTER(C.c_int64))]
    L.tsl_result_final_merged_peak.argtypes = [vp]
    L.tsl_result_final_merged_peak.restype = C.c_int64
    L.tsl_result_within_budget.argtypes = [vp]
    L.tsl_result_diagnostic.argtypes = [vp]
    L.tsl_result_diagnostic.restype = C.c_char_p
    L.tsl_result_stats.argtypes = [vp, C.POINTER(abi.TslStats)]
    L.tsl_result_save_plans.argtypes = [vp]
    L.tsl_result_save_plans.restype = vp
    L.tsl_result_report_json.argtypes = [vp, C.c_int32]
    L.tsl_result_report_json.restype = vp
    L.tsl_result_destroy.argtypes = [vp]
    L.tsl_free.argtypes = [vp]
    L.tsl_execute_plan.argtypes = [vp, vp, C.c_int32, C.POINTER(abi.TslConfig), C.POINTER(abi.TslExecConfig),
                                   C.POINTER(abi.TslExecReport)]
    L.tsl_execute_plans.argtypes = [vp, vp, C.POINTER(abi.TslConfig), C.POINTER(abi.TslExecConfig),
                                    C.POINTER(abi.TslExecReport), C.POINTER(abi.TslExecReport)]
    _libs[path] = L
    return L


def _raise(L, rc: int):
    msg = L.tsl_last_error().decode()
    if rc == abi.TSL_ERR_VALIDATION:
        raise ValidationError(rc, msg)
    raise PlannerError(rc, msg)


def _take(L, p) -> str:
    s = C.cast(p, C.c_char_p).value.decode()
    L.tsl_free(p)
    return s


def _collect(L, res, descs, with_views: bool = True) -> dict:
    out: dict = {"jobs": {}, "reports_json": {}}
    if with_views:
        for i in range(L.tsl_result_n_jobs(res)):
            v = abi.TslJobView()
            rc = L.tsl_result_job(res, i, C.byref(v))
            if rc:
                _raise(L, rc)
            jid = v.job_id.decode()
            job = next(d for d in descs if d.graph["job_id"] == jid)
            out["jobs"][jid] = abi.view_to_dict(v, job)
            out["reports_json"][jid] = _take(L, L.tsl_result_report_json(res, i))
    h = C.POINTER(C.c_int64)()
    n = L.tsl_result_history(res, C.byref(h))
    out["merged_peak_history"] = [h[i] for i in range(n)]
    out["final_merged_peak"] = L.tsl_result_final_merged_peak(res)
    out["within_budget"] = bool(L.tsl_result_within_budget(res))
    out["diagnostic"] = L.tsl_result_diagnostic(res).decode()
    out["plans_json"] = _take(L, L.tsl_result_save_plans(res))
    st = abi.TslStats()
    L.tsl_result_stats(res, C.byref(st))
    out["stats"] = {f: getattr(st, f) for f, _ in abi.TslStats._fields_}
    return out


class PreparedPlan:
    """Inputs resident on the device; run() launches only the kernel."""

    def __init__(self, planner: "Planner", handle, descs, n_groups: int):
        self._p = planner
        self._h = handle
        self._descs = descs
        self.n_groups = n_groups

    def run(self, repeats: int = 1) -> float:
        ms = C.c_double()
        rc = self._p.lib.tsl_plan_run(self._h, repeats, C.byref(ms))
        if rc:
            _raise(self._p.lib, rc)
        return ms.value

    def launch_async(self, stream_handle: int = 0):
        """One launch on a cudaStream_t handle (torch.cuda.Stream().cuda_stream);
        0 means the planner context's own stream."""
        rc = self._p.lib.tsl_plan_launch_async(self._h, C.c_void_p(stream_handle or None))
        if rc:
            _raise(self._p.lib, rc)

    def collect(self, with_views: bool = True) -> List[dict]:
        L = self._p.lib
        arr = (C.c_void_p * self.n_groups)()
        rc = L.tsl_plan_collect(self._h, arr)
        if rc:
            _raise(L, rc)
        outs = []
        for g in range(self.n_groups):
            try:
                outs.append(_collect(L, arr[g], self._descs, with_views))
            finally:
                L.tsl_result_destroy(arr[g])
        return outs

    def close(self):
        if self._h:
            self._p.lib.tsl_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Planner:
    """One CUDA device context (streams, device/pinned buffers reused across calls)."""

    def __init__(self, device: int = 0, lib_path: Optional[str] = None):
        self.lib = load_library(lib_path)
        self._ctx = C.c_void_p()
        rc = self.lib.tsl_create(device, C.byref(self._ctx))
        if rc:
            _raise(self.lib, rc)

    def close(self):
        if self._ctx:
            self.lib.tsl_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def build_plan(self, jobs: Sequence, config: dict, with_views: bool = True) -> dict:
        """build_plan over [(graph, latencies)] -> dict (plans_json = save_plans text)."""
        descs, arr = abi.pack_jobs(jobs)
        cfg = abi.make_config(**config)
        res = C.c_void_p()
        t0 = time.perf_counter()
        rc = self.lib.tsl_build_plan(self._ctx, arr, len(descs), C.byref(cfg), C.byref(res))
        t1 = time.perf_counter()
        if rc:
            _raise(self.lib, rc)
        try:
            out = _collect(self.lib, res, descs, with_views)
        finally:
            self.lib.tsl_result_destroy(res)
        out["ms"] = (t1 - t0) * 1e3
        return out

    @staticmethod
    def _configs(config, n_groups: int):
        """One shared config dict, or a list with one config per group."""
        cfgs = list(config) if isinstance(config, (list, tuple)) else [config]
        if len(cfgs) not in (1, n_groups):
            raise ValueError("need one config or one per group")
        keep = [abi.make_config(**c) for c in cfgs]  # owns each config's ratio-map arrays
        arr = (abi.TslConfig * len(cfgs))(*keep)
        return arr, len(cfgs), keep

    def _pack_groups(self, groups: Sequence[Sequence]):
        flat = [j for grp in groups for j in grp]
        descs, arr = abi.pack_jobs(flat)
        offs = (C.c_int32 * (len(groups) + 1))()
        k = 0
        for i, grp in enumerate(groups):
            offs[i] = k
            k += len(grp)
        offs[len(groups)] = k
        return descs, arr, offs

    def build_plan_groups(self, groups: Sequence[Sequence], config, with_views: bool = True) -> List[dict]:
        """Independent build_plan calls (one per group) in ONE kernel launch.
        `config` is one dict shared by all groups or a list, one per group."""
        cfgs, ncfg, keep = self._configs(config, len(groups))
        descs, arr, offs = self._pack_groups(groups)
        res = (C.c_void_p * len(groups))()
        rc = self.lib.tsl_build_plan_groups(self._ctx, arr, offs, len(groups), cfgs, ncfg, res)
        if rc:
            _raise(self.lib, rc)
        outs = []
        for g in range(len(groups)):
            try:
                outs.append(_collect(self.lib, res[g], descs, with_views))
            finally:
                self.lib.tsl_result_destroy(res[g])
        return outs

    def prepare(self, groups: Sequence[Sequence], config) -> PreparedPlan:
        cfgs, ncfg, keep = self._configs(config, len(groups))
        descs, arr, offs = self._pack_groups(groups)
        h = C.c_void_p()
        rc = self.lib.tsl_plan_prepare(self._ctx, arr, offs, len(groups), cfgs, ncfg, C.byref(h))
        if rc:
            _raise(self.lib, rc)
        return PreparedPlan(self, h, descs, len(groups))

    def build_and_execute(self, jobs: Sequence, config: dict, tick_ns: int = 1000, iterations: int = 3,
                          bytes_per_unit: int = 16, mempool: bool = False) -> dict:
        """build_plan, then replay every job's plan on the device (plan
        executor): {"plan": build_plan dict, "exec": {job_id: report dict}}."""
        descs, arr = abi.pack_jobs(jobs)
        cfg = abi.make_config(**config)
        res = C.c_void_p()
        rc = self.lib.tsl_build_plan(self._ctx, arr, len(descs), C.byref(cfg), C.byref(res))
        if rc:
            _raise(self.lib, rc)
        try:
            out = {"plan": _collect(self.lib, res, descs), "exec": {}}
            ex = abi.TslExecConfig(tick_ns, iterations, bytes_per_unit, 0, 1 if mempool else 0)
            for i in range(self.lib.tsl_result_n_jobs(res)):
                rep = abi.TslExecReport()
                rc = self.lib.tsl_execute_plan(self._ctx, res, i, C.byref(cfg), C.byref(ex), C.byref(rep))
                if rc:
                    _raise(self.lib, rc)
                v = abi.TslJobView()
                self.lib.tsl_result_job(res, i, C.byref(v))
                d = {f: getattr(rep, f) for f, _ in abi.TslExecReport._fields_}
                d["iteration_ms"] = list(rep.iteration_ms)[: rep.iterations]
                out["exec"][v.job_id.decode()] = d
        finally:
            self.lib.tsl_result_destroy(res)
        return out

    def build_and_execute_all(self, jobs: Sequence, config: dict, tick_ns: int = 1000, iterations: int = 3,
                              bytes_per_unit: int = 16, vanilla: bool = False, mempool: bool = False) -> dict:
        """build_plan, then replay ALL jobs' plans together on the device (one
        compute stream per job, one FIFO copy stream, one allocator):
        {"plan": build_plan dict, "exec": {job_id: report}, "merged": report}."""
        descs, arr = abi.pack_jobs(jobs)
        cfg = abi.make_config(**config)
        res = C.c_void_p()
        rc = self.lib.tsl_build_plan(self._ctx, arr, len(descs), C.byref(cfg), C.byref(res))
        if rc:
            _raise(self.lib, rc)

        def as_dict(rep):
            d = {f: getattr(rep, f) for f, _ in abi.TslExecReport._fields_}
            d["iteration_ms"] = list(rep.iteration_ms)[: rep.iterations]
            return d

        try:
            out = {"plan": _collect(self.lib, res, descs), "exec": {}}
            ex = abi.TslExecConfig(tick_ns, iterations, bytes_per_unit, 1 if vanilla else 0, 1 if mempool else 0)
            n = self.lib.tsl_result_n_jobs(res)
            per = (abi.TslExecReport * max(1, n))()
            merged = abi.TslExecReport()
            rc = self.lib.tsl_execute_plans(self._ctx, res, C.byref(cfg), C.byref(ex), per, C.byref(merged))
            if rc:
                _raise(self.lib, rc)
            for i in range(n):
                v = abi.TslJobView()
                self.lib.tsl_result_job(res, i, C.byref(v))
                out["exec"][v.job_id.decode()] = as_dict(per[i])
            out["merged"] = as_dict(merged)
        finally:
            self.lib.tsl_result_destroy(res)
        return out

    def analyze_job(self, graph: dict, latencies: dict, plan: dict) -> dict:
        jd = abi.JobDesc(graph, latencies)
        pd = abi.PlanDesc(plan, jd)
        res = C.c_void_p()
        rc = self.lib.tsl_analyze_job(self._ctx, C.byref(jd.desc), C.byref(pd.desc), C.byref(res))
        if rc:
            _raise(self.lib, rc)
        try:
            out = _collect(self.lib, res, [jd])
        finally:
            self.lib.tsl_result_destroy(res)
        jid = graph["job_id"]
        return {"report": out["jobs"][jid]["report"], "report_json": out["reports_json"][jid]}


def replay_metrics(vanilla: dict, scheduled: dict) -> dict:
    """compute_metrics (simulator.cpp:598-632) on two device replays of the
    same build (build_and_execute_all with vanilla=True / False): memory
    saving ratio MSR = (vanilla peak - scheduled peak) / vanilla peak, extra
    overhead ratio EOR = (scheduled time - vanilla time) / vanilla time, where
    a replay's time is the sum over jobs of its mean iteration time, and
    CBR = MSR / EOR (inf when EOR == 0). Peaks are the device allocator's
    high-water marks, times the measured iteration times."""
    if set(vanilla["exec"]) != set(scheduled["exec"]):
        raise PlannerError(abi.TSL_ERR_ARGUMENT, "traces cover different job sets")

    def time_cost(out):
        return sum(sum(r["iteration_ms"]) / len(r["iteration_ms"]) for r in out["exec"].values() if r["iteration_ms"])

    vmp, emp = float(vanilla["merged"]["hwm"]), float(scheduled["merged"]["hwm"])
    vtc, etc = time_cost(vanilla), time_cost(scheduled)
    if vmp <= 0:
        raise PlannerError(abi.TSL_ERR_ARGUMENT, "vanilla peak must be positive")
    if vtc <= 0:
        raise PlannerError(abi.TSL_ERR_ARGUMENT, "vanilla time cost must be positive")
    msr = (vmp - emp) / vmp
    eor = (etc - vtc) / vtc
    return {"msr": msr, "eor": eor, "cbr": float("inf") if eor == 0 else msr / eor}
