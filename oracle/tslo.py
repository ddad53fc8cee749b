"""TEST INFRASTRUCTURE: ctypes bridge to the restated CPU oracle
(oracle/build/libtsl_oracle.so, built from oracle/tensile_oracle.cpp).

Same inputs as the product's C-ABI (include/tensile_b200.h); results are
returned as python values. Only tests/, smoke() and bench.py's cpu_baseline
arm use this module.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import time

from paper_2105_13336_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libtsl_oracle.so")
_lib = None


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"oracle not built: {LIB_PATH} (run make -C oracle oracle)")
        L = C.CDLL(LIB_PATH)
        L.tslo_last_error.restype = C.c_char_p
        L.tslo_build_plan.argtypes = [C.POINTER(abi.TslJobDesc), C.c_int32, C.POINTER(abi.TslConfig),
                                      C.POINTER(C.c_void_p)]
        L.tslo_initial_peaks.argtypes = [C.POINTER(abi.TslJobDesc), C.c_int32, C.POINTER(C.c_int64)]
        L.tslo_analyze_job.argtypes = [C.POINTER(abi.TslJobDesc), C.POINTER(abi.TslPlanDesc), C.POINTER(C.c_void_p)]
        L.tslo_result_n_jobs.argtypes = [C.c_void_p]
        L.tslo_result_job.argtypes = [C.c_void_p, C.c_int32, C.POINTER(abi.TslJobView)]
        L.tslo_result_history.argtypes = [C.c_void_p, C.POINTER(C.POINTER(C.c_int64))]
        L.tslo_result_final_merged_peak.argtypes = [C.c_void_p]
        L.tslo_result_final_merged_peak.restype = C.c_int64
        L.tslo_result_within_budget.argtypes = [C.c_void_p]
        L.tslo_result_diagnostic.argtypes = [C.c_void_p]
        L.tslo_result_diagnostic.restype = C.c_char_p
        L.tslo_result_save_plans.argtypes = [C.c_void_p]
        L.tslo_result_save_plans.restype = C.c_void_p
        L.tslo_result_report_json.argtypes = [C.c_void_p, C.c_int32]
        L.tslo_result_report_json.restype = C.c_void_p
        L.tslo_result_destroy.argtypes = [C.c_void_p]
        L.tslo_free.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _take(p) -> str:
    s = C.cast(p, C.c_char_p).value.decode()
    lib().tslo_free(p)
    return s


def _collect(L, res, descs) -> dict:
    out = {"jobs": {}, "reports_json": {}}
    for i in range(L.tslo_result_n_jobs(res)):
        v = abi.TslJobView()
        L.tslo_result_job(res, i, C.byref(v))
        jid = v.job_id.decode()
        job = next(d for d in descs if d.graph["job_id"] == jid)
        out["jobs"][jid] = abi.view_to_dict(v, job)
        out["reports_json"][jid] = _take(L.tslo_result_report_json(res, i))
    h = C.POINTER(C.c_int64)()
    n = L.tslo_result_history(res, C.byref(h))
    out["merged_peak_history"] = [h[i] for i in range(n)]
    out["final_merged_peak"] = L.tslo_result_final_merged_peak(res)
    out["within_budget"] = bool(L.tslo_result_within_budget(res))
    out["diagnostic"] = L.tslo_result_diagnostic(res).decode()
    out["plans_json"] = _take(L.tslo_result_save_plans(res))
    return out


def build_plan(jobs, config: dict, max_swap_ratios=None) -> dict:
    """Oracle build_plan over [(graph, latencies)] -> dict (plans_json = save_plans text)."""
    L = lib()
    if max_swap_ratios:
        config = dict(config, max_swap_ratios=max_swap_ratios)
    descs, arr = abi.pack_jobs(jobs)
    cfg = abi.make_config(**config)
    res = C.c_void_p()
    t0 = time.perf_counter()
    rc = L.tslo_build_plan(arr, len(descs), C.byref(cfg), C.byref(res))
    t1 = time.perf_counter()
    if rc != 0:
        raise OracleError(rc, L.tslo_last_error().decode())
    try:
        out = _collect(L, res, descs)
    finally:
        L.tslo_result_destroy(res)
    out["ms"] = (t1 - t0) * 1e3
    return out


def analyze_job(graph, latencies, plan: dict) -> dict:
    L = lib()
    jd = abi.JobDesc(graph, latencies)
    pd = abi.PlanDesc(plan, jd)
    res = C.c_void_p()
    rc = L.tslo_analyze_job(C.byref(jd.desc), C.byref(pd.desc), C.byref(res))
    if rc != 0:
        raise OracleError(rc, L.tslo_last_error().decode())
    try:
        out = _collect(L, res, [jd])
    finally:
        L.tslo_result_destroy(res)
    jid = graph["job_id"]
    return {"report": out["jobs"][jid]["report"], "report_json": out["reports_json"][jid]}


def report_dict(report_json: str) -> dict:
    return json.loads(report_json)


def initial_peaks(jobs) -> dict:
    """{job_id: initial peak} (make_job_context's report: empty plan, release
    at last use)."""
    descs, arr = abi.pack_jobs(jobs)
    out = (C.c_int64 * max(1, len(jobs)))()
    rc = lib().tslo_initial_peaks(arr, len(jobs), out)
    if rc:
        raise OracleError(rc, lib().tslo_last_error().decode())
    return {g["job_id"]: int(out[i]) for i, (g, _) in enumerate(jobs)}
