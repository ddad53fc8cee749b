"""TEST INFRASTRUCTURE: ctypes bridge to the UNMODIFIED reference library.

oracle/_ref/libmemsched_ref.so is the reference's own C++ hot path
(/root/reference/proj/src/{graph,access,plan,peak,swap_planner,
recompute_planner,orchestrator,workload,simulator,scenario}.cpp) compiled in
place by oracle/Makefile, plus oracle/ref_shim.cpp's C entry points. JSON in
the reference's formats crosses the boundary.
"""
from __future__ import annotations

import ctypes
import json
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libmemsched_ref.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference library not built: {LIB_PATH} (run make -C oracle ref)")
        L = ctypes.CDLL(LIB_PATH)
        cp = ctypes.POINTER(ctypes.c_char_p)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_free.argtypes = [ctypes.c_void_p]
        L.ref_generate_workload.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                                            ctypes.c_char_p, ctypes.c_uint64, ctypes.c_double,
                                            ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p)]
        L.ref_random_job.argtypes = [ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p),
                                     ctypes.POINTER(ctypes.c_void_p)]
        L.ref_initial_peaks.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.ref_build_plan.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                     ctypes.POINTER(ctypes.c_void_p)]
        L.ref_planned_random_job.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.POINTER(ctypes.c_void_p)]
        L.ref_analyze_job.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        del cp
        _lib = L
    return _lib


class ReferenceError_(RuntimeError):
    pass


def _take(p: ctypes.c_void_p) -> str:
    s = ctypes.cast(p, ctypes.c_char_p).value.decode()
    lib().ref_free(p)
    return s


def _check(rc: int):
    if rc != 0:
        raise ReferenceError_(lib().ref_last_error().decode())


def generate_workload(family: str, batch: int = 32, seed: int = 0, depth: int = 0, job_id: str = "",
                      lat_seed: int = 13, usage: float = 0.5):
    """Reference generate_workload + true_latency_table -> (graph dict, latency dict)."""
    g, l = ctypes.c_void_p(), ctypes.c_void_p()
    _check(lib().ref_generate_workload(family.encode(), batch, seed, depth, job_id.encode(), lat_seed, usage,
                                       ctypes.byref(g), ctypes.byref(l)))
    return json.loads(_take(g)), json.loads(_take(l))


def random_job(seed: int):
    g, l = ctypes.c_void_p(), ctypes.c_void_p()
    _check(lib().ref_random_job(seed, ctypes.byref(g), ctypes.byref(l)))
    return json.loads(_take(g)), json.loads(_take(l))


def _wire_config(config) -> dict:
    """JSON cannot carry NaN / infinity: non-finite max_swap_ratios travel as
    strings, which ref_shim.cpp's parse_config converts back with std::stod."""
    r = config.get("max_swap_ratios")
    if not r or all(math.isfinite(v) for v in r.values()):
        return config
    c = dict(config)
    c["max_swap_ratios"] = {k: (v if math.isfinite(v) else repr(float(v))) for k, v in r.items()}
    return c


def request(jobs, config) -> str:
    return json.dumps({"config": _wire_config(config), "jobs": [{"graph": g, "latencies": l} for g, l in jobs]})


def initial_peaks(jobs) -> dict:
    out = ctypes.c_void_p()
    _check(lib().ref_initial_peaks(request(jobs, {"pcie_bandwidth": 1, "transfer_setup": 0,
                                                  "memory_budget": 0}).encode(), ctypes.byref(out)))
    return json.loads(_take(out))


def build_plan(jobs, config, repeats: int = 1):
    """Returns (save_plans text, result dict with history/reports/times_ms)."""
    p, r = ctypes.c_void_p(), ctypes.c_void_p()
    _check(lib().ref_build_plan(request(jobs, config).encode(), repeats, ctypes.byref(p), ctypes.byref(r)))
    return _take(p), json.loads(_take(r))


def planned_random_job(seed: int, max_swaps: int = 3, bw: int = 4, setup: int = 1) -> dict:
    out = ctypes.c_void_p()
    _check(lib().ref_planned_random_job(seed, max_swaps, bw, setup, ctypes.byref(out)))
    return json.loads(_take(out))


def analyze_job(graph, latencies, plan) -> dict:
    out = ctypes.c_void_p()
    req = json.dumps({"graph": graph, "latencies": latencies, "plan": plan})
    _check(lib().ref_analyze_job(req.encode(), ctypes.byref(out)))
    return json.loads(_take(out))


def simulate(jobs, plans: dict, config: dict) -> dict:
    """memsched::simulate: jobs [(graph, true latencies, launch_tick)], plans a
    save_plans document ({job: plan}), config {"mode", "iterations", ...}."""
    L = lib()
    L.ref_simulate.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    out = ctypes.c_void_p()
    req = json.dumps({"jobs": [{"graph": g, "latencies": l, "launch_tick": t} for g, l, t in jobs],
                      "plans": plans, "config": config})
    _check(L.ref_simulate(req.encode(), ctypes.byref(out)))
    return json.loads(_take(out))


def _call_json(fn_name, argtypes, *args):
    L = lib()
    fn = getattr(L, fn_name)
    fn.argtypes = argtypes + [ctypes.POINTER(ctypes.c_void_p)]
    out = ctypes.c_void_p()
    _check(fn(*args, ctypes.byref(out)))
    return _take(out)


def training_samples(graph: dict, seed: int, per_op: int, noise: float):
    """generate_training_samples (workload.cpp:211-248): [(kind, values, label)]."""
    s = _call_json("ref_training_samples", [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_double],
                   json.dumps(graph).encode(), seed, per_op, noise)
    return [tuple(x) for x in json.loads(s)]


def linear_samples(noise: float, seed: int):
    """test_latency.cpp:44-62's samples: [(kind, values, label)]."""
    s = _call_json("ref_linear_samples", [ctypes.c_double, ctypes.c_uint64], noise, seed)
    return [tuple(x) for x in json.loads(s)]


def predictor_roundtrip(document: str) -> str:
    return _call_json("ref_predictor_roundtrip", [ctypes.c_char_p], document.encode())


def predict_latencies(graph: dict, predictor_doc: str, usage: float) -> dict:
    s = _call_json("ref_predict_latencies", [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_double],
                   json.dumps(graph).encode(), predictor_doc.encode(), usage)
    return json.loads(s)


def run_scenario(document: str, base_dir: str, modes=("vanilla", "scheduled", "passive")) -> dict:
    """run_scenario: {"stats": {mode: ModeStats::to_json text}, "csv": {mode: trace CSV},
    "plans": save_plans text, "replan_count", "diagnostic"}."""
    L = lib()
    L.ref_run_scenario.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    out = ctypes.c_void_p()
    _check(L.ref_run_scenario(document.encode(), base_dir.encode(), ",".join(modes).encode(), ctypes.byref(out)))
    return json.loads(_take(out))


def plan_scenario(document: str, base_dir: str):
    """The reference CLI's `plan` (load_scenario + plan_scenario):
    (plans.json text, peaks.json text, diagnostic)."""
    L = lib()
    L.ref_plan_scenario.argtypes = [ctypes.c_char_p, ctypes.c_char_p] + [ctypes.POINTER(ctypes.c_void_p)] * 3
    p, k, d = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    _check(L.ref_plan_scenario(document.encode(), base_dir.encode(), ctypes.byref(p), ctypes.byref(k),
                               ctypes.byref(d)))
    return _take(p), _take(k), _take(d)
