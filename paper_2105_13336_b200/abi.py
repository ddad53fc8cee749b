"""ctypes mirror of include/tensile_b200.h and graph marshalling.

A graph here is the reference's graph document (the dict form of
memsched::save_graph / load_graph, graph.cpp:187-243):
    {"job_id": str,
     "tensors": [{"id", "size", "kind"}],
     "ops": [{"id", "kind", "inputs", "outputs", "attributes", "phase"}]}
and a latency table is {op_id: ticks} (the reference's std::map<OpId, Tick>).
`JobDesc` packs one (graph, latencies) pair into the C-ABI's integer SoA form
(tensor/op indices, CSR operand lists) and keeps the buffers alive.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

KINDS = {"input": 0, "interim": 1, "parameter": 2, "updated_parameter": 3, "output": 4}
KIND_NAMES = {v: k for k, v in KINDS.items()}
PHASES = {"forward_backward": 0, "optimize": 1}
LATENCY_MISSING = -(2 ** 63)

TSL_OK = 0
TSL_ERR_VALIDATION = 1
TSL_ERR_CUDA = 2
TSL_ERR_INTERNAL = 3
TSL_ERR_ARGUMENT = 4
TSL_ERR_CAPACITY = 5

_p64 = C.POINTER(C.c_int64)
_p32 = C.POINTER(C.c_int32)
_p8 = C.POINTER(C.c_int8)
_pstr = C.POINTER(C.c_char_p)


class TslConfig(C.Structure):
    _fields_ = [("pcie_bandwidth", C.c_int64), ("transfer_setup", C.c_int64), ("memory_budget", C.c_int64),
                ("ewma_alpha", C.c_double), ("replan_threshold", C.c_double), ("stall_epsilon", C.c_double),
                ("stall_min_iters", C.c_int32), ("cold_start_gpu_usage", C.c_double),
                ("n_max_swap_ratios", C.c_int32), ("max_swap_ratio_jobs", _pstr),
                ("max_swap_ratio_values", C.POINTER(C.c_double))]


class TslJobDesc(C.Structure):
    _fields_ = [("job_id", C.c_char_p), ("n_tensors", C.c_int32), ("tensor_ids", _pstr),
                ("tensor_sizes", _p64), ("tensor_kinds", _p8), ("n_ops", C.c_int32), ("op_ids", _pstr),
                ("op_kinds", _pstr), ("op_phases", _p8), ("op_in_offsets", _p32), ("op_inputs", _p32),
                ("op_out_offsets", _p32), ("op_outputs", _p32), ("op_latencies", _p64)]


class TslJobView(C.Structure):
    _fields_ = [("job_id", C.c_char_p), ("version", C.c_int64),
                ("n_swap", C.c_int32), ("ev_id", _p64), ("ev_tensor", _p32), ("ev_dir", _p8),
                ("ev_trigger", _p64), ("ev_delta", _p64), ("ev_start", _p64), ("ev_end", _p64),
                ("ev_earliest", _p64), ("ev_latest", _p64), ("ev_wraps", _p8), ("ev_pair", _p64),
                ("ev_serves", _p64),
                ("n_recompute", C.c_int32), ("rc_id", _p64), ("rc_tensor", _p32), ("rc_target", _p64),
                ("rc_regen_op", _p32), ("rc_latency", _p64), ("rc_saving", _p64),
                ("n_release", C.c_int32), ("release_flags", _p64),
                ("memory_peak", C.c_int64), ("peak_time", C.c_int64), ("has_last_input_access", C.c_int8),
                ("last_input_access", C.c_int64), ("n_peak_tensors", C.c_int32), ("peak_tensors", _p32),
                ("n_curve", C.c_int32), ("curve_time", _p64), ("curve_bytes", _p64),
                ("iteration_period", C.c_int64), ("n_accesses", C.c_int32)]


class TslPlanDesc(C.Structure):
    _fields_ = [("n_swap", C.c_int32), ("ev_id", _p64), ("ev_tensor", _p32), ("ev_dir", _p8),
                ("ev_trigger", _p64), ("ev_delta", _p64), ("ev_start", _p64), ("ev_end", _p64),
                ("ev_wraps", _p8), ("ev_pair", _p64), ("ev_serves", _p64),
                ("n_recompute", C.c_int32), ("rc_id", _p64), ("rc_tensor", _p32), ("rc_target", _p64),
                ("rc_regen_op", _p32), ("rc_latency", _p64), ("rc_saving", _p64),
                ("n_release", C.c_int32), ("release_flags", _p64), ("version", C.c_int64)]


class TslStats(C.Structure):
    _fields_ = [("kernel_ms", C.c_double), ("total_ms", C.c_double), ("n_accesses", C.c_int64),
                ("loop_iterations", C.c_int64), ("evaluations", C.c_int64), ("timeline_events", C.c_int64),
                ("candidates", C.c_int64), ("candidate_accesses", C.c_int64), ("busy_intervals", C.c_int64),
                ("algorithmic_bytes", C.c_int64), ("kernel_launches", C.c_int64),
                ("cyc_sequence", C.c_int64), ("cyc_evaluate", C.c_int64), ("cyc_swap", C.c_int64),
                ("cyc_recompute", C.c_int64), ("cyc_total", C.c_int64), ("rescored", C.c_int64),
                ("cyc_spec", C.c_int64), ("cyc_conflict", C.c_int64), ("cyc_sweep", C.c_int64),
                ("cyc_merge", C.c_int64), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("prep_ms", C.c_double), ("cyc_rescore", C.c_int64),
                ("cyc_apply", C.c_int64), ("debug", C.c_int64 * 4), ("cyc_pendsort", C.c_int64), ("fitprof", C.c_int64 * 9), ("evalprof", C.c_int64 * 7),
                ("queryprof", C.c_int64 * 16), ("comp_rescored", C.c_int64),
                ("stageprof", C.c_int64 * 24)]


class TslExecConfig(C.Structure):
    _fields_ = [("tick_ns", C.c_int64), ("iterations", C.c_int32), ("bytes_per_unit", C.c_int64),
                ("vanilla", C.c_int32), ("mempool", C.c_int32)]


class TslExecReport(C.Structure):
    _fields_ = [("predicted_peak", C.c_int64), ("hwm", C.c_int64), ("final_footprint", C.c_int64),
                ("iterations", C.c_int32), ("iteration_ms", C.c_double * 8), ("planned_iteration_ms", C.c_double),
                ("swap_outs", C.c_int32), ("swap_ins", C.c_int32), ("bytes_d2h", C.c_int64), ("bytes_h2d", C.c_int64),
                ("verify_errors", C.c_int32), ("violations", C.c_int32), ("kernels", C.c_int32),
                ("total_ms", C.c_double), ("pool_used_hwm", C.c_int64), ("pool_reserved_hwm", C.c_int64),
                ("pool_allocs", C.c_int64)]


def make_config(pcie_bandwidth: int = 1, transfer_setup: int = 0, memory_budget: int = 0,
                ewma_alpha: float = 0.3, replan_threshold: float = 0.2, stall_epsilon: float = 0.0005,
                stall_min_iters: int = 100, cold_start_gpu_usage: float = 0.5,
                max_swap_ratios: Optional[Dict[str, float]] = None, **_ignored) -> TslConfig:
    """PlannerConfig (config.hpp:9-18) with the reference defaults. The
    max_swap_ratios map's arrays stay alive with the returned struct (`_keep`)."""
    ratios = dict(max_swap_ratios or {})
    jobs = (C.c_char_p * max(1, len(ratios)))(*[k.encode() for k in ratios])
    vals = (C.c_double * max(1, len(ratios)))(*[float(v) for v in ratios.values()])
    cfg = TslConfig(int(pcie_bandwidth), int(transfer_setup), int(memory_budget), float(ewma_alpha),
                    float(replan_threshold), float(stall_epsilon), int(stall_min_iters),
                    float(cold_start_gpu_usage), len(ratios), C.cast(jobs, _pstr),
                    C.cast(vals, C.POINTER(C.c_double)))
    cfg._keep = (jobs, vals)
    return cfg


def _arr(values, dtype):
    a = np.ascontiguousarray(np.asarray(values, dtype=dtype))
    if a.size == 0:
        a = np.zeros(1, dtype=dtype)
    return a


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


class _CStrings:
    """A `const char* const*` table: the strings NUL-joined in one buffer and
    a pointer array into it (built with numpy, not one ctypes object per id)."""

    def __init__(self, strings: List[str]):
        blob = ("\0".join(strings) + "\0").encode()
        self.buf = np.frombuffer(blob, dtype=np.uint8).copy()
        ends = np.flatnonzero(self.buf == 0)  # ids are C strings: no NUL inside
        starts = np.empty(max(1, len(strings)), dtype=np.uint64)
        starts[0] = 0
        starts[1:len(strings)] = ends[:len(strings) - 1] + 1
        self.addrs = starts + np.uint64(self.buf.ctypes.data)
        self.ptrs = self.addrs.ctypes.data_as(_pstr)


def _offsets(counts: List[int]) -> np.ndarray:
    out = np.zeros(len(counts) + 1, dtype=np.int32)
    np.cumsum(counts, out=out[1:])
    return out


class JobDesc:
    """One (graph, latencies) job packed for the C-ABI."""

    def __init__(self, graph: dict, latencies: Dict[str, int]):
        self.graph = graph
        tensors = graph["tensors"]
        ops = graph["ops"]
        self.tensor_ids: List[str] = [t["id"] for t in tensors]
        self.op_ids: List[str] = [o["id"] for o in ops]
        tindex: Dict[str, int] = {}
        for i, t in enumerate(self.tensor_ids):
            tindex.setdefault(t, i)
        self.tindex = tindex
        self.oindex = {o: i for i, o in enumerate(self.op_ids)}

        self._tids = _CStrings(self.tensor_ids)
        self._oids = _CStrings(self.op_ids)
        self._okinds = _CStrings([o["kind"] for o in ops])
        self._sizes = _arr([t["size"] for t in tensors], np.int64)
        self._kinds = _arr([KINDS[t["kind"]] for t in tensors], np.int8)
        self._phases = _arr([PHASES[o["phase"]] for o in ops], np.int8)
        tget = tindex.get  # a dangling reference packs to -1; the library reports it
        self._ins = _arr([tget(t, -1) for o in ops for t in o["inputs"]], np.int32)
        self._outs = _arr([tget(t, -1) for o in ops for t in o["outputs"]], np.int32)
        self._ioff = _offsets([len(o["inputs"]) for o in ops])
        self._ooff = _offsets([len(o["outputs"]) for o in ops])
        self._lat = _arr([latencies.get(o, LATENCY_MISSING) for o in self.op_ids], np.int64)
        self._jid = graph["job_id"].encode()
        self.desc = TslJobDesc(self._jid, len(tensors), self._tids.ptrs, _ptr(self._sizes, C.c_int64),
                               _ptr(self._kinds, C.c_int8), len(ops), self._oids.ptrs, self._okinds.ptrs,
                               _ptr(self._phases, C.c_int8), _ptr(self._ioff, C.c_int32),
                               _ptr(self._ins, C.c_int32), _ptr(self._ooff, C.c_int32),
                               _ptr(self._outs, C.c_int32), _ptr(self._lat, C.c_int64))


def pack_jobs(jobs: Sequence[Tuple]):
    """[(graph, latencies), ...] -> (list[JobDesc], TslJobDesc array)."""
    # a job object passed several times (the requests of a replan sequence)
    # is packed once: identical descriptors let the library load it once
    memo = {}
    descs = []
    for g, l in jobs:
        key = (id(g), id(l))
        if key not in memo:
            memo[key] = JobDesc(g, l)
        descs.append(memo[key])
    arr = (TslJobDesc * max(1, len(descs)))(*[d.desc for d in descs])
    return descs, arr


class PlanDesc:
    """A plan dict in save_plans form -> tsl_plan_desc for analyze_job."""

    def __init__(self, plan: dict, job: JobDesc):
        sw = plan.get("swap_events", [])
        rc = plan.get("recompute_events", [])
        self._id = _arr([e["event_id"] for e in sw], np.int64)
        self._tensor = _arr([job.tindex[e["tensor"]] for e in sw], np.int32)
        self._dir = _arr([0 if e["direction"] == "out" else 1 for e in sw], np.int8)
        self._trig = _arr([e["trigger_access"] for e in sw], np.int64)
        self._delta = _arr([e["delta_time"] for e in sw], np.int64)
        self._start = _arr([e["start_time"] for e in sw], np.int64)
        self._end = _arr([e["end_time"] for e in sw], np.int64)
        self._wraps = _arr([1 if e["wraps_iteration"] else 0 for e in sw], np.int8)
        self._pair = _arr([e["pair_id"] for e in sw], np.int64)
        self._serves = _arr([e["serves_access"] for e in sw], np.int64)
        self._rid = _arr([e["event_id"] for e in rc], np.int64)
        self._rt = _arr([job.tindex[e["tensor"]] for e in rc], np.int32)
        self._rtarget = _arr([e["target_access"] for e in rc], np.int64)
        self._rop = _arr([job.oindex[e["regen_op"]] for e in rc], np.int32)
        self._rlat = _arr([e["recompute_latency"] for e in rc], np.int64)
        self._rsav = _arr([e["memory_saving"] for e in rc], np.int64)
        self._flags = _arr(sorted(plan.get("release_flags", [])), np.int64)
        p64 = lambda a: _ptr(a, C.c_int64)  # noqa: E731
        self.desc = TslPlanDesc(len(sw), p64(self._id), _ptr(self._tensor, C.c_int32), _ptr(self._dir, C.c_int8),
                                p64(self._trig), p64(self._delta), p64(self._start), p64(self._end),
                                _ptr(self._wraps, C.c_int8), p64(self._pair), p64(self._serves),
                                len(rc), p64(self._rid), _ptr(self._rt, C.c_int32), p64(self._rtarget),
                                _ptr(self._rop, C.c_int32), p64(self._rlat), p64(self._rsav),
                                len(plan.get("release_flags", [])), p64(self._flags),
                                int(plan.get("version", 0)))


def _np(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def view_to_dict(v: TslJobView, job: JobDesc) -> dict:
    """Job view -> {"plan": save_plans entry, "report": PeakReport fields, ...} (python values)."""
    n = v.n_swap
    ids, ten, dr = _np(v.ev_id, n, np.int64), _np(v.ev_tensor, n, np.int32), _np(v.ev_dir, n, np.int8)
    trig, delta = _np(v.ev_trigger, n, np.int64), _np(v.ev_delta, n, np.int64)
    st, en = _np(v.ev_start, n, np.int64), _np(v.ev_end, n, np.int64)
    ea, la = _np(v.ev_earliest, n, np.int64), _np(v.ev_latest, n, np.int64)
    wr, pr, sv = _np(v.ev_wraps, n, np.int8), _np(v.ev_pair, n, np.int64), _np(v.ev_serves, n, np.int64)
    swaps = [{"event_id": int(ids[i]), "tensor": job.tensor_ids[ten[i]], "direction": "out" if dr[i] == 0 else "in",
              "trigger_access": int(trig[i]), "delta_time": int(delta[i]), "wraps_iteration": bool(wr[i]),
              "start_time": int(st[i]), "end_time": int(en[i]), "pair_id": int(pr[i]),
              "serves_access": int(sv[i]), "earliest_time": int(ea[i]), "latest_time": int(la[i])}
             for i in range(n)]
    m = v.n_recompute
    rid, rt, rtar = _np(v.rc_id, m, np.int64), _np(v.rc_tensor, m, np.int32), _np(v.rc_target, m, np.int64)
    rop, rlat, rsav = _np(v.rc_regen_op, m, np.int32), _np(v.rc_latency, m, np.int64), _np(v.rc_saving, m, np.int64)
    recs = [{"event_id": int(rid[i]), "tensor": job.tensor_ids[rt[i]], "target_access": int(rtar[i]),
             "regen_op": job.op_ids[rop[i]], "recompute_latency": int(rlat[i]), "memory_saving": int(rsav[i])}
            for i in range(m)]
    flags = [int(x) for x in _np(v.release_flags, v.n_release, np.int64)]
    pt = _np(v.peak_tensors, v.n_peak_tensors, np.int32)
    ct, cb = _np(v.curve_time, v.n_curve, np.int64), _np(v.curve_bytes, v.n_curve, np.int64)
    return {
        "job_id": v.job_id.decode(),
        "plan": {"version": int(v.version), "swap_events": swaps, "recompute_events": recs, "release_flags": flags},
        "report": {"memory_peak": int(v.memory_peak), "peak_tensors": [job.tensor_ids[t] for t in pt],
                   "last_input_access": int(v.last_input_access) if v.has_last_input_access else None,
                   "peak_time": int(v.peak_time),
                   "footprint_curve": [[int(a), int(b)] for a, b in zip(ct, cb)]},
        "iteration_period": int(v.iteration_period),
        "n_accesses": int(v.n_accesses),
    }
