"""LatencyPredictor over the C-ABI (tsl_latency_*, csrc/tsl_latency.cpp): the
reference's cold-start latency model (latency.hpp:45-66) -- per op kind a
least-squares fit of latency ~ features + usage^2 + intercept, predictions
clamped at zero, JSON in the reference's format -- and predict_latencies
(orchestrator.cpp:72-87) for Orchestrator.plan_cold_start."""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import abi
from .planner import PlannerError, ValidationError, load_library


def _lib(path: Optional[str] = None):
    L = load_library(path)
    if not getattr(L, "_lat_bound", False):
        vp = C.c_void_p
        L.tsl_latency_fit.argtypes = [C.c_int32, C.POINTER(C.c_char_p), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(vp)]
        L.tsl_latency_from_json.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.tsl_latency_to_json.argtypes = [vp]
        L.tsl_latency_to_json.restype = vp
        L.tsl_latency_predict.argtypes = [vp, C.c_char_p, C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_double)]
        L.tsl_latency_r2.argtypes = [vp, C.c_char_p, C.POINTER(C.c_double)]
        L.tsl_predict_latencies.argtypes = [vp, C.POINTER(abi.TslJobDesc), C.POINTER(C.c_int32),
                                            C.POINTER(C.c_double), C.c_double, C.POINTER(C.c_int64)]
        L.tsl_latency_destroy.argtypes = [vp]
        L._lat_bound = True
    return L


class LatencyPredictor:
    def __init__(self, handle, lib):
        self._h = handle
        self.L = lib

    def _raise(self, rc):
        msg = self.L.tsl_last_error().decode()
        raise (ValidationError if rc == abi.TSL_ERR_VALIDATION else PlannerError)(rc, msg)

    @classmethod
    def fit(cls, samples: Sequence[Tuple[str, Sequence[float], float]], lib_path: Optional[str] = None):
        """samples: (op_kind, feature values (dims, attributes, usage), label)."""
        L = _lib(lib_path)
        kinds = (C.c_char_p * max(1, len(samples)))(*[k.encode() for k, _, _ in samples])
        offs = np.zeros(len(samples) + 1, dtype=np.int32)
        offs[1:] = np.cumsum([len(v) for _, v, _ in samples])
        vals = np.ascontiguousarray(np.concatenate([np.asarray(v, dtype=np.float64) for _, v, _ in samples])
                                    if samples else np.zeros(1))
        labels = np.ascontiguousarray(np.asarray([y for _, _, y in samples] or [0.0], dtype=np.float64))
        h = C.c_void_p()
        rc = L.tsl_latency_fit(len(samples), kinds, offs.ctypes.data_as(C.POINTER(C.c_int32)),
                               vals.ctypes.data_as(C.POINTER(C.c_double)),
                               labels.ctypes.data_as(C.POINTER(C.c_double)), C.byref(h))
        if rc:
            cls(None, L)._raise(rc)
        return cls(h, L)

    @classmethod
    def from_json(cls, document: str, lib_path: Optional[str] = None):
        L = _lib(lib_path)
        h = C.c_void_p()
        rc = L.tsl_latency_from_json(document.encode(), C.byref(h))
        if rc:
            cls(None, L)._raise(rc)
        return cls(h, L)

    def to_json(self) -> str:
        p = self.L.tsl_latency_to_json(self._h)
        s = C.cast(p, C.c_char_p).value.decode()
        self.L.tsl_free(p)
        return s

    def predict(self, op_kind: str, values: Sequence[float]) -> float:
        v = (C.c_double * max(1, len(values)))(*values)
        out = C.c_double()
        rc = self.L.tsl_latency_predict(self._h, op_kind.encode(), v, len(values), C.byref(out))
        if rc:
            self._raise(rc)
        return out.value

    def r2(self, op_kind: str) -> float:
        out = C.c_double()
        rc = self.L.tsl_latency_r2(self._h, op_kind.encode(), C.byref(out))
        if rc:
            self._raise(rc)
        return out.value

    def predict_latencies(self, graph: dict, gpu_usage: float) -> Dict[str, int]:
        """predict_latencies (orchestrator.cpp:72-87) -> {op: ticks}."""
        descs, arr = abi.pack_jobs([(graph, {o["id"]: 0 for o in graph["ops"]})])
        attrs = [list(o.get("attributes", [])) for o in graph["ops"]]
        offs = np.zeros(len(attrs) + 1, dtype=np.int32)
        offs[1:] = np.cumsum([len(a) for a in attrs])
        flat = np.ascontiguousarray(np.asarray([x for a in attrs for x in a] or [0.0], dtype=np.float64))
        out = (C.c_int64 * max(1, len(graph["ops"])))()
        rc = self.L.tsl_predict_latencies(self._h, arr, offs.ctypes.data_as(C.POINTER(C.c_int32)),
                                          flat.ctypes.data_as(C.POINTER(C.c_double)), float(gpu_usage), out)
        if rc:
            self._raise(rc)
        return {o["id"]: int(out[k]) for k, o in enumerate(graph["ops"])}

    def close(self):
        if self._h:
            self.L.tsl_latency_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
