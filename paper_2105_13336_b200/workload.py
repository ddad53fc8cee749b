"""Synthetic workload graphs (host-side fixture generator, not the hot path).

Restates the reference's deterministic generator so the benchmark and the
multi-GPU driver can build the named traces without the reference library:
  generate_workload      workload.cpp:27-163 (families vgg16, resnet50,
                         inception_v3, inception_v4, densenet, chain)
  true_latency_table     workload.cpp:165-209 (splitmix LatencyOracle)
The "random" family draws from libstdc++'s mt19937_64 distributions and is
only used through reference-generated fixtures (tests/golden/).
Outputs are graph documents in the reference's JSON form (graph.cpp:225-243).
tests/test_workload.py checks every family byte-for-byte against the
reference generator.
"""
from __future__ import annotations

import math
from typing import Dict, List, Tuple

MASK = (1 << 64) - 1


def _index_id(prefix: str, i: int) -> str:  # workload.cpp:12-18 (2-digit pad only)
    return f"{prefix}{'0' if i < 10 else ''}{i}"


def _llround(x: float) -> int:
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def _profile(family: str, depth: int):  # workload.cpp:27-92
    act: List[int] = []
    par: List[int] = []
    skips: Dict[int, int] = {}

    def ramp_down(layers, hi, lo):
        for i in range(layers):
            t = float(i) / (layers - 1) if layers > 1 else 0.0
            act.append(max(1, _llround(hi + t * (lo - hi))))

    def ramp_up_params(layers, lo, hi):
        for i in range(layers):
            t = float(i) / (layers - 1) if layers > 1 else 0.0
            par.append(max(1, _llround(lo + t * (hi - lo))))

    if family == "vgg16":
        ramp_down(13, 64, 4)
        act.extend([2, 2, 1])
        ramp_up_params(13, 2, 32)
        par.extend([512, 256, 128])
    elif family == "resnet50":
        ramp_down(50, 32, 2)
        ramp_up_params(50, 2, 48)
        for i in range(4, 50, 3):
            skips[i] = i - 3
    elif family == "inception_v3":
        ramp_down(48, 48, 3)
        ramp_up_params(48, 2, 40)
        for i in range(6, 48, 5):
            skips[i] = i - 4
    elif family == "inception_v4":
        ramp_down(55, 48, 3)
        ramp_up_params(55, 2, 44)
        for i in range(6, 55, 5):
            skips[i] = i - 4
    elif family == "densenet":
        for i in range(58):
            act.append(8 + i // 2)
        ramp_up_params(58, 2, 24)
        for i in range(3, 58, 2):
            skips[i] = i - 2
    elif family == "chain":
        d = depth if depth > 0 else 8
        act.extend([16] * d)
        par.extend([8] * d)
    else:
        raise ValueError(f"unknown workload family: {family}")
    return act, par, skips


def generate_workload(family: str = "chain", batch_size: int = 32, seed: int = 0, depth: int = 0,
                      job_id: str = "") -> dict:
    """generate_workload (workload.cpp:96-163) -> graph document."""
    if batch_size < 1:
        raise ValueError("batch_size must be at least 1")
    act_u, par_u, skips = _profile(family, depth)
    L = len(act_u)
    b = batch_size
    act = lambda i: _index_id("a", i)  # noqa: E731
    grad = lambda i: _index_id("g", i)  # noqa: E731
    weight = lambda i: _index_id("w", i)  # noqa: E731
    wgrad = lambda i: _index_id("wg", i)  # noqa: E731
    tensors = [{"id": "x", "size": act_u[0] * b, "kind": "input"}]
    for i in range(1, L + 1):
        a_size = act_u[i - 1] * b
        w_size = par_u[i - 1] * 16
        if i < L:
            tensors.append({"id": act(i), "size": a_size, "kind": "interim"})
        tensors.append({"id": weight(i), "size": w_size, "kind": "parameter"})
        tensors.append({"id": weight(i) + "_new", "size": w_size, "kind": "updated_parameter"})
        if i > 1:
            tensors.append({"id": grad(i - 1), "size": a_size, "kind": "interim"})
        tensors.append({"id": wgrad(i), "size": par_u[i - 1] * b, "kind": "interim"})
    tensors.append({"id": "y", "size": act_u[-1] * b, "kind": "output"})
    ops = []
    for i in range(1, L + 1):
        inputs = ["x" if i == 1 else act(i - 1), weight(i)]
        if i in skips:
            inputs.append(act(skips[i]))
        ops.append({"id": _index_id("f", i), "kind": "forward", "inputs": inputs,
                    "outputs": ["y" if i == L else act(i)],
                    "attributes": [float(i), float(act_u[i - 1])], "phase": "forward_backward"})
    for i in range(L, 0, -1):
        outs = [grad(i - 1)] if i > 1 else []
        outs.append(wgrad(i))
        ops.append({"id": _index_id("b", i), "kind": "backward",
                    "inputs": ["y" if i == L else grad(i), "x" if i == 1 else act(i - 1), weight(i)],
                    "outputs": outs, "attributes": [float(i), float(act_u[i - 1])],
                    "phase": "forward_backward"})
    for i in range(1, L + 1):
        ops.append({"id": _index_id("u", i), "kind": "update", "inputs": [weight(i), wgrad(i)],
                    "outputs": [weight(i) + "_new"], "attributes": [float(i)], "phase": "optimize"})
    return {"job_id": job_id or family, "tensors": tensors, "ops": ops}


def _mix(z: int) -> int:  # workload.cpp:168-173
    z = (z + 0x9E3779B97F4A7C15) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def _kind_key(seed: int, kind: str) -> int:
    h = seed & MASK
    for ch in kind.encode():
        h = _mix(h ^ ch)
    return h


def _unit(bits: int) -> float:
    return float(bits >> 11) / float(1 << 53)


def latency_value(seed: int, op_kind: str, total_input_bytes: float, gpu_usage: float) -> float:
    """LatencyOracle::value (workload.cpp:188-195)."""
    k = _kind_key(seed, op_kind)
    base = 4.0 + 16.0 * _unit(_mix(k ^ 1))
    per_byte = 0.005 + 0.02 * _unit(_mix(k ^ 2))
    usage_coeff = 2.0 + 8.0 * _unit(_mix(k ^ 3))
    return base + per_byte * total_input_bytes + usage_coeff * gpu_usage


def true_latency_table(graph: dict, seed: int, gpu_usage: float = 0.5) -> Dict[str, int]:
    """true_latency_table (workload.cpp:197-209)."""
    sizes = {t["id"]: t["size"] for t in graph["tensors"]}
    out = {}
    for op in graph["ops"]:
        total = 0.0
        for t in op["inputs"]:
            total += float(sizes[t])
        out[op["id"]] = max(1, _llround(latency_value(seed, op["kind"], total, gpu_usage)))
    return out


def job(family: str, batch: int, job_id: str = "", lat_seed: int = 13, depth: int = 0) -> Tuple[dict, dict]:
    g = generate_workload(family, batch, 0, depth, job_id)
    return g, true_latency_table(g, lat_seed)
