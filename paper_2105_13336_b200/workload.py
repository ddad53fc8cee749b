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


# ---------------------------------------------------------------------------
# C4: GPT-2-medium training trace (not in the reference's
# generator). One job: `micro_batches` sequences of `seq` tokens through
# `layers` transformer blocks (d_model, `heads` attention heads), forward +
# backward per micro-batch with per-head attention ops, weight-gradient
# accumulation across micro-batches, then one `update` op per parameter
# tensor -- the weights and their two Adam moments are separate parameters,
# each with its own update op (graph.cpp:89-110 allows one parameter per
# update). Sizes are fp16 bytes (moments fp32). Defaults give ~1.0 M accesses.
# ---------------------------------------------------------------------------
def gpt2_workload(layers: int = 24, d_model: int = 1024, heads: int = 16, seq: int = 1024,
                  micro_batches: int = 70, job_id: str = "gpt2m") -> dict:
    if layers < 1 or heads < 1 or micro_batches < 1 or d_model % heads:
        raise ValueError("gpt2_workload: bad shape")
    H, D, S, L, M = heads, d_model, seq, layers, micro_batches
    hd = D // H
    f16 = 2
    tensors: List[dict] = []
    ops: List[dict] = []

    def T(tid, size, kind="interim"):
        tensors.append({"id": tid, "size": int(size), "kind": kind})
        return tid

    def OP(oid, kind, ins, outs, phase="forward_backward"):
        ops.append({"id": oid, "kind": kind, "inputs": list(ins), "outputs": list(outs),
                    "attributes": [], "phase": phase})

    # parameters of block l: name -> size (bytes); the moments are fp32
    pshape = {"ln1g": D, "ln1b": D, "wqkv": D * 3 * D, "bqkv": 3 * D, "wo": D * D, "bo": D,
              "ln2g": D, "ln2b": D, "w1": D * 4 * D, "b1": 4 * D, "w2": 4 * D * D, "b2": D}
    pnames = list(pshape)
    for l in range(L):
        for p in pnames:
            base = f"p.l{l:02d}.{p}"
            T(base, pshape[p] * f16, "parameter")
            T(base + ".m1", pshape[p] * 4, "parameter")
            T(base + ".m2", pshape[p] * 4, "parameter")
    act = S * D * f16
    qkvh = S * hd * f16
    att = S * S * f16
    mlp = S * 4 * D * f16
    for m in range(M):
        mp = f"m{m:03d}"
        h = T(f"{mp}.x", act, "input")
        saved = []
        for l in range(L):
            lp = f"{mp}.f.l{l:02d}"
            P = lambda n: f"p.l{l:02d}.{n}"  # noqa: E731
            if m == 0:
                # optimizer-state statistics early in the iteration: every
                # moment has a use before its own update op (a moment read only
                # by its update makes the reference's wrapped swap-in land on
                # the updated version's TGA tick: "swap-in of resident tensor")
                OP(f"{lp}.0.opt", "adam_stats", [P(n) + sfx for n in pnames for sfx in (".m1", ".m2")],
                   [T(f"{lp}.ostat", 64)])
            ln1 = T(f"{lp}.ln1", act)
            OP(f"{lp}.a.ln1", "layernorm", [h, P("ln1g"), P("ln1b")], [ln1])
            q = [T(f"{lp}.q{k:02d}", qkvh) for k in range(H)]
            kk = [T(f"{lp}.k{k:02d}", qkvh) for k in range(H)]
            v = [T(f"{lp}.v{k:02d}", qkvh) for k in range(H)]
            OP(f"{lp}.b.qkv", "matmul", [ln1, P("wqkv"), P("bqkv")], q + kk + v)
            c = []
            for k in range(H):
                s_ = T(f"{lp}.s{k:02d}", att)
                p_ = T(f"{lp}.p{k:02d}", att)
                c_ = T(f"{lp}.c{k:02d}", qkvh)
                OP(f"{lp}.c.h{k:02d}.1score", "attn_score", [q[k], kk[k]], [s_])
                OP(f"{lp}.c.h{k:02d}.2softmax", "softmax", [s_], [p_])
                OP(f"{lp}.c.h{k:02d}.3ctx", "attn_ctx", [p_, v[k]], [c_])
                c.append(c_)
            ao = T(f"{lp}.ao", act)
            OP(f"{lp}.d.proj", "matmul", c + [P("wo"), P("bo")], [ao])
            h1 = T(f"{lp}.h1", act)
            OP(f"{lp}.e.res1", "add", [h, ao], [h1])
            ln2 = T(f"{lp}.ln2", act)
            OP(f"{lp}.f.ln2", "layernorm", [h1, P("ln2g"), P("ln2b")], [ln2])
            f1 = T(f"{lp}.f1", mlp)
            OP(f"{lp}.g.fc1", "matmul", [ln2, P("w1"), P("b1")], [f1])
            f2 = T(f"{lp}.f2", mlp)
            OP(f"{lp}.h.gelu", "gelu", [f1], [f2])
            f3 = T(f"{lp}.f3", act)
            OP(f"{lp}.i.fc2", "matmul", [f2, P("w2"), P("b2")], [f3])
            ho = T(f"{lp}.ho", act)
            OP(f"{lp}.j.res2", "add", [h1, f3], [ho])
            saved.append((h, ln1, q, kk, v, c, h1, ln2, f1, f2))
            h = ho
        loss = T(f"{mp}.loss", 4 * S, "output")
        dh = T(f"{mp}.dy", act)
        OP(f"{mp}.g.loss", "loss", [h], [loss, dh])
        for l in range(L - 1, -1, -1):
            lp = f"{mp}.h.l{L - 1 - l:02d}"
            P = lambda n: f"p.l{l:02d}.{n}"  # noqa: E731
            G = lambda n: f"{mp}.dw.l{l:02d}.{n}"  # noqa: E731
            h_in, ln1, q, kk, v, c, h1, ln2, f1, f2 = saved[l]
            df2 = T(f"{lp}.df2", mlp)
            OP(f"{lp}.a.fc2b", "matmul_b", [dh, f2, P("w2")], [df2, T(G("w2"), pshape["w2"] * f16),
                                                              T(G("b2"), pshape["b2"] * f16)])
            df1 = T(f"{lp}.df1", mlp)
            OP(f"{lp}.b.gelub", "gelu_b", [df2, f1], [df1])
            dln2 = T(f"{lp}.dln2", act)
            OP(f"{lp}.c.fc1b", "matmul_b", [df1, ln2, P("w1")], [dln2, T(G("w1"), pshape["w1"] * f16),
                                                                T(G("b1"), pshape["b1"] * f16)])
            dh1a = T(f"{lp}.dh1a", act)
            OP(f"{lp}.d.ln2b", "layernorm_b", [dln2, h1, P("ln2g")], [dh1a, T(G("ln2g"), pshape["ln2g"] * f16),
                                                                     T(G("ln2b"), pshape["ln2b"] * f16)])
            dh1 = T(f"{lp}.dh1", act)
            OP(f"{lp}.e.res2b", "add", [dh, dh1a], [dh1])
            dc = [T(f"{lp}.dc{k:02d}", qkvh) for k in range(H)]
            OP(f"{lp}.f.projb", "matmul_b", [dh1] + c + [P("wo")], dc + [T(G("wo"), pshape["wo"] * f16),
                                                                       T(G("bo"), pshape["bo"] * f16)])
            dq, dk, dv = [], [], []
            for k in range(H):
                dp_ = T(f"{lp}.dp{k:02d}", att)
                dv_ = T(f"{lp}.dv{k:02d}", qkvh)
                s_p = f"{mp}.f.l{l:02d}.p{k:02d}"
                OP(f"{lp}.g.h{k:02d}.1ctxb", "attn_ctx_b", [dc[k], s_p, v[k]], [dp_, dv_])
                ds_ = T(f"{lp}.ds{k:02d}", att)
                OP(f"{lp}.g.h{k:02d}.2softmaxb", "softmax_b", [dp_, s_p], [ds_])
                dq_ = T(f"{lp}.dq{k:02d}", qkvh)
                dk_ = T(f"{lp}.dk{k:02d}", qkvh)
                OP(f"{lp}.g.h{k:02d}.3scoreb", "attn_score_b", [ds_, q[k], kk[k]], [dq_, dk_])
                dq.append(dq_); dk.append(dk_); dv.append(dv_)
            dln1 = T(f"{lp}.dln1", act)
            OP(f"{lp}.h.qkvb", "matmul_b", dq + dk + dv + [ln1, P("wqkv")],
               [dln1, T(G("wqkv"), pshape["wqkv"] * f16), T(G("bqkv"), pshape["bqkv"] * f16)])
            dha = T(f"{lp}.dha", act)
            OP(f"{lp}.i.ln1b", "layernorm_b", [dln1, h_in, P("ln1g")], [dha, T(G("ln1g"), pshape["ln1g"] * f16),
                                                                       T(G("ln1b"), pshape["ln1b"] * f16)])
            dhn = T(f"{lp}.dh", act)
            OP(f"{lp}.j.res1b", "add", [dh1, dha], [dhn])
            dh = dhn
            # weight-gradient accumulation across micro-batches
            if m > 0:
                for p in pnames:
                    acc = T(f"{mp}.acc.l{l:02d}.{p}", pshape[p] * f16)
                    prev = f"m{m - 1:03d}.dw.l{l:02d}.{p}" if m == 1 else f"m{m - 1:03d}.acc.l{l:02d}.{p}"
                    OP(f"{mp}.i.acc.l{l:02d}.{p}", "accumulate", [prev, G(p)], [acc])
        # the last micro-batch's input gradient leaves the graph through a sink
        OP(f"{mp}.j.sink", "sink", [dh], [T(f"{mp}.dx", act, "output")])
    last = f"m{M - 1:03d}"
    for l in range(L):
        for p in pnames:
            base = f"p.l{l:02d}.{p}"
            g_ = f"{last}.dw.l{l:02d}.{p}" if M == 1 else f"{last}.acc.l{l:02d}.{p}"
            for sfx, sz in (("", pshape[p] * f16), (".m1", pshape[p] * 4), (".m2", pshape[p] * 4)):
                T(base + sfx + "_new", sz, "updated_parameter")
                OP(f"u.l{l:02d}.{p}{sfx}", "update", [base + sfx, g_], [base + sfx + "_new"], "optimize")
    return {"job_id": job_id, "tensors": tensors, "ops": ops}


def c4_job(micro_batches: int = 70, layers: int = 24, heads: int = 16, lat_seed: int = 13,
           job_id: str = "gpt2m") -> Tuple[dict, dict]:
    g = gpt2_workload(layers=layers, heads=heads, micro_batches=micro_batches, job_id=job_id)
    return g, true_latency_table(g, lat_seed)
