"""Test fixtures re-expressed from the reference's test support
(/root/reference/proj/tests/support/fixtures.hpp:18-86) and the hand-built
profile stores of its suites (test_simulator.cpp:25-63, :177-205,
acceptance_main.cpp:241-306), as JSON / JSONL text both engines consume."""
from __future__ import annotations

import json
import math


def dense_model(layers, heads, kv_heads, head_dim, intermediate, vocab=32000, ffn="silu",
                dtype="fp16"):
    return json.dumps({"name": "fixture", "num_hidden_layers": layers,
                       "hidden_size": heads * head_dim, "num_attention_heads": heads,
                       "num_key_value_heads": kv_heads, "head_dim": head_dim,
                       "intermediate_size": intermediate, "vocab_size": vocab,
                       "torch_dtype": dtype, "hidden_act": ffn})


def moe_model(layers, heads, kv_heads, head_dim, expert_intermediate, experts, per_tok,
              vocab=32000):
    d = json.loads(dense_model(layers, heads, kv_heads, head_dim, expert_intermediate, vocab))
    d["num_local_experts"] = experts
    d["num_experts_per_tok"] = per_tok
    return json.dumps(d)


def cluster(levels, mem_bytes, peak_fp16, mem_bw, freqs=(2.0,), tdp=700.0):
    """levels: [(fan_out, bandwidth, latency), ...]; fp8 peak = 2x fp16 (fixtures.hpp:54-69)."""
    return json.dumps({
        "levels": [{"fan_out": f, "link_bandwidth_bytes_per_s": b, "link_latency_s": l}
                   for f, b, l in levels],
        "device": {"name": "fixture-gpu", "memory_capacity_bytes": mem_bytes,
                   "peak_flops": {"fp16": peak_fp16, "fp8": 2.0 * peak_fp16},
                   "peak_mem_bandwidth_bytes_per_s": mem_bw,
                   "frequency_options_ghz": list(freqs), "tdp_watts": tdp}})


def trace_jsonl(requests):
    """requests: [(id, ctx, gen, arrival)]"""
    return "".join(json.dumps({"id": i, "context_len": c, "gen_len": g, "arrival_s": a}) + "\n"
                   for i, c, g, a in requests)


def burst(n, ctx, gen):
    return trace_jsonl([(i, ctx, gen, 0.0) for i in range(n)])


def _compute(op, t, k, w, sec, jou, freq=2.0, dtype="fp16"):
    return json.dumps({"table": "compute", "op": op, "dtype": dtype, "freq_ghz": freq,
                       "axes": {"context_tokens": t, "tasks": k, "hidden_dim": w},
                       "seconds": sec, "joules": jou})


def _coll(op, devices, nodes, payload, sec, jou):
    return json.dumps({"table": "collective", "op": op,
                       "axes": {"payload_bytes": payload, "num_devices": devices,
                                "num_nodes": nodes}, "seconds": sec, "joules": jou})


def step_costs(op, t):
    return (0.0001 if op == "attention" else 0.0002) * t


def knee_costs(op, t):
    return max(0.010, 0.001 * t)


def tiny_store(ctx_knots, f=step_costs, freq=2.0):
    """test_simulator.cpp:25-46 for the 2-head toy model (attention width 16,
    swiglu width 12); joules = 10 x seconds; collectives payload*1e-12 s."""
    lines = []
    for t in ctx_knots:
        for k in (1.0, 2.0):
            lines.append(_compute("attention", t, k, 16, f("attention", t), 10 * f("attention", t), freq))
            lines.append(_compute("gemm", t, k, 12, f("gemm", t), 10 * f("gemm", t), freq))
    for kind in ("p2p", "allreduce", "allgather", "all_to_all"):
        for dev in (2, 4):
            if kind == "p2p" and dev != 2:
                continue
            for payload in (1.0, 1e9):
                lines.append(_coll(kind, dev, 1, payload, payload * 1e-12, 0.0))
    return "\n".join(lines) + "\n"


def tiny_model(layers=1):
    return dense_model(layers, 2, 2, 4, 8, 16)


def convex_task_store(task_widths):
    """test_simulator.cpp:177-205: costs convex in tasks; free collectives.
    task_widths: [(op, width)] for the model's cells."""
    def base(k):
        return 1.0 if k <= 1 else 2.2 if k <= 2 else 4.8 if k <= 4 else 10.4
    lines = []
    for t in (0.5, 1.0, 2.0, 4.0, 8.0, 16.0, 64.0, 1024.0):
        for k in (1.0, 2.0, 4.0, 8.0):
            for op, w in task_widths:
                lines.append(_compute(op, t, k, w, 1e-3 * base(k) * t, 1e-3 * base(k) * t))
    for kind in ("p2p", "allreduce", "allgather", "all_to_all"):
        for dev in (2, 4):
            if kind == "p2p" and dev != 2:
                continue
            for payload in (1.0, 1e9):
                lines.append(_coll(kind, dev, 1, payload, 0.0, 0.0))
    return "\n".join(lines) + "\n"


def crafted_store(cell_widths):
    """acceptance_main.cpp:241-306: 2x8 cluster, inter-node AllReduce 20x
    slower, compute superlinear in tokens (t^1.5)."""
    lines = []
    ctx = [0.25, 0.5] + [float(2 ** i) for i in range(14)]
    tasks = [1, 2, 4, 8, 16, 32]
    for op, w in cell_widths:
        coeff = 1e-9 if op == "attention" else 2e-9
        for t in ctx:
            for k in tasks:
                v = coeff * k * math.pow(t, 1.5)
                lines.append(_compute(op, t, k, w, v, 100 * v))
    payloads = [1, float(1 << 20), float(1 << 24), float(1 << 28), 4294967296.0]
    groups = [(2, 1, 450e9, 1e-6), (4, 1, 450e9, 1e-6), (8, 1, 450e9, 1e-6), (16, 2, 20e9, 5e-6)]
    for dev, nodes, bw, lat in groups:
        for kind in ("allreduce", "allgather", "reduce_scatter", "all_to_all"):
            factor = (dev - 1.0) / dev
            if kind == "allreduce":
                factor *= 2.0
            for p in payloads:
                s = lat + p * factor / bw
                lines.append(_coll(kind, dev, nodes, p, s, s * dev * 100))
    for p in payloads:
        lines.append(_coll("p2p", 2, 1, p, 1e-6 + p / 450e9, (1e-6 + p / 450e9) * 100))
        lines.append(_coll("p2p", 2, 2, p, 5e-6 + p / 20e9, (5e-6 + p / 20e9) * 100))
    return "\n".join(lines) + "\n"
