"""Named fixture cases re-expressed from the reference's own suites
(/root/reference/proj/tests/test_simulator.cpp, test_batching.cpp,
acceptance_main.cpp), plus seeded random batching fixtures.  Each returns a
cases.Case that the reference, the CPU oracle and the GPU engine all run."""
from __future__ import annotations

import json
import random

import fixtures as fx
from cases import Case
from paper_2411_17651_b200.host import Problem

TP1 = [("tp", 1, 1), ("tp", 1, 1)]
ONE_DEV = fx.cluster([(1, 1e9, 0.0)], 1e12, 1e12, 1e12)


def single_request():                     # test_simulator.cpp:81-104
    return Case(fx.tiny_model(), ONE_DEV, fx.tiny_store([1, 100]),
                fx.trace_jsonl([(0, 100, 2, 0.0)]), plans=[(1, 1, TP1)])


def empty_trace():                        # test_simulator.cpp:67-79
    return Case(fx.tiny_model(), ONE_DEV, fx.tiny_store([1, 100]), "", plans=[(1, 1, TP1)])


def pipeline_two_stages():                # test_simulator.cpp:106-128
    return Case(fx.tiny_model(2), fx.cluster([(2, 1e9, 1e-6)], 1e12, 1e12, 1e12),
                fx.tiny_store([1, 100]), fx.trace_jsonl([(0, 100, 2, 0.0)]), plans=[(1, 2, TP1)])


def dp2_full():                           # test_simulator.cpp:130-148
    return Case(fx.tiny_model(), fx.cluster([(2, 1e9, 0.0)], 1e12, 1e12, 1e12),
                fx.tiny_store([1, 100]), fx.burst(8, 100, 3), plans=[(2, 1, TP1)])


def dp1_half():
    return Case(fx.tiny_model(), ONE_DEV, fx.tiny_store([1, 100]), fx.burst(4, 100, 3),
                plans=[(1, 1, TP1)])


def free_collectives():                   # test_simulator.cpp:209-219
    m = fx.dense_model(4, 8, 8, 8, 24, 512)
    return Case(m, fx.cluster([(4, 1e9, 0.0)], 1e12, 1e12, 1e12),
                fx.convex_task_store([("attention", 32.0), ("gemm", 9.0)]), fx.burst(8, 64, 8),
                objective="latency", freqs=[2.0])


def _synth(model, cluster, max_ctx, trace):
    p = Problem(model, cluster).synth_store(max_ctx)
    if isinstance(trace, tuple):
        p.synth_trace(*trace)
        return p.store_jsonl(), p.trace_jsonl()
    return p.store_jsonl(), trace


def prohibitive_internode():              # test_simulator.cpp:221-245
    m = fx.dense_model(32, 32, 8, 128, 14336)
    c = fx.cluster([(8, 450e9, 1e-6), (2, 20e9, 5e-6)], 24e9, 989e12, 3.35e12)
    s, t = _synth(m, c, 16384, (2000, 600, 100, 30, 2.0, 24, 42))
    return Case(m, c, s, t, objective="latency")


def energy_vs_latency(objective, freqs):  # test_simulator.cpp:247-262
    m = fx.dense_model(8, 8, 4, 64, 1024)
    c = fx.cluster([(4, 450e9, 1e-6)], 8e9, 200e12, 2e12, (0.8, 2.0), 500)
    s, t = _synth(m, c, 8192, (400, 100, 60, 20, 4.0, 16, 5))
    return Case(m, c, s, t, objective=objective, freqs=freqs)


def _scale_seconds(jsonl, factor):
    out = []
    for line in jsonl.splitlines():
        rec = json.loads(line)
        rec["seconds"] = rec["seconds"] * factor
        out.append(json.dumps(rec))
    return "\n".join(out) + "\n"


def time_scaled(factor):                  # test_simulator.cpp:307-324, acceptance #10
    m = fx.dense_model(8, 8, 4, 64, 1024)
    c = fx.cluster([(4, 450e9, 1e-6)], 8e9, 200e12, 2e12)
    s, _ = _synth(m, c, 8192, "")
    return Case(m, c, _scale_seconds(s, factor) if factor != 1.0 else s, fx.burst(12, 500, 40))


def utilization():                        # test_simulator.cpp:326-344
    m = fx.dense_model(8, 8, 4, 64, 1024)
    c = fx.cluster([(4, 450e9, 1e-6)], 8e9, 200e12, 2e12)
    s, t = _synth(m, c, 8192, (600, 150, 80, 20, 8.0, 24, 3))
    return Case(m, c, s, t)


def fp8_model():                          # test_simulator.cpp:365-380
    m = fx.dense_model(8, 8, 4, 64, 1024, dtype="fp8")
    c = fx.cluster([(4, 450e9, 1e-6)], 8e9, 200e12, 2e12)
    s, t = _synth(m, c, 8192, (400, 100, 50, 15, 4.0, 12, 23))
    return Case(m, c, s, t)


def ttft_anchor(anchor):                  # test_simulator.cpp:382-398
    return Case(fx.tiny_model(), ONE_DEV, fx.tiny_store([1, 100]),
                fx.trace_jsonl([(0, 100, 4, 0.0), (1, 100, 4, 0.0)]), plans=[(1, 1, TP1)],
                max_batch_size=1, ttft_anchor=anchor)


def contiguous_schedule():                # test_batching.cpp:91-112
    return Case(fx.tiny_model(), ONE_DEV, fx.tiny_store([1, 100]),
                fx.trace_jsonl([(0, 100, 3, 0.0)]), plans=[(1, 1, TP1)])


def chunked_schedule():                   # test_batching.cpp:114-131
    return Case(fx.tiny_model(), ONE_DEV, fx.tiny_store([1, 100]),
                fx.trace_jsonl([(0, 100, 2, 0.0)]), plans=[(1, 1, TP1)],
                batching="chunked", chunk_size=32)


def tiny_budget_cluster(mem_bytes):
    """Tiny model on one device: kv = 32 B/token, static = 1152 B, so
    budget = 0.9*mem - 1152 bytes (planner.cpp:347-366)."""
    return fx.cluster([(1, 1e9, 0.0)], mem_bytes, 1e12, 1e12)


def overflow_eviction():                  # test_batching.cpp:143-183 (ledger in tokens x 32 B)
    # budget 3348 B = 104.6 tokens: two 40-token prompts admit, decode growth overflows
    return Case(fx.tiny_model(), tiny_budget_cluster(5000.0), fx.tiny_store([1, 100, 1024]),
                fx.trace_jsonl([(0, 40, 20, 0.0), (1, 40, 20, 0.0)]), plans=[(1, 1, TP1)])


def lone_outgrowing():                    # test_batching.cpp:185-193
    return Case(fx.tiny_model(), tiny_budget_cluster(3400.0), fx.tiny_store([1, 100, 1024]),
                fx.trace_jsonl([(0, 50, 100, 0.0)]), plans=[(1, 1, TP1)])


def crafted_2x8():                        # acceptance_main.cpp:241-306 (criteria 5 and 9)
    m = fx.dense_model(32, 32, 8, 128, 14336)
    c = fx.cluster([(8, 450e9, 1e-6), (2, 20e9, 5e-6)], 24e9, 989e12, 3.35e12)
    return Case(m, c, fx.crafted_store([("attention", 128 * 2.5), ("gemm", 3 * 14336 / 32)]),
                fx.burst(32, 2000, 100))


def random_batching(seed):
    """Seeded random traces/policies in the spirit of test_batching.cpp:195-263
    and acceptance #3, on the tiny model with a small KV budget so admission
    blocking, LIFO eviction, re-admission and rejection all occur."""
    rng = random.Random(seed)
    n = 1 + rng.randrange(30)
    t, reqs = 0.0, []
    for i in range(n):
        t += rng.randrange(6) * 0.0005
        reqs.append((i, 1 + rng.randrange(80), 1 + rng.randrange(40), t))
    mem = 1400.0 + 40.0 * rng.randrange(200)
    cfg = {}
    if rng.randrange(3) == 0:
        cfg["max_batch_size"] = 1 + rng.randrange(6)
    if rng.randrange(2):
        cfg["batching"] = "chunked"
        cfg["chunk_size"] = 1 + rng.randrange(24)
    if rng.randrange(4) == 0:
        cfg["ttft_anchor"] = "admission"
    return Case(fx.tiny_model(), tiny_budget_cluster(mem), fx.tiny_store([1, 4, 16, 100, 1024]),
                fx.trace_jsonl(reqs), plans=[(1, 1, TP1)], **cfg)


def random_batching_wide(seed):
    """Seeded traces whose batches repeatedly grow past one warp (32 slots)
    and shrink again, so the speculation kernel's lane-resident slots spill to
    the slot arrays, come back and compact lazily, under KV pressure (LIFO
    eviction, re-admission, rejection), chunked prefill and batch caps."""
    rng = random.Random(10_000 + seed)
    n = 60 + rng.randrange(90)
    grow = seed % 2 == 1  # short prompts, long generations: decode growth overflows the ledger
    t, reqs = 0.0, []
    for i in range(n):
        t += rng.randrange(3) * 0.0005
        ctx = 1 + rng.randrange(8 if grow else 60)
        gen = (20 + rng.randrange(60)) if grow else 1 + rng.randrange(60)
        reqs.append((i, ctx, gen, t))
    mem = (3000.0 + 200.0 * rng.randrange(200)) if grow else 20000.0 + 400.0 * rng.randrange(250)
    cfg = {}
    if rng.randrange(4) == 0:
        cfg["max_batch_size"] = 33 + rng.randrange(40)
    if rng.randrange(3) == 0:
        cfg["batching"] = "chunked"
        cfg["chunk_size"] = 1 + rng.randrange(48)
    if rng.randrange(4) == 0:
        cfg["ttft_anchor"] = "admission"
    return Case(fx.tiny_model(), tiny_budget_cluster(mem), fx.tiny_store([1, 4, 16, 100, 1024]),
                fx.trace_jsonl(reqs), plans=[(1, 1, TP1)], **cfg)


NAMED = {
    "single_request": single_request, "empty_trace": empty_trace,
    "pipeline_two_stages": pipeline_two_stages, "dp2_full": dp2_full, "dp1_half": dp1_half,
    "free_collectives": free_collectives, "prohibitive_internode": prohibitive_internode,
    "energy_latency": lambda: energy_vs_latency("latency", [2.0]),
    "energy_energy": lambda: energy_vs_latency("energy", [0.8, 2.0]),
    "time_scaled_1": lambda: time_scaled(1.0), "time_scaled_3.7": lambda: time_scaled(3.7),
    "utilization": utilization, "fp8_model": fp8_model,
    "ttft_arrival": lambda: ttft_anchor("arrival"), "ttft_admission": lambda: ttft_anchor("admission"),
    "contiguous_schedule": contiguous_schedule, "chunked_schedule": chunked_schedule,
    "overflow_eviction": overflow_eviction, "lone_outgrowing": lone_outgrowing,
    "crafted_2x8": crafted_2x8,
}
