"""Seeded random realistic search problems, engine vs the compiled reference
(oracle/_ref/refdrv), every field bit for bit.  Complements the tiny-model
batching fixtures: real planner output (dense and MoE, fp16 / fp8), synthesized
profile tables with clamping, 1-2 level clusters, DVFS frequencies, lognormal
traces, both objectives, chunked prefill, batch caps and TTFT anchors."""
import json
import math
import random

import pytest

import pyoracle
from cases import Case, same_as_reference
from paper_2411_17651_b200.host import Problem

pytestmark = pytest.mark.gpu


def _model(rng):
    layers = rng.choice([4, 8, 12, 16])
    hidden = rng.choice([1024, 2048, 4096])
    heads = rng.choice([8, 16, 32])
    kv = rng.choice([h for h in (1, 2, 4, 8) if heads % h == 0])
    m = {"name": "fuzz", "num_hidden_layers": layers, "hidden_size": hidden,
         "num_attention_heads": heads, "num_key_value_heads": kv,
         "intermediate_size": hidden * rng.choice([2, 3, 4]), "vocab_size": 32000,
         "torch_dtype": rng.choice(["fp16", "fp16", "fp8"]), "hidden_act": "silu"}
    if rng.random() < 0.35:
        m["num_local_experts"] = rng.choice([4, 8, 16])
        m["num_experts_per_tok"] = rng.choice([1, 2])
    return m


def _cluster(rng, tight=False):
    leaf = rng.choice([2, 4, 8])
    levels = [{"fan_out": leaf, "link_bandwidth_bytes_per_s": 450e9, "link_latency_s": 1e-6}]
    if rng.random() < 0.5:
        levels.append({"fan_out": rng.choice([2, 3]), "link_bandwidth_bytes_per_s": 50e9,
                       "link_latency_s": 5e-6})
    freqs = sorted(rng.sample([0.8, 1.2, 1.6, 2.0], rng.choice([1, 2, 3])))
    mem = rng.choice([2.5e9, 4e9, 6e9]) if tight else rng.choice([16e9, 40e9, 80e9])
    dev = {"name": "fuzz-gpu", "memory_capacity_bytes": mem,
           "peak_flops": {"fp16": 989e12, "fp8": 1979e12},
           "peak_mem_bandwidth_bytes_per_s": 3.35e12, "frequency_options_ghz": freqs,
           "tdp_watts": 700}
    return json.dumps({"levels": levels, "device": dev}), freqs


def _trace(rng, n):
    t, lines = 0.0, []
    rate = rng.choice([2.0, 20.0, 200.0])
    for i in range(n):
        t += rng.expovariate(rate)
        ctx = max(1, round(rng.lognormvariate(math.log(rng.choice([64, 512, 2048])), 0.8)))
        gen = max(1, round(rng.lognormvariate(math.log(rng.choice([16, 128])), 0.7)))
        lines.append(json.dumps({"id": i, "context_len": ctx, "gen_len": gen, "arrival_s": t}))
    return "\n".join(lines) + "\n"


def make_case(seed, tight=False):
    """tight: device memory close to the weights' footprint, so KV budgets are
    small — admission blocking, LIFO eviction and rejection under real plans."""
    rng = random.Random(seed)
    model = _model(rng)
    cluster, freqs = _cluster(rng, tight)
    prob = Problem(json.dumps(model), cluster)
    prob.synth_store(rng.choice([4096.0, 32768.0]))  # small grids clamp long prompts
    cfg = {"objective": rng.choice(["latency", "energy"])}
    if len(freqs) > 1 and rng.random() < 0.7:
        cfg["freqs"] = freqs
    if rng.random() < 0.4:
        cfg["batching"] = "chunked"
        cfg["chunk_size"] = rng.choice([16, 128, 512])
    if rng.random() < 0.3:
        cfg["max_batch_size"] = rng.choice([2, 8, 32])
    if rng.random() < 0.3:
        cfg["ttft_anchor"] = "admission"
    return Case(json.dumps(model), cluster, prob.store_jsonl(), _trace(rng, rng.choice([60, 200, 400])),
                **cfg)


@pytest.mark.skipif(not pyoracle.have_refdrv(), reason="oracle/_ref/refdrv not built")
@pytest.mark.parametrize("seed,tight", [(s, False) for s in range(24)] + [(s, True) for s in range(100, 140)])
def test_fuzz_search_matches_reference(engine, workdir, seed, tight):
    try:
        case = make_case(seed, tight)
    except Exception as e:  # the planner finds no plan that fits: both sides must agree
        pytest.skip(f"no feasible plan for this random cluster/model: {e}")
    rc, err, ref = case.reference(workdir, f"fuzz{seed}{'t' if tight else ''}")
    if rc != 0:
        with pytest.raises(Exception):
            case.gpu(engine)
        return
    same_as_reference(case.gpu(engine), ref)


@pytest.mark.skipif(not pyoracle.have_refdrv(), reason="oracle/_ref/refdrv not built")
@pytest.mark.parametrize("seed", range(100, 112))
def test_fuzz_tight_small_tally_logs(engine, workdir, monkeypatch, seed):
    """Memory-tight random problems (evictions, re-admissions) with replica
    groups whose tally logs hold one record per request: the replicas whose
    logs overflow make the search rerun chained — bit-exact either way."""
    monkeypatch.setenv("PSG_CHAIN_REPLICAS", "2")
    monkeypatch.setenv("PSG_RLOG_PER_REQ", "1")
    try:
        case = make_case(seed, True)
    except Exception as e:
        pytest.skip(f"no feasible plan for this random cluster/model: {e}")
    rc, err, ref = case.reference(workdir, f"fuzz{seed}t")
    if rc != 0:
        with pytest.raises(Exception):
            case.gpu(engine)
        return
    same_as_reference(case.gpu(engine), ref)
