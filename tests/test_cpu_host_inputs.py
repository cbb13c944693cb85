"""The native host side reproduces the reference's inputs exactly: plan sets
(generate_plans, every ExecutionPlan field), synthesized profile tables
(serialize() byte-identical) and traces (serialize_trace byte-identical) —
against the compiled reference driver, plus loader error behaviour."""
import json
import os

import pytest

import fixtures as fx
import pyoracle
from paper_2411_17651_b200.errors import DataError, InfeasibleError
from paper_2411_17651_b200.host import Problem, problem_for
from paper_2411_17651_b200.workloads import WORKLOADS

needs_ref = pytest.mark.skipif(not pyoracle.have_refdrv(), reason="oracle/_ref not built")


def ref_dumps(workdir, tag, model, cluster, extra):
    d = os.path.join(workdir, "host_" + tag)
    os.makedirs(d, exist_ok=True)
    mp, cp = os.path.join(d, "model.json"), os.path.join(d, "cluster.json")
    open(mp, "w").write(model)
    open(cp, "w").write(cluster)
    args = ["--model", mp, "--cluster", cp] + extra
    rc, _, err = pyoracle.refdrv(["synth"] + args + ["--out-store", d + "/store.jsonl",
                                                      "--out-trace", d + "/trace.jsonl"])
    assert rc == 0, err
    rc, _, err = pyoracle.refdrv(["search"] + args + ["--plans", "0:1000000", "--no-search",
                                                       "--out-plans", d + "/plans.json"])
    return d, rc, err


FIXTURE_PROBLEMS = {
    "dense_2level": (fx.dense_model(16, 8, 4, 64, 1024), fx.cluster([(2, 400e9, 1e-6), (2, 40e9, 4e-6)],
                                                                    32e9, 200e12, 2e12, (1.5,))),
    "moe_1node": (fx.moe_model(16, 8, 4, 64, 1024, 8, 2), fx.cluster([(8, 450e9, 1e-6)], 80e9,
                                                                      100e12, 2e12, (1.0, 2.0), 500)),
    "gpt_mlp_3level": (fx.dense_model(12, 12, 12, 64, 3072, ffn="gelu"),
                       fx.cluster([(4, 450e9, 1e-6), (2, 50e9, 5e-6), (2, 25e9, 9e-6)], 40e9, 300e12, 2e12)),
    "fp8_dense": (fx.dense_model(8, 8, 4, 64, 1024, dtype="fp8"), fx.cluster([(4, 450e9, 1e-6)], 8e9, 200e12, 2e12)),
}


@needs_ref
@pytest.mark.parametrize("key", ["c1", "c2", "c2fp8", "c3", "c4", "c5_1k", "c5", "c5fp8dvfs"])
def test_workload_inputs_match_reference(workdir, key):
    w = WORKLOADS[key]
    prob = problem_for(w)
    extra = w.refdrv_args(w.materialize(os.path.join(workdir, "wl_" + key)))
    model, cluster = w.model_json, w.cluster
    d, rc, err = ref_dumps(workdir, key, model, cluster, extra[4:])
    assert rc == 0, err
    assert open(d + "/store.jsonl").read() == prob.store_jsonl()
    assert open(d + "/trace.jsonl").read() == prob.trace_jsonl()
    assert json.loads(open(d + "/plans.json").read()) == json.loads(prob.plans_json())


@needs_ref
@pytest.mark.parametrize("key", sorted(FIXTURE_PROBLEMS))
def test_fixture_plans_and_tables_match_reference(workdir, key):
    model, cluster = FIXTURE_PROBLEMS[key]
    extra = ["--synth-profiles", "8192", "--synth-trace", "300,120,40,15,2,12,1000"]
    d, rc, err = ref_dumps(workdir, key, model, cluster, extra)
    prob = Problem(model, cluster).synth_store(8192).synth_trace(300, 120, 40, 15, 2, 12, 1000)
    assert open(d + "/store.jsonl").read() == prob.store_jsonl()
    assert open(d + "/trace.jsonl").read() == prob.trace_jsonl()
    if rc == 3:  # reference: InfeasibleError
        with pytest.raises(InfeasibleError):
            prob.generate_plans()
        return
    assert rc == 0, err
    prob.generate_plans()
    assert json.loads(open(d + "/plans.json").read()) == json.loads(prob.plans_json())


def test_store_round_trip_is_byte_identical():
    prob = problem_for(WORKLOADS["c1"])
    text = prob.store_jsonl()
    again = Problem(WORKLOADS["c1"].model_json, WORKLOADS["c1"].cluster).load_store(text)
    assert again.store_jsonl() == text


def test_trace_load_sorts_by_arrival_and_accepts_aliases():
    prob = Problem(fx.tiny_model(), fx.cluster([(1, 1e9, 0)], 1e12, 1e12, 1e12))
    prob.load_trace('{"ContextTokens": 5, "GeneratedTokens": 2, "TIMESTAMP": 3.0}\n'
                    '{"id": 7, "context_len": "4", "gen_len": 1, "arrival_s": 1.0}\n')
    lines = [json.loads(x) for x in prob.trace_jsonl().splitlines()]
    assert [l["id"] for l in lines] == [7, 0]
    assert lines[1]["context_len"] == 5


@pytest.mark.parametrize("bad,match", [
    ('{"table":"unknown","axes":{},"seconds":1,"joules":1}', "unknown table kind"),
    ('{"table":"compute","op":"gemm","dtype":"fp16","freq_ghz":1,"axes":{"context_tokens":1,'
     '"tasks":1,"hidden_dim":1},"seconds":-1,"joules":1}', "negative"),
    ('{"table":"collective","op":"allreduce","axes":{"payload_bytes":1,"num_devices":1,'
     '"num_nodes":1},"seconds":1,"joules":1}', "< 2 devices"),
])
def test_store_loader_rejects_bad_tables(bad, match):
    prob = Problem(fx.tiny_model(), fx.cluster([(1, 1e9, 0)], 1e12, 1e12, 1e12))
    with pytest.raises(DataError, match=match):
        prob.load_store(bad + "\n")


def test_incomplete_grid_and_duplicates_rejected():
    prob = Problem(fx.tiny_model(), fx.cluster([(1, 1e9, 0)], 1e12, 1e12, 1e12))
    rec = lambda t, k, s: json.dumps({"table": "compute", "op": "gemm", "dtype": "fp16", "freq_ghz": 1.0,
                                      "axes": {"context_tokens": t, "tasks": k, "hidden_dim": 64},
                                      "seconds": s, "joules": s})
    with pytest.raises(DataError, match="complete grid"):
        prob.load_store(rec(512, 4, 0.01) + "\n" + rec(1024, 8, 0.02) + "\n")
    with pytest.raises(DataError, match="duplicate"):
        prob.load_store(rec(512, 4, 0.01) + "\n" + rec(512, 4, 0.02) + "\n")


def test_model_config_validation():
    with pytest.raises(DataError, match="hidden_size"):
        Problem(json.dumps({"num_hidden_layers": 2, "hidden_size": 10, "num_attention_heads": 4,
                            "intermediate_size": 8, "vocab_size": 10}),
                fx.cluster([(1, 1e9, 0)], 1e12, 1e12, 1e12))
    with pytest.raises(DataError, match="missing required key"):
        Problem(json.dumps({"hidden_size": 8}), fx.cluster([(1, 1e9, 0)], 1e12, 1e12, 1e12))


def test_infeasible_model_raises():
    big = fx.dense_model(80, 64, 8, 128, 28672, vocab=128256)
    prob = Problem(big, fx.cluster([(1, 1e9, 0)], 1e9, 1e12, 1e12))
    with pytest.raises(InfeasibleError):
        prob.generate_plans()
