"""GPU engine vs the pinned CPU oracle on every named reference fixture and on
seeded random batching fixtures (admission blocking, LIFO eviction,
re-admission, rejection, chunked prefill, batch caps, both TTFT anchors);
error parity with the reference; clamp reporting; entry sharding; device
ranking."""
import json

import numpy as np
import pytest

import catalog
import fixtures as fx
from cases import Case, same_results
from paper_2411_17651_b200.errors import DataError, InfeasibleError
from paper_2411_17651_b200.inputs import Config, Plans

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", sorted(catalog.NAMED))
def test_engine_matches_oracle_on_fixture(engine, name):
    case = catalog.NAMED[name]()
    same_results(case.gpu(engine), case.oracle(), tally_rtol=0.0)


@pytest.mark.parametrize("seed", range(200))
def test_engine_matches_oracle_on_random_batching(engine, seed):
    case = catalog.random_batching(seed)
    g = case.gpu(engine)
    same_results(g, case.oracle())
    e = g.entries[0]
    assert e["num_completed"] + e["num_rejected"] == len(case.prob.trace)


@pytest.mark.parametrize("spec", ["1", "0"])
@pytest.mark.parametrize("seed", range(40))
def test_engine_matches_oracle_on_wide_batches(engine, monkeypatch, seed, spec):
    """Batches crossing 32 slots both ways: the speculation kernel's
    lane-resident slots (spill / fill / lazy compaction) and the plain
    kernel's slot arrays give the oracle's results."""
    monkeypatch.setenv("PSG_SPECULATE", spec)
    case = catalog.random_batching_wide(seed)
    g = case.gpu(engine)
    same_results(g, case.oracle())
    e = g.entries[0]
    assert e["num_completed"] + e["num_rejected"] == len(case.prob.trace)


def test_known_answers_on_device(engine):
    e = catalog.single_request().gpu(engine).entries[0]
    assert abs(e["e2e_latency"] - 0.0303) <= 1e-12 * 0.0303
    assert abs(e["total_energy"] - 0.303) <= 1e-12 * 0.303
    r = catalog.free_collectives().gpu(engine)
    assert r.encoding(0) == "dp1:pp1:MHA-tp4x1:SwiGLU-tp4x1"
    assert catalog.chunked_schedule().gpu(engine).entries[0]["num_iterations"] == 5


def test_missing_table_is_a_data_error_with_the_reference_message(engine):
    case = catalog.single_request()
    store = "\n".join(l for l in case.store_jsonl.splitlines() if '"gemm"' not in l) + "\n"
    bad = Case(case.model, case.cluster_json, store, case.trace_jsonl, plans=[(1, 1, catalog.TP1)])
    with pytest.raises(DataError, match="no compute table for op=gemm dtype=fp16 freq=2 GHz"):
        bad.gpu(engine)


def test_missing_table_unused_when_every_request_is_rejected(engine):
    # the reference only throws when an iteration queries the table
    case = catalog.lone_outgrowing()
    store = "\n".join(l for l in case.store_jsonl.splitlines() if '"gemm"' not in l) + "\n"
    huge = fx.trace_jsonl([(0, 100000, 5, 0.0)])
    c = Case(case.model, case.cluster_json, store, huge, plans=[(1, 1, catalog.TP1)])
    e = c.gpu(engine).entries[0]
    assert e["num_rejected"] == 1 and e["num_iterations"] == 0


def test_chunked_with_zero_chunk_is_a_data_error(engine):
    case = catalog.chunked_schedule()
    with pytest.raises(DataError, match="chunk_size >= 1"):
        case.gpu(engine, chunk_size=0)


def test_empty_plan_list_is_infeasible(engine):
    case = catalog.single_request()
    empty = Plans([])
    with pytest.raises(InfeasibleError):
        engine.search(empty, case.prob.cluster, case.prob.store, case.prob.trace, Config())


def test_clamped_queries_are_flagged(engine):
    # tiny store spans ctx [1, 100]: a 300-token prompt clamps above
    case = Case(fx.tiny_model(), catalog.ONE_DEV, fx.tiny_store([1, 100]),
                fx.trace_jsonl([(0, 300, 2, 0.0)]), plans=[(1, 1, catalog.TP1)])
    r = case.gpu(engine)
    assert (r.compute_clamp & 2).any()          # context axis, above
    assert not (r.compute_clamp & 1).any()


def test_entry_subset_matches_full_search(engine):
    case = catalog.utilization()
    full = case.gpu(engine, rank=False)
    n = len(full)
    parts = [list(range(0, n, 2)), list(range(1, n, 2))]
    for sub in parts:
        r = case.gpu(engine, rank=False, entry_subset=sub)
        assert list(r.entries["entry_index"]) == sub
        for k, e in enumerate(sub):
            for f in ("e2e_latency", "total_energy", "num_iterations", "p95_latency"):
                assert r.entries[k][f] == full.entries[e][f]
            assert np.array_equal(r.report(k)[0], full.report(e)[0])


def test_device_rank_keys_match_search_order(engine):
    case = catalog.utilization()
    ranked = case.gpu(engine)
    unranked = case.gpu(engine, rank=False)
    enc = case.prob.plans.struct.enc_rank
    keys = np.zeros(len(unranked), dtype=[("num_rejected", "<i8"), ("objective_metric", "<f8"),
                                          ("other_metric", "<f8"), ("enc_rank", "<i4"),
                                          ("pad_", "<i4"), ("freq_ghz", "<f8"), ("entry_index", "<i8")])
    ent = unranked.entries
    keys["num_rejected"] = ent["num_rejected"]
    keys["objective_metric"] = ent["e2e_latency"]
    keys["other_metric"] = ent["total_energy"]
    keys["enc_rank"] = [enc[int(p)] for p in ent["plan_index"]]
    keys["freq_ghz"] = ent["freq_ghz"]
    keys["entry_index"] = ent["entry_index"]
    perm = np.random.default_rng(0).permutation(len(keys))
    order = engine.rank_keys(keys[perm])
    assert list(keys[perm][order]["entry_index"]) == list(ranked.entries["entry_index"])


def test_repeated_request_ids_are_rejected(engine):
    """The reference keys per-request state by id (simulator.cpp:103-110); a
    trace that repeats an id has no reproducible result, so the engine refuses
    it loudly instead of guessing."""
    from paper_2411_17651_b200.errors import UsageError
    case = catalog.Case(fx.tiny_model(), catalog.ONE_DEV, fx.tiny_store([1, 100]),
                        fx.trace_jsonl([(0, 10, 2, 0.0), (1, 10, 2, 0.0), (0, 12, 3, 0.1)]),
                        plans=[(1, 1, catalog.TP1)])
    with pytest.raises(UsageError, match="ids must be unique"):
        case.gpu(engine)
