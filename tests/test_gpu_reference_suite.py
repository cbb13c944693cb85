"""Simulator cases of the reference's own suite (tests/test_simulator.cpp)
restated on the engine, each also compared with the compiled reference:
- :150-172 block extrapolation (every plan of the 6 rounds' models and 2-level
  cluster, synthesized tables, synth_trace);
- :272-305 batch-cap sweep known answers and SLO trade-off directions;
- :346-363 determinism (repeated and concurrent searches give identical bytes)."""
import pytest

import catalog
import fixtures as fx
import pyoracle
from cases import Case, same_as_reference
from paper_2411_17651_b200.host import Problem

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not pyoracle.have_refdrv(), reason="oracle/_ref/refdrv not built")


@needs_ref
@pytest.mark.parametrize("layers", [4, 8, 12, 16])
@pytest.mark.parametrize("round_", [0, 3, 5])
def test_block_extrapolation_configurations(engine, workdir, layers, round_):
    # test_simulator.cpp:150-172: make_dense_model(layers, 8, 4, 32, 768, 4000),
    # 2-level cluster at 1.5 GHz, GridSpec max 4096, synth_trace seed 1000 + round
    model = fx.dense_model(layers, 8, 4, 32, 768, vocab=4000)
    cluster = fx.cluster([(2, 400e9, 1e-6), (2, 40e9, 4e-6)], 32e9, 200e12, 2e12, freqs=(1.5,))
    p = Problem(model, cluster).synth_store(4096.0).synth_trace(300, 120, 40, 15, 2.0, 12,
                                                                 1000 + round_)
    case = Case(model, cluster, p.store_jsonl(), p.trace_jsonl())
    rc, err, ref = case.reference(workdir, f"blk{layers}_{round_}")
    assert rc == 0, err
    same_as_reference(case.gpu(engine), ref)


def _sweep_case():
    # tiny model, 1-device cluster, knee costs over {1,4,8,10,16,32,64,1024},
    # burst of 16 requests (ctx 1, gen 64)
    return Case(fx.tiny_model(), catalog.ONE_DEV,
                fx.tiny_store([1, 4, 8, 10, 16, 32, 64, 1024], fx.knee_costs),
                fx.burst(16, 1, 64), plans=[(1, 1, catalog.TP1)])


@needs_ref
def test_batch_cap_sweep_known_answers(engine, workdir):
    case = _sweep_case()
    p = case.prob
    t = engine.sweep_max_batch(p.plans, 0, p.cluster, p.store, p.trace, case.config(), 4, 256)
    assert t["observed_max_batch"] == 16
    caps = [r[0] for r in t["rows"]]
    assert caps[0] == 4 and caps[1] == 8 and caps[3] == 16
    tpot = [r[1] for r in t["rows"]]
    e2e = [r[3] for r in t["rows"]]
    assert tpot[1] < tpot[3]   # shrinking the cap 16 -> 8 improves TPOT
    assert e2e[0] > e2e[3]     # over-restricting to 4 hurts end-to-end latency
    uncapped = engine.simulate_plan(p.plans, 0, p.cluster, p.store, p.trace, case.config())
    assert e2e[3] == uncapped.entries[0]["e2e_latency"]
    assert tpot[3] == uncapped.entries[0]["mean_tpot"]
    one = engine.simulate_plan(p.plans, 0, p.cluster, p.store, p.trace, case.config(max_batch_size=1))
    assert all(one.entries[0]["e2e_latency"] >= x for x in e2e)
    rc, err, ref = case.reference_sweep(workdir, "known_sweep", 4, 256)
    assert rc == 0, err
    assert t["rows"] == ref["rows"] and t["observed_max_batch"] == ref["observed_max_batch"]


def test_search_is_deterministic(engine, workdir):
    case = catalog.NAMED["utilization"]()
    p = case.prob
    a = engine.search(p.plans, p.cluster, p.store, p.trace, case.config())
    b = engine.search(p.plans, p.cluster, p.store, p.trace, case.config())
    many = engine.search_many([(p.plans, p.cluster, p.store, p.trace, case.config())] * 3)
    for r in [b] + many:
        assert r.entries.tobytes() == a.entries.tobytes()
        assert r.per_request.tobytes() == a.per_request.tobytes()
        assert r.rejected_ids.tobytes() == a.rejected_ids.tobytes()
