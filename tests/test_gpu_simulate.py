"""simulate_plan with per-iteration records and sweep_max_batch on the engine
 against the compiled reference:
- IterationRecord stream (simulator.cpp:158-170: clock_start, duration,
  energy, batch_size, stage_seconds, stage_joules) bit-identical, replicas in
  order, and the report scalars unchanged by emission;
- SweepTable (simulator.cpp:298-329) rows bit-identical."""
import numpy as np
import pytest

import catalog
import fixtures as fx
from cases import Case, same_as_reference
from paper_2411_17651_b200.host import Problem

pytestmark = pytest.mark.gpu

SINGLE_PLAN = ["single_request", "pipeline_two_stages", "dp2_full", "dp1_half", "ttft_arrival",
               "ttft_admission", "contiguous_schedule", "chunked_schedule", "overflow_eviction",
               "lone_outgrowing"]


def _realistic(dp, pp, cells, n=160, **cfg):
    m = fx.dense_model(16, 16, 8, 128, 4096)
    c = fx.cluster([(4, 450e9, 1e-6), (2, 20e9, 5e-6)], 24e9, 989e12, 3.35e12)
    p = Problem(m, c).synth_store(16384)
    p.synth_trace(700.0, 300.0, 90.0, 40.0, 400.0, n, 11)
    return Case(m, c, p.store_jsonl(), p.trace_jsonl(), plans=[(dp, pp, cells)], **cfg)


REALISTIC = {
    "dp1_pp1": lambda: _realistic(1, 1, [("tp", 1, 8), ("tp", 2, 4)]),
    "dp2_pp2": lambda: _realistic(2, 2, [("tp", 1, 2), ("tp", 2, 1)]),
    "dp1_pp4_chunked": lambda: _realistic(1, 4, [("tp", 1, 2), ("tp", 1, 2)],
                                          batching="chunked", chunk_size=128),
    "dp1_pp2_capped": lambda: _realistic(1, 2, [("tp", 1, 4), ("tp", 2, 2)], max_batch_size=7),
}


def _check_iterations(engine, case, workdir, tag):
    rc, err, ref, its = case.reference_iterations(workdir, tag)
    p = case.prob
    cfg = case.config()
    freq = float(cfg.freqs[0]) if len(case.cfg.get("freqs", [])) else 0.0
    if rc != 0:
        with pytest.raises(Exception):
            engine.simulate_plan(p.plans, 0, p.cluster, p.store, p.trace, cfg, freq, True)
        return
    res = engine.simulate_plan(p.plans, 0, p.cluster, p.store, p.trace, cfg, freq, True)
    same_as_reference(res, ref)
    assert len(res.iterations) == len(its) == int(ref[0]["num_iterations"])
    if not its:
        return
    ref_cs = np.array([r["clock_start_s"] for r in its])
    ref_d = np.array([r["duration_s"] for r in its])
    ref_e = np.array([r["energy_j"] for r in its])
    ref_b = np.array([r["batch_size"] for r in its])
    assert np.array_equal(res.iterations["clock_start"], ref_cs)
    assert np.array_equal(res.iterations["duration"], ref_d)
    assert np.array_equal(res.iterations["energy"], ref_e)
    assert np.array_equal(res.iterations["batch_size"], ref_b)
    assert np.array_equal(res.stage_seconds, np.array([r["stage_seconds"] for r in its]))
    assert np.array_equal(res.stage_joules, np.array([r["stage_joules"] for r in its]))
    # emission does not change the report (macro-stepped run == stepwise run)
    plain = engine.simulate_plan(p.plans, 0, p.cluster, p.store, p.trace, cfg, freq, False)
    assert plain.entries.tobytes() == res.entries.tobytes()
    assert len(plain.iterations) == 0


@pytest.mark.parametrize("name", SINGLE_PLAN)
def test_iterations_named(engine, workdir, name):
    _check_iterations(engine, catalog.NAMED[name](), workdir, "it_" + name)


@pytest.mark.parametrize("name", sorted(REALISTIC))
def test_iterations_realistic(engine, workdir, name):
    _check_iterations(engine, REALISTIC[name](), workdir, "it_" + name)


@pytest.mark.parametrize("seed", range(20))
def test_iterations_random(engine, workdir, seed):
    _check_iterations(engine, catalog.random_batching(seed), workdir, f"it_rand{seed}")


def _check_sweep(engine, case, workdir, tag, segments, subset):
    rc, err, ref = case.reference_sweep(workdir, tag, segments, subset)
    assert rc == 0, err
    p = case.prob
    got = engine.sweep_max_batch(p.plans, 0, p.cluster, p.store, p.trace, case.config(),
                                 segments, subset)
    assert got["observed_max_batch"] == ref["observed_max_batch"]
    assert got["rows"] == ref["rows"]


@pytest.mark.parametrize("name,segments,subset", [
    ("dp1_pp1", 4, 256), ("dp2_pp2", 5, 64), ("dp1_pp4_chunked", 3, 40), ("dp1_pp2_capped", 6, 100)])
def test_sweep_realistic(engine, workdir, name, segments, subset):
    _check_sweep(engine, REALISTIC[name](), workdir, f"sw_{name}_{segments}", segments, subset)


@pytest.mark.parametrize("seed", range(10))
def test_sweep_random(engine, workdir, seed):
    _check_sweep(engine, catalog.random_batching(seed), workdir, f"sw_rand{seed}", 1 + seed % 5,
                 1 + 7 * seed)


def test_sweep_rejects_zero_segments(engine):
    from paper_2411_17651_b200.errors import DataError
    case = REALISTIC["dp1_pp1"]()
    p = case.prob
    with pytest.raises(DataError, match="segments must be >= 1"):
        engine.sweep_max_batch(p.plans, 0, p.cluster, p.store, p.trace, case.config(), 0)


def test_emit_requires_single_entry(engine):
    from paper_2411_17651_b200.errors import UsageError
    case = catalog.NAMED["free_collectives"]()
    p = case.prob
    with pytest.raises(UsageError):
        engine.search(p.plans, p.cluster, p.store, p.trace, case.config(emit_iterations=True))
