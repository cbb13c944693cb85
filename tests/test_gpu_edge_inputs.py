"""Inputs the reference's search() accepts although its trace loader would
refuse them (traces.cpp:64-67): zero / negative generation lengths finish at
the prefill iteration and free ctx + 1 ledger tokens (batching.cpp:78-108).
Non-finite arrivals have no place in the clock order and are refused with a
usage error (PSG_ERR_USAGE) instead of stalling the event loop."""
import random

import numpy as np
import pytest

import catalog
import fixtures as fx
import pyoracle
from cases import Case, same_results
from paper_2411_17651_b200.errors import UsageError
from paper_2411_17651_b200.inputs import Config, Trace

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = random.Random(500 + seed)
    n = 20 + rng.randrange(40)
    t, ids, ctx, gen, arr = 0.0, [], [], [], []
    for i in range(n):
        t += rng.randrange(4) * 0.0005
        ids.append(i)
        ctx.append(1 + rng.randrange(60))
        gen.append(rng.choice([0, -3, 1, 2]) if rng.randrange(3) == 0 else 1 + rng.randrange(40))
        arr.append(t)
    mem = 1400.0 + 40.0 * rng.randrange(120)
    base = Case(fx.tiny_model(), catalog.tiny_budget_cluster(mem),
                fx.tiny_store([1, 4, 16, 100, 1024]), fx.burst(1, 10, 2), plans=[(1, 1, catalog.TP1)])
    return base, Trace(ids, ctx, gen, arr)


@pytest.mark.parametrize("seed", range(24))
def test_short_generations_match_the_oracle(engine, seed):
    case, trace = _case(seed)
    p = case.prob
    for cfg in (Config(), Config(batching="chunked", chunk_size=7), Config(max_batch_size=3)):
        g = engine.search(p.plans, p.cluster, p.store, trace, cfg)
        o = pyoracle.oracle_search(p.plans, p.cluster, p.store, trace, cfg)
        same_results(g, o)


@pytest.mark.parametrize("bad", [float("inf"), float("nan")])
def test_non_finite_arrival_is_a_usage_error(engine, bad):
    case, _ = _case(0)
    p = case.prob
    trace = Trace([0, 1], [10, 10], [4, 4], [0.0, bad])
    with pytest.raises(UsageError, match="finite"):
        engine.search(p.plans, p.cluster, p.store, trace, Config())
