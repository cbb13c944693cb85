"""TTFT-SLO-constrained ranking (BASELINE.json configs[2]; the paper's
energy-under-SLO use case).  The reference's search() has
no SLO (simulator.cpp:277-294), so the expected result is derived from the
reference's own outputs: each entry's nearest-rank quantile of its
per-request TTFTs (the p95 rule of simulator.cpp:223-225) decides whether it
meets the SLO, and the expected ranking is the reference's ranking stably
partitioned into entries that meet it followed by those that miss it."""
import numpy as np
import pytest

import pyoracle
from harness import RefCase, compare_to_ref

pytestmark = pytest.mark.gpu
needs = pytest.mark.skipif(not pyoracle.have_refdrv(), reason="oracle/_ref/refdrv not built")


def nearest(values, q):
    v = np.sort(values)
    n = len(v)
    rank = int(np.ceil(q * n))
    return v[min(n - 1, rank - 1 if rank else 0)]


def expected(ref, slo, q):
    met = [len(e["per_request"]) > 0 and nearest(e["per_request"]["ttft"], q) <= slo for e in ref]
    order = [i for i in range(len(ref)) if met[i]] + [i for i in range(len(ref)) if not met[i]]
    return [ref[i] for i in order], [met[i] for i in order]


@needs
@pytest.mark.parametrize("key,slo,q", [("c3slo", 0.5, 0.99), ("c3slo", 0.2, 0.5),
                                       ("c4e", 30.0, 0.9), ("c1", 1e-9, 0.99)])
def test_slo_ranking_partitions_the_reference_ranking(engine, workdir, key, slo, q):
    case = RefCase(key, workdir)
    res = engine.search(case.plans, case.cluster, case.store, case.trace,
                        case.config(ttft_slo=slo, slo_quantile=q))
    want, met = expected(case.ref, slo, q)
    bad = compare_to_ref(res, want, tally_rtol=0.0)
    assert not bad, "\n".join(bad)
    assert list(res.entries["slo_met"] == 1) == met
    for i, e in enumerate(want):
        if len(e["per_request"]):
            assert res.entries["slo_ttft"][i] == nearest(e["per_request"]["ttft"], q)


@needs
def test_slo_off_is_the_reference_ranking(engine, workdir):
    case = RefCase("c3slo", workdir)
    res = engine.search(case.plans, case.cluster, case.store, case.trace, case.config(ttft_slo=0.0))
    assert not compare_to_ref(res, case.ref)
    assert not res.entries["slo_met"].any() and not res.entries["slo_ttft"].any()


@needs
def test_slo_ranking_matches_the_oracle_restatement(engine, workdir):
    case = RefCase("c3slo", workdir)
    cfg = case.config()
    g = engine.search(case.plans, case.cluster, case.store, case.trace, cfg)
    o = pyoracle.oracle_search(case.plans, case.cluster, case.store, case.trace, cfg)
    assert np.array_equal(g.entries["entry_index"], o.entries["entry_index"])
    assert np.array_equal(g.entries["slo_ttft"], o.entries["slo_ttft"])
    assert np.array_equal(g.entries["slo_met"], o.entries["slo_met"])
    assert 0 < int(g.entries["slo_met"].sum()) < len(g)  # the SLO splits the design space
