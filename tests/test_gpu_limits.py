"""Plans and stores beyond the first engine's fixed on-chip limits, which the
reference accepts (it has no such limits):

  * deep pipelines — one p2p boundary per stage pair (planner.cpp:330-346):
    pp64 / pp128 plans price 63 / 127 boundaries, indexed by their distinct
    p2p curves (a boundary spans 1 or 2 nodes, planner.cpp:344);
  * collective curves too large for the 96 KB shared-memory staging budget
    (staged in the unit's global region instead);

each against the compiled reference (simulate_plan through refdrv) and the
CPU restatement, bit for bit."""
import pytest

import catalog
import fixtures as fx
import pyoracle
from cases import Case, same_as_reference, same_results

pytestmark = pytest.mark.gpu
needs = pytest.mark.skipif(not pyoracle.have_refdrv(), reason="oracle/_ref/refdrv not built")

TP1 = [("tp", 1, 1), ("tp", 1, 1)]


def deep_case(layers, dp, pp, nodes, n_req=160):
    m = fx.dense_model(layers, 8, 4, 64, 1024)
    c = fx.cluster([(8, 450e9, 1e-6), (nodes, 50e9, 5e-6)], 16e9, 200e12, 2e12)
    s, t = catalog._synth(m, c, 8192, (300, 120, 60, 25, 6.0, n_req, 77))
    return Case(m, c, s, t, plans=[(dp, pp, TP1)])


@needs
@pytest.mark.parametrize("layers,dp,pp,nodes", [(128, 1, 128, 16), (64, 2, 64, 16), (96, 1, 96, 12)],
                         ids=["pp128", "dp2-pp64", "pp96"])
@pytest.mark.parametrize("mixtab", ["1", "2"], ids=["auto", "tables"])
def test_deep_pipeline_matches_reference(engine, workdir, monkeypatch, layers, dp, pp, nodes, mixtab):
    # tables: every entry gets a mixed-iteration table (stage folds of up to
    # 127 boundaries over two distinct p2p curves, psg_tables.cu)
    monkeypatch.setenv("PSG_MIXTAB", mixtab)
    monkeypatch.setenv("PSG_MIXSEL", "0" if mixtab == "2" else "1")
    case = deep_case(layers, dp, pp, nodes)
    rc, err, ref = case.reference(workdir, f"deep{layers}_{dp}_{pp}")
    assert rc == 0, err
    g = case.gpu(engine)
    same_as_reference(g, ref)
    same_results(g, case.oracle())
    assert g.entries[0]["num_iterations"] > 0


def long_curve_store(n_knots):
    """The tiny fixture store with every collective curve resampled on
    n_knots payload knots (3 doubles per knot staged per curve)."""
    lines = [l for l in fx.tiny_store([1, 4, 16, 100, 1024]).splitlines() if '"collective"' not in l]
    payloads = [1.0 + i * (1e9 / n_knots) for i in range(n_knots)]
    for kind in ("p2p", "allreduce", "allgather", "all_to_all"):
        for dev in (2, 4):
            if kind == "p2p" and dev != 2:
                continue
            for i, pl in enumerate(payloads):
                lines.append(fx._coll(kind, dev, 1, pl, pl * 1e-12 + 1e-7 * (i % 7), pl * 1e-11))
    return "\n".join(lines) + "\n"


@needs
@pytest.mark.parametrize("n_knots", [6000, 20000])
@pytest.mark.parametrize("plan", [(1, 2, TP1), (1, 1, [("tp", 1, 2), ("tp", 1, 2)])],
                         ids=["pp2-p2p", "tp2-allreduce"])
def test_curves_beyond_shared_memory_match_reference(engine, workdir, n_knots, plan):
    model = fx.tiny_model(2)
    cl = fx.cluster([(2, 1e9, 1e-6)], 1e12, 1e12, 1e12)
    reqs = [(i, 5 + (i * 37) % 90, 2 + (i * 11) % 30, 0.0004 * i) for i in range(60)]
    case = Case(model, cl, long_curve_store(n_knots), fx.trace_jsonl(reqs),
                plans=[plan])
    rc, err, ref = case.reference(workdir, f"curves{n_knots}_{plan[1]}")
    assert rc == 0, err
    g = case.gpu(engine)
    same_as_reference(g, ref)
    same_results(g, case.oracle())
