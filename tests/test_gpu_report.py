"""Report materialization: the native streaming
writers (paper_2411_17651_b200/csrc/host/report.cpp) reproduce the reference's
own output files byte for byte —
- ranked.json of `plansim search` (tools/plansim_main.cpp:128-131),
- report.json + iterations JSONL of `plansim simulate` (:166-172,
  simulator.cpp:331-385),
- the `plansim sweep` table (:184-199) —
produced here by oracle/_ref/refdrv with the CLI's recipe — every byte,
MFU/MBU included (one running tally across replicas)."""
import os

import pytest

from harness import RefCase
from test_gpu_simulate import REALISTIC
from paper_2411_17651_b200.engine import write_sweep_json

pytestmark = pytest.mark.gpu


def _same_text(ours: str, ref: str, allow_tally: bool):
    a, b = ours.split("\n"), ref.split("\n")
    assert len(a) == len(b), (len(a), len(b))
    tally_lines = 0
    for i, (x, y) in enumerate(zip(a, b)):
        if x == y:
            continue
        key = y.strip().split(":")[0]
        assert allow_tally and key in ('"mfu"', '"mbu"'), (i, x, y)
        vx, vy = float(x.split(":")[1].rstrip(",")), float(y.split(":")[1].rstrip(","))
        assert abs(vx - vy) <= 1e-9 * max(abs(vx), abs(vy)), (i, x, y)
        tally_lines += 1
    return tally_lines


@pytest.mark.parametrize("key,extra", [("c1", ()), ("c4", ()), ("c4e", ()),
                                       ("c3", ("--batching", "chunked", "--chunk", "512"))])
def test_ranked_json_matches_reference_cli(engine, workdir, tmp_path, key, extra):
    case = RefCase(key, workdir, extra=extra, out_ranked=True)
    kw = {}
    if "--batching" in extra:
        kw = dict(batching="chunked", chunk_size=512)
    res = engine.search(case.plans, case.cluster, case.store, case.trace, case.config(**kw))
    out = str(tmp_path / "ranked.json")
    res.write_ranked_json(out)
    ours, ref = open(out).read(), open(case.ranked_path).read()
    assert _same_text(ours, ref, allow_tally=False) == 0
    assert any(p["model_dp"] > 1 for p in case.plans.dicts)


@pytest.mark.parametrize("name", sorted(REALISTIC))
def test_simulate_report_and_iterations_match_reference_cli(engine, workdir, tmp_path, name):
    case = REALISTIC[name]()
    rc, err, ref, its = case.reference_iterations(workdir, "rep_" + name)
    assert rc == 0, err
    d = os.path.join(workdir, "case_rep_" + name)
    p = case.prob
    res = engine.simulate_plan(p.plans, 0, p.cluster, p.store, p.trace, case.config(), 0.0, True)
    res.write_report_json(0, str(tmp_path / "report.json"))
    res.write_iterations_jsonl(str(tmp_path / "it.jsonl"))
    dp = case.plan_specs[0][0]
    _same_text(open(tmp_path / "report.json").read(), open(os.path.join(d, "report.json")).read(),
               allow_tally=False)
    assert open(tmp_path / "it.jsonl").read() == open(os.path.join(d, "iterations.jsonl")).read()


@pytest.mark.parametrize("name,segments,subset", [("dp1_pp1", 4, 256), ("dp2_pp2", 5, 64),
                                                  ("dp1_pp2_capped", 6, 100)])
def test_sweep_table_matches_reference_cli(engine, workdir, tmp_path, name, segments, subset):
    case = REALISTIC[name]()
    rc, err, ref = case.reference_sweep(workdir, f"rsw_{name}", segments, subset)
    assert rc == 0, err
    p = case.prob
    got = engine.sweep_max_batch(p.plans, 0, p.cluster, p.store, p.trace, case.config(),
                                 segments, subset)
    write_sweep_json(got, str(tmp_path / "sweep.json"))
    ref_text = open(os.path.join(workdir, f"case_rsw_{name}", "sweep.json")).read()
    assert open(tmp_path / "sweep.json").read() == ref_text
