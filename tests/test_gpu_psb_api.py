"""The native C++ host API (include/psb/plansim_b200.hpp: psb::search,
psb::simulate_plan with emit_iterations, psb::sweep_max_batch), driven by
tests/native/psb_api_check.cpp, agrees exactly with the Python front end over
the same C ABI — whose results the other GPU tests pin to the reference."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2411_17651_b200.engine import Engine
from paper_2411_17651_b200.host import Problem
from paper_2411_17651_b200.inputs import Config
from paper_2411_17651_b200.workloads import WORKLOADS

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(REPO, "paper_2411_17651_b200")


def _fnv(h, v):
    b = int(np.float64(v).view(np.uint64))
    return ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF


@pytest.mark.parametrize("key,plan_k,segments,subset", [("c1", 3, 4, 300), ("c4", 1, 3, 64)])
def test_psb_api_matches_engine(tmp_path, engine, key, plan_k, segments, subset):
    exe = tmp_path / "psb_api_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(REPO, "include"),
                    os.path.join(REPO, "tests", "native", "psb_api_check.cpp"), "-L", PKG, "-lpsg",
                    f"-Wl,-rpath,{PKG}", "-o", str(exe)], check=True)
    w = WORKLOADS[key]
    paths = w.materialize(str(tmp_path / key))
    kind, params = w.trace
    assert kind == "synth"
    out = subprocess.run([str(exe), paths["model"], paths["cluster"], repr(w.max_context),
                          ",".join(repr(float(x)) for x in params), str(plan_k), str(segments),
                          str(subset)], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr
    got = json.loads(out.stdout.strip().splitlines()[-1])

    prob = Problem(w.model_json, w.cluster).synth_store(w.max_context).synth_trace(*params)
    prob.generate_plans()
    res = engine.search(prob.plans, prob.cluster, prob.store, prob.trace, Config())
    assert got["entries"] == len(res)
    assert got["best_plan"] == int(res.entries[0]["plan_index"])
    assert float.fromhex(got["best_e2e"]) == res.entries[0]["e2e_latency"]

    sim = engine.simulate_plan(prob.plans, plan_k, prob.cluster, prob.store, prob.trace,
                               Config(), 0.0, True)
    assert float.fromhex(got["sim_e2e"]) == sim.entries[0]["e2e_latency"]
    assert got["sim_iterations"] == int(sim.entries[0]["num_iterations"]) == got["records"]
    h = 1469598103934665603
    for k, it in enumerate(sim.iterations):
        for v in (it["clock_start"], it["duration"], it["energy"], float(it["batch_size"])):
            h = _fnv(h, v)
        for v in sim.stage_seconds[k]:
            h = _fnv(h, v)
        for v in sim.stage_joules[k]:
            h = _fnv(h, v)
    assert got["records_hash"] == f"{h:016x}"

    sw = engine.sweep_max_batch(prob.plans, plan_k, prob.cluster, prob.store, prob.trace,
                                Config(), segments, subset)
    assert got["observed"] == sw["observed_max_batch"]
    assert [(r[0], float.fromhex(r[1]), float.fromhex(r[2]), float.fromhex(r[3]))
            for r in got["rows"]] == sw["rows"]
