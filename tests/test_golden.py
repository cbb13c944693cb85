"""Committed golden vectors (tests/golden/*.json, made by make_golden.py from
the compiled reference) vs the CPU restatement oracle (CPU) and the GPU
engine (GPU).  Inputs are built by the native host library, which is proven
identical to the reference's own inputs in test_cpu_host_inputs.py."""
import hashlib
import json
import os

import numpy as np
import pytest

import catalog
import pyoracle
from paper_2411_17651_b200.host import problem_for
from paper_2411_17651_b200.inputs import Config
from paper_2411_17651_b200.workloads import WORKLOADS

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = sorted(f[:-5] for f in os.listdir(GOLDEN) if f.endswith(".json"))
FAST_CONFIGS = {"config_c1", "config_c4e"}  # CPU oracle budget (the others run on GPU)


def load(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)["entries"]


def run(name, engine=None):
    if name.startswith("config_"):
        w = WORKLOADS[name[len("config_"):]]
        prob = problem_for(w)
        cfg = Config(objective=w.objective, freqs=w.freqs)
        args = (prob.plans, prob.cluster, prob.store, prob.trace, cfg)
        return engine.search(*args) if engine else pyoracle.oracle_search(*args)
    case = catalog.NAMED[name]()
    return case.gpu(engine) if engine else case.oracle()


def check(res, golden, tally_rtol):
    assert len(res) == len(golden)
    for k, g in enumerate(golden):
        e = res.entries[k]
        assert res.encoding(k) == g["encoding"], k
        for f in ("plan_index", "num_completed", "num_rejected", "num_iterations", "max_batch_observed"):
            assert int(e[f]) == g[f], (k, f)
        for f in ("freq_ghz", "e2e_latency", "total_energy", "p95_latency", "mean_ttft", "mean_tpot"):
            assert float(e[f]) == float.fromhex(g[f]), (k, f, float(e[f]), float.fromhex(g[f]))
        for f in ("mfu", "mbu"):
            want = float.fromhex(g[f])
            assert np.isclose(float(e[f]), want, rtol=tally_rtol, atol=0), (k, f)
        pr, rj = res.report(k)
        assert hashlib.sha256(np.ascontiguousarray(pr).tobytes()).hexdigest() == g["per_request_sha256"], k
        assert hashlib.sha256(np.ascontiguousarray(rj).tobytes()).hexdigest() == g["rejected_sha256"], k


@pytest.mark.parametrize("name", [n for n in NAMES if not n.startswith("config_") or n in FAST_CONFIGS])
def test_oracle_matches_golden(name):
    check(run(name), load(name), tally_rtol=0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_engine_matches_golden(engine, name):
    check(run(name, engine), load(name), tally_rtol=0.0)
