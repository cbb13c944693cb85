"""The drop-in boundary over the reference's own C++ types: plansim_gpu::search
(paper_2411_17651_b200/csrc/shim) vs plansim::search, both called in one
process (oracle/_ref/shim_parity) on the same ExecutionPlan / Trace /
ProfileStore objects — ranked order, every SimulationReport field, per-request
metrics, rejected ids, clamp warnings and exception parity."""
import json
import os
import subprocess

import pytest

import pyoracle
from paper_2411_17651_b200.workloads import WORKLOADS

pytestmark = pytest.mark.gpu
SHIM = os.path.join(os.path.dirname(pyoracle.REFDRV), "shim_parity")
needs = pytest.mark.skipif(not os.path.exists(SHIM), reason="oracle/_ref/shim_parity not built")


def run(args):
    p = subprocess.run([SHIM] + [str(a) for a in args], capture_output=True, text=True, timeout=900)
    line = next((json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")), None)
    return p.returncode, line, p.stderr


CASES = [
    ("c1", []),
    ("c4", ["--jobs", "4"]),
    ("c4e", ["--jobs", "4"]),
    ("c3", ["--batching", "chunked", "--chunk", "512", "--jobs", "4"]),
    ("c1", ["--max-batch", "3", "--anchor", "admission"]),
]


@needs
@pytest.mark.parametrize("key,extra", CASES, ids=[k + "".join(e) for k, e in CASES])
def test_drop_in_search_matches_reference(workdir, key, extra):
    w = WORKLOADS[key]
    args = w.refdrv_args(w.materialize(os.path.join(workdir, "shim_" + key))) + extra
    rc, line, err = run(args)
    assert rc == 0, (line, err)
    assert line["mismatches"] == 0


@needs
def test_drop_in_clamp_warnings_match(workdir):
    # a 4096-token grid clamps every longer prompt: warnings must match
    w = WORKLOADS["c1"]
    args = w.refdrv_args(w.materialize(os.path.join(workdir, "shim_clamp")))
    args[args.index("--synth-profiles") + 1] = "256"
    rc, line, err = run(args)
    assert rc == 0, (line, err)
    assert line["warnings"] > 0


@needs
def test_drop_in_raises_the_reference_data_error(workdir):
    w = WORKLOADS["c1"]
    args = w.refdrv_args(w.materialize(os.path.join(workdir, "shim_err"))) + ["--drop-table", "gemm"]
    rc, line, err = run(args)
    assert rc == 4 and line["error_parity"], (line, err)


SINGLE = [
    ("c1", ["--single", "0", "--sweep-segments", "4", "--sweep-subset", "200"]),
    ("c1", ["--single", "7", "--sweep-segments", "5", "--sweep-subset", "64",
            "--batching", "chunked", "--chunk", "96"]),
    ("c4", ["--single", "3", "--sweep-segments", "3", "--sweep-subset", "128"]),
    ("c3", ["--single", "5", "--sweep-segments", "2", "--sweep-subset", "300"]),
]


@needs
@pytest.mark.parametrize("key,extra", SINGLE, ids=[k + "".join(e) for k, e in SINGLE])
def test_drop_in_simulate_plan_iterations_and_sweep(workdir, key, extra):
    """plansim_gpu::simulate_plan with emit_iterations (every IterationRecord)
    and plansim_gpu::sweep_max_batch (every SweepRow) vs the reference."""
    w = WORKLOADS[key]
    args = w.refdrv_args(w.materialize(os.path.join(workdir, "shim1_" + key))) + extra
    rc, line, err = run(args)
    assert rc == 0, (line, err)
    assert line["mismatches"] == 0, line
    assert line["iterations"] > 0 and line["sweep_rows"] > 0


SHARDED = [
    ("c4", "2", "2"),    # 140 entries over two contexts
    ("c3", "4", "4"),    # 104 entries over four contexts
    ("c4e", "8", "3"),   # more jobs than contexts: min(jobs, contexts)
]


@needs
@pytest.mark.parametrize("key,jobs,per_dev", SHARDED, ids=[f"{k}-j{j}-c{c}" for k, j, c in SHARDED])
def test_drop_in_jobs_shard_over_contexts(workdir, key, jobs, per_dev):
    """jobs -> devices: entries sharded longest-first over several engine
    contexts (here several on the one device of the box), merged by the device
    ranking — the same RankedPlans as the reference's search with `jobs`
    threads (simulator.cpp:251-275)."""
    w = WORKLOADS[key]
    args = w.refdrv_args(w.materialize(os.path.join(workdir, "shimj_" + key))) + ["--jobs", jobs]
    env = dict(os.environ, PSG_SHIM_CONTEXTS_PER_DEVICE=per_dev)
    p = subprocess.run([SHIM] + [str(a) for a in args], capture_output=True, text=True,
                       timeout=900, env=env)
    line = next((json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")), None)
    assert p.returncode == 0, (line, p.stderr)
    assert line["mismatches"] == 0, line


@needs
def test_drop_in_is_safe_for_concurrent_callers(workdir):
    """Four threads call plansim_gpu::search at once (one cached context per
    device, locked per call): each gets the single caller's result."""
    w = WORKLOADS["c1"]
    args = w.refdrv_args(w.materialize(os.path.join(workdir, "shimt"))) + ["--threads", "4"]
    rc, line, err = run(args)
    assert rc == 0, (line, err)
    assert line["mismatches"] == 0, line
