"""Fixture cases runnable by all three engines on identical inputs:
the compiled reference (refdrv), the CPU restatement oracle and the GPU engine."""
from __future__ import annotations

import json
import os

import numpy as np

import pyoracle
from harness import SCALARS
from paper_2411_17651_b200.host import Problem
from paper_2411_17651_b200.inputs import Config


class Case:
    def __init__(self, model, cluster, store, trace, plans=None, **cfg):
        """plans: None -> generate_plans; else [(dp, pp, [(mode, cdp, intra), ...]), ...]"""
        self.model, self.cluster_json, self.store_jsonl, self.trace_jsonl = model, cluster, store, trace
        self.plan_specs = plans
        self.cfg = cfg
        self.prob = Problem(model, cluster).load_store(store).load_trace(trace)
        if plans is None:
            self.prob.generate_plans()
        else:
            for dp, pp, cells in plans:
                self.prob.build_plan(dp, pp, cells)

    def config(self, **kw):
        c = dict(self.cfg)
        c.update(kw)
        return Config(**c)

    def oracle(self, **kw):
        p = self.prob
        return pyoracle.oracle_search(p.plans, p.cluster, p.store, p.trace, self.config(**kw))

    def gpu(self, engine, **kw):
        p = self.prob
        return engine.search(p.plans, p.cluster, p.store, p.trace, self.config(**kw))

    def _ref_args(self, workdir, tag):
        d = os.path.join(workdir, "case_" + tag)
        os.makedirs(d, exist_ok=True)
        files = {}
        for name, text in (("model.json", self.model), ("cluster.json", self.cluster_json),
                           ("store.jsonl", self.store_jsonl), ("trace.jsonl", self.trace_jsonl)):
            files[name] = os.path.join(d, name)
            with open(files[name], "w") as f:
                f.write(text)
        args = ["--model", files["model.json"], "--cluster", files["cluster.json"],
                "--profiles", files["store.jsonl"], "--trace", files["trace.jsonl"],
                "--out-result", os.path.join(d, "ref.bin")]
        c = self.cfg
        if c.get("objective"):
            args += ["--objective", c["objective"]]
        if c.get("freqs"):
            args += ["--freqs", ",".join(repr(float(x)) for x in c["freqs"])]
        if c.get("batching"):
            args += ["--batching", c["batching"]]
        if "chunk_size" in c:
            args += ["--chunk", c["chunk_size"]]
        if c.get("max_batch_size"):
            args += ["--max-batch", c["max_batch_size"]]
        if c.get("ttft_anchor"):
            args += ["--anchor", c["ttft_anchor"]]
        return d, args

    def _plan_spec(self):
        assert self.plan_specs is not None and len(self.plan_specs) == 1, \
            "reference simulate runs one plan"
        dp, pp, cells = self.plan_specs[0]
        return ",".join([str(dp), str(pp)] + [f"{m}:{a}:{b}" for m, a, b in cells])

    def reference(self, workdir, tag):
        """Runs the compiled reference on the same files; returns its entries."""
        d, args = self._ref_args(workdir, tag)
        if self.plan_specs is None:
            rc, line, err = pyoracle.refdrv(["search"] + args + ["--jobs", "1"])
        else:
            rc, line, err = pyoracle.refdrv(["simulate"] + args + ["--plan-spec", self._plan_spec()])
        return rc, err, (pyoracle.read_refdump(os.path.join(d, "ref.bin"))[0] if rc == 0 else None)

    def reference_iterations(self, workdir, tag):
        """simulate_plan with emit_iterations (iterations_to_jsonl records);
        the CLI's report / JSONL / summary files are left in case_<tag>/."""
        d, args = self._ref_args(workdir, tag)
        path = os.path.join(d, "iterations.jsonl")
        rc, line, err = pyoracle.refdrv(["simulate"] + args + ["--plan-spec", self._plan_spec(),
                                                               "--emit-iterations", path,
                                                               "--out-report",
                                                               os.path.join(d, "report.json"),
                                                               "--out-summary",
                                                               os.path.join(d, "summary.txt")])
        if rc != 0:
            return rc, err, None, None
        with open(path) as f:
            its = [json.loads(x) for x in f if x.strip()]
        return rc, err, pyoracle.read_refdump(os.path.join(d, "ref.bin"))[0], its

    def reference_sweep(self, workdir, tag, segments, subset):
        """sweep_max_batch: (observed_max_batch, [(cap, mean_tpot, mean_ttft, e2e)])."""
        d, args = self._ref_args(workdir, tag)
        rc, line, err = pyoracle.refdrv(["sweep"] + args + ["--plan-spec", self._plan_spec(),
                                                            "--segments", str(segments),
                                                            "--subset", str(subset),
                                                            "--out-sweep",
                                                            os.path.join(d, "sweep.json")])
        if rc != 0:
            return rc, err, None
        doc = line
        rows = [(int(r[0]), float.fromhex(r[1]), float.fromhex(r[2]), float.fromhex(r[3]))
                for r in doc["rows"]]
        return rc, err, {"observed_max_batch": doc["observed_max_batch"], "rows": rows}


def same_as_reference(res, ref_entries, tally_rtol=0.0):
    """Bit-exact equality of a SearchResult with reference entries."""
    assert len(res) == len(ref_entries)
    for i, e in enumerate(ref_entries):
        g = res.entries[i]
        for f in SCALARS:
            if f in ("mfu", "mbu") and tally_rtol:
                assert np.isclose(g[f], e[f], rtol=tally_rtol, atol=0), (i, f, g[f], e[f])
            else:
                assert g[f] == e[f], (i, f, g[f], e[f])
        pr, rj = res.report(i)
        assert np.array_equal(pr, e["per_request"]), i
        assert np.array_equal(rj, e["rejected"]), i


def same_results(a, b, tally_rtol=0.0):
    """Bit-exact equality of two SearchResults (GPU vs oracle)."""
    assert len(a) == len(b)
    for f in a.entries.dtype.names:
        if f in ("per_request_offset", "rejected_offset"):
            continue
        if f in ("mfu", "mbu") and tally_rtol:
            assert np.allclose(a.entries[f], b.entries[f], rtol=tally_rtol, atol=0), f
        else:
            assert np.array_equal(a.entries[f], b.entries[f]), f
    for k in range(len(a)):
        pa, ra = a.report(k)
        pb, rb = b.report(k)
        assert np.array_equal(pa, pb), k
        assert np.array_equal(ra, rb), k
