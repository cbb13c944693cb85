"""Shared parity helpers: run the compiled reference on a workload and load the
exact same inputs (plans / store / trace dumped by the reference itself) into
the engine's SoA structures."""
from __future__ import annotations

import hashlib
import os

import numpy as np

import pyoracle
from paper_2411_17651_b200.inputs import Cluster, Config, Plans, Store, Trace
from paper_2411_17651_b200.workloads import WORKLOADS

SCALARS = ("plan_index", "freq_ghz", "e2e_latency", "total_energy", "p95_latency",
           "mean_ttft", "mean_tpot", "mfu", "mbu", "num_completed", "num_rejected",
           "num_iterations", "max_batch_observed")
EXACT_TALLY = ("mfu", "mbu")  # per-replica partial tallies


class RefCase:
    def __init__(self, key, workdir, extra=(), jobs=None, out_ranked=False, digest=False):
        self.key = key
        w = WORKLOADS[key]
        d = os.path.join(workdir, key + "".join(str(x) for x in extra).replace("-", "_"))
        os.makedirs(d, exist_ok=True)
        paths = w.materialize(d)
        self.paths = paths
        self.dump = os.path.join(d, "ref.bin")
        self.plans_path = os.path.join(d, "plans.json")
        self.store_path = os.path.join(d, "store.jsonl")
        self.trace_path = os.path.join(d, "trace.jsonl")
        jobs = jobs or os.cpu_count() or 1
        args = ["search"] + w.refdrv_args(paths) + list(extra) + [
            "--jobs", jobs, "--out-result", self.dump, "--out-plans", self.plans_path,
            "--out-store", self.store_path, "--out-trace", self.trace_path]
        if digest:  # per-request arrays as SHA-256 digests (C5-100k: 1.2 GB otherwise)
            args.append("--digest")
        self.ranked_path = os.path.join(d, "ranked.json") if out_ranked else None
        if out_ranked:
            args += ["--out-ranked", self.ranked_path]
        rc, self.line, err = pyoracle.refdrv(args)
        assert rc == 0, err
        self.ref, self.warnings = pyoracle.read_refdump(self.dump)
        self.plans = Plans.from_json(open(self.plans_path).read())
        self.store = Store.from_jsonl(open(self.store_path).read())
        self.trace = Trace.from_jsonl(open(self.trace_path).read())
        self.cluster = Cluster.from_json(open(paths["cluster"]).read())
        self.workload = w

    def config(self, **kw):
        cfg = dict(objective=self.workload.objective, freqs=self.workload.freqs,
                   ttft_slo=self.workload.ttft_slo, slo_quantile=self.workload.slo_quantile)
        cfg.update(kw)
        return Config(**cfg)


def compare_to_ref(res, ref, tally_rtol=0.0):
    """Bit-exact comparison of every reported field; returns a list of problems."""
    bad = []
    if len(res.entries) != len(ref):
        return [f"entry count {len(res.entries)} != {len(ref)}"]
    for i, e in enumerate(ref):
        g = res.entries[i]
        if res.encoding(i) != e["encoding"]:
            bad.append(f"rank {i}: plan {res.encoding(i)} != {e['encoding']}")
        for f in SCALARS:
            gv, rv = g[f], e[f]
            if f in EXACT_TALLY and tally_rtol > 0:
                if not np.isclose(gv, rv, rtol=tally_rtol, atol=0):
                    bad.append(f"rank {i} {e['encoding']}: {f} {gv!r} vs {rv!r}")
            elif gv != rv:
                bad.append(f"rank {i} {e['encoding']}: {f} {gv!r} != {rv!r}")
        pr, rj = res.report(i)
        if "per_request_sha256" in e:  # digest dump
            if (len(pr) != e["n_per_request"] or
                    hashlib.sha256(np.ascontiguousarray(pr).tobytes()).hexdigest()
                    != e["per_request_sha256"]):
                bad.append(f"rank {i} {e['encoding']}: per_request digest differs")
            if (len(rj) != e["n_rejected"] or
                    hashlib.sha256(np.ascontiguousarray(rj).tobytes()).hexdigest()
                    != e["rejected_sha256"]):
                bad.append(f"rank {i} {e['encoding']}: rejected_ids digest differs")
        elif not np.array_equal(pr, e["per_request"]):
            bad.append(f"rank {i} {e['encoding']}: per_request differs")
        if "rejected" in e and not np.array_equal(rj, e["rejected"]):
            bad.append(f"rank {i} {e['encoding']}: rejected_ids differ")
        if len(bad) > 20:
            break
    return bad
