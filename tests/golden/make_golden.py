"""Generates tests/golden/*.json from the compiled reference (oracle/_ref/refdrv).

    python tests/golden/make_golden.py

Each golden file pins one case run through the UNMODIFIED reference library:
every ranked entry's scalar report fields (floats as exact hex), the entry's
plan encoding, and a sha256 over its per-request metrics (id, ttft, tpot,
e2e, gen_len as little-endian int64/f64) and over its rejected ids.  The GPU
and CPU-oracle tests compare against these without needing the reference
at run time.
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, os.path.join(REPO, "tests"))

FLOATS = ("freq_ghz", "e2e_latency", "total_energy", "p95_latency", "mean_ttft", "mean_tpot",
          "mfu", "mbu")
INTS = ("plan_index", "num_completed", "num_rejected", "num_iterations", "max_batch_observed")


def digest(arr) -> str:
    import numpy as np
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def entry_record(e):
    rec = {"encoding": e["encoding"]}
    for f in FLOATS:
        rec[f] = float(e[f]).hex()
    for f in INTS:
        rec[f] = int(e[f])
    rec["per_request_sha256"] = digest(e["per_request"])
    rec["rejected_sha256"] = digest(e["rejected"])
    return rec


def main():
    import tempfile

    import catalog
    from harness import RefCase
    out = {}
    with tempfile.TemporaryDirectory() as wd:
        for name in sorted(catalog.NAMED):
            case = catalog.NAMED[name]()
            rc, err, ref = case.reference(wd, name)
            assert rc == 0, err
            out[name] = [entry_record(e) for e in ref]
        for key in ("c1", "c3", "c4", "c4e"):
            case = RefCase(key, wd)
            out["config_" + key] = [entry_record(e) for e in case.ref]
    for name, recs in out.items():
        with open(os.path.join(HERE, name + ".json"), "w") as f:
            json.dump({"source": "oracle/_ref/refdrv (reference plansim::search / simulate_plan)",
                       "entries": recs}, f, indent=1)
    print(f"wrote {len(out)} golden files")


if __name__ == "__main__":
    main()
