"""Dev tool: time the engine on reference-dumped inputs of a workload.

    python tools/probe.py c2 c5_10k --reps 3

Inputs come from the compiled reference driver (oracle) so this is a
developer probe, not the benchmark (bench.py builds inputs with the native
host library).
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, os.path.join(REPO, "tests"))

from harness import RefCase, compare_to_ref  # noqa: E402
from paper_2411_17651_b200.engine import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("keys", nargs="+")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--workdir", default="/tmp/psg_probe")
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    eng = Engine(0)
    for key in args.keys:
        t0 = time.time()
        case = RefCase(key, args.workdir)
        ref_s = case.line["search_s_best"]
        cfg = case.config()
        best = None
        for _ in range(args.reps):
            res = eng.search(case.plans, case.cluster, case.store, case.trace, cfg, copy=False)
            if best is None or res.ms["total"] < best.ms["total"]:
                best = res
        res = eng.search(case.plans, case.cluster, case.store, case.trace, cfg)
        out = {"key": key, "entries": len(res), "plan_iterations": res.total_iterations,
               "ref_search_s": ref_s, "ref_jobs": case.line["jobs"], "ms": best.ms,
               "plan_iter_per_s_sim": res.total_iterations / (best.ms["sim"] / 1e3),
               "plan_iter_per_s_total": res.total_iterations / (best.ms["total"] / 1e3),
               "setup_s": time.time() - t0}
        if args.check:
            bad = compare_to_ref(res, case.ref, tally_rtol=1e-9)
            out["parity_problems"] = len(bad)
            out["first_problems"] = bad[:5]
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
