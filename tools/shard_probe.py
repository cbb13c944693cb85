"""Dev tool: strong scaling of one bench step, measured one rank at a time on
this GPU.  For each world size, the step's (plan, frequency) entries are
sharded longest-first exactly as `bench.py --scaling strong` does
(distributed.lpt_shards), and every rank's share runs as its own concurrent
search (psg_search_many) on this device; the strong-scaled step time is the
slowest rank's device span (the ranking all_gather of 48-byte records is
not included).

    python tools/shard_probe.py c5 --worlds 1 2 4 8
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from bench import WORKLOAD_SETS  # noqa: E402
from paper_2411_17651_b200 import distributed as pdist  # noqa: E402
from paper_2411_17651_b200.engine import Engine  # noqa: E402
from paper_2411_17651_b200.host import problem_for  # noqa: E402
from paper_2411_17651_b200.inputs import Config  # noqa: E402
from paper_2411_17651_b200.workloads import WORKLOADS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--worlds", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    keys, _ = WORKLOAD_SETS[args.config]
    ws = [WORKLOADS[k] for k in keys]
    probs = [problem_for(w) for w in ws]
    eng = Engine(0)
    costs = pdist.entry_costs(probs, [w.freqs for w in ws])
    for world in args.worlds:
        shards = pdist.lpt_shards(costs, len(probs), world)
        spans, iters = [], 0
        for r in range(world):
            jobs = [(p.plans, p.cluster, p.store, p.trace,
                     Config(objective=w.objective, freqs=w.freqs, detail=True, rank=False,
                            entry_subset=shards[r][i], ttft_slo=w.ttft_slo, slo_quantile=w.slo_quantile))
                    for i, (p, w) in enumerate(zip(probs, ws)) if shards[r][i]]
            best = None
            for _ in range(args.reps):
                res = eng.search_many(jobs, copy=False)
                best = eng.last_span_ms if best is None else min(best, eng.last_span_ms)
            iters += sum(x.total_iterations for x in res)
            spans.append(best)
        t = max(spans)
        print(f"{args.config} world {world}: step {t:.2f} ms (ranks {min(spans):.2f}-{t:.2f}), "
              f"{iters / (t / 1e3):.3g} plan-iter/s, {iters} plan-iterations", flush=True)


if __name__ == "__main__":
    main()
