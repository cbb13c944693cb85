"""Dev tool: per-phase cycle breakdown of the longest simulation units.

    PSG_LIBRARY=libpsg_prof.so python tools/phase_profile.py c2 [--top 5]

Runs one search on reference-dumped inputs with the profiler build and
prints, for the critical units, where their cycles go (slots documented in
psg_sim.cu).
"""
import argparse
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, os.path.join(REPO, "tests"))

NAMES = ["admit", "mixed_scan", "mixed_eval", "mixed_adv", "dec_cost", "run_setup", "tight",
         "finish", "evict", "refill", "#mixed", "#runs", "#dec_eval", "#finish", "#spec_hits", "total",
         "spec_wait_cyc", "miss_eval_cyc", "miss_nojob", "miss_items", "miss_decode", "miss_tok",
         "miss_unstarted", "ev_query_cyc", "ev_chain_cyc", "ev_stage_cyc",
         "arr_finish_cyc", "#arr_finish", "#arr_admit", "#arr_mixed", "admit_adm_cyc", "arr_pass_cyc"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("keys", nargs="+")
    ap.add_argument("--top", type=int, default=5)
    ap.add_argument("--enc", action="append", default=[], help="also show units whose encoding contains this")
    ap.add_argument("--per-dp", action="store_true", help="the longest unit of each DP degree instead of the top units")
    ap.add_argument("--workdir", default="/tmp/psg_probe")
    ap.add_argument("--native", action="store_true",
                    help="build inputs with the native host library instead of the reference driver")
    args = ap.parse_args()
    os.environ.setdefault("PSG_LIBRARY", "libpsg_prof.so")
    for key in args.keys:
        run(key, args)


def run(key, args):
    args.key = key
    out = os.path.join(args.workdir, f"phase_{args.key}.bin")
    os.makedirs(args.workdir, exist_ok=True)
    os.environ["PSG_PHASE_PROFILE"] = out
    from paper_2411_17651_b200.engine import Engine
    if args.native:
        from paper_2411_17651_b200.host import problem_for
        from paper_2411_17651_b200.inputs import Config
        from paper_2411_17651_b200.workloads import WORKLOADS

        class _Case:
            pass
        w = WORKLOADS[args.key]
        prob = problem_for(w)
        case = _Case()
        case.plans, case.cluster, case.store, case.trace = prob.plans, prob.cluster, prob.store, prob.trace
        case.workload = w
        case.config = lambda: Config(objective=w.objective, freqs=w.freqs)
    else:
        from harness import RefCase
        case = RefCase(args.key, args.workdir)
    eng = Engine(0)
    res = eng.search(case.plans, case.cluster, case.store, case.trace, case.config())
    raw = np.fromfile(out, dtype=np.uint64).reshape(-1, 2 + len(NAMES))
    meta, cnt = raw[:, :2].view(np.int64), raw[:, 2:]
    chain = os.environ.get("PSG_CHAIN_REPLICAS", "2")
    groups = int(os.environ.get("PSG_REPLICA_GROUPS", "2")) if chain == "2" else 1
    if chain != "0":
        # the replicas of a group run in order on one warp: aggregate per
        # (entry, group) — replica groups are contiguous replica ranges
        keys, rows_of = [], {}
        for u in range(len(meta)):
            e, r = int(meta[u, 0]), int(meta[u, 1])
            R = int((meta[:, 0] == e).sum())
            G = max(1, min(R, groups))
            g = next(k for k in range(G) if r < (k + 1) * R // G)
            rows_of.setdefault((e, g), []).append(u)
        agg = np.zeros((len(rows_of), cnt.shape[1]), dtype=np.uint64)
        m2 = np.zeros((len(rows_of), 2), dtype=np.int64)
        for i, ((e, g), rows) in enumerate(sorted(rows_of.items())):
            agg[i] = cnt[rows].sum(axis=0)
            m2[i] = (e, -len(rows))  # replica column: -(replicas in the group)
        meta, cnt = m2, agg
    order = np.argsort(-cnt[:, 15].astype(np.float64))
    F = max(1, len(case.workload.freqs))
    tots = cnt[:, 15].astype(np.float64)
    print(f"{args.key}: sim {res.ms['sim']:.2f} ms, units {len(raw)}, "
          f"sum/max {tots.sum() / tots.max():.1f}, units >50% of max: {(tots > 0.5 * tots.max()).sum()}, "
          f"totals: {' '.join(f'{k}={cnt[:, k].sum()}' for k in range(10, 14))}")
    by_dp = {}
    for u in range(len(cnt)):
        enc = case.plans.encodings[int(meta[u, 0]) // F]
        by_dp.setdefault(enc.split(":")[0], []).append(float(cnt[u, 15]) / 1.965e6)
    print("  by DP: " + "  ".join(f"{k}: n={len(v)} max={max(v):.2f} med={sorted(v)[len(v) // 2]:.2f} ms"
                                  for k, v in sorted(by_dp.items(), key=lambda kv: -max(kv[1]))))
    shown = order[:args.top]
    if args.per_dp:
        seen, shown = set(), []
        for u in order:
            dp = case.plans.encodings[int(meta[u, 0]) // F].split(":")[0]
            if dp not in seen:
                seen.add(dp)
                shown.append(u)
    shown = list(shown) + [u for u in order if u not in set(shown) and any(
        e in case.plans.encodings[int(meta[u, 0]) // F] for e in args.enc)]
    for u in shown:
        tot = float(cnt[u, 15])
        enc = case.plans.encodings[int(meta[u, 0]) // F]
        parts = " ".join(f"{NAMES[k]}={100 * cnt[u, k] / tot:.1f}%" for k in range(10))
        counts = " ".join(f"{NAMES[k]}={int(cnt[u, k])}" for k in range(10, 15))
        hits, miss = max(1, int(cnt[u, 14])), max(1, int(cnt[u, 10]) - int(cnt[u, 14]))
        counts += f" | wait/hit={int(cnt[u, 16]) // hits} cyc, eval/miss={int(cnt[u, 17]) // miss} cyc"
        counts += " | " + " ".join(f"{NAMES[k]}={int(cnt[u, k])}" for k in range(18, 23))
        own = max(1, int(cnt[u, 10]) - int(cnt[u, 14]))
        counts += " | per own eval: " + " ".join(f"{NAMES[k]}={int(cnt[u, k]) // own}" for k in range(23, 26))
        if cnt.shape[1] > 26 + 5:
            counts += (f" | slot-array mode: {100 * cnt[u, 31] / tot:.1f}% of cycles, finish "
                       f"{int(cnt[u, 26]) // max(1, int(cnt[u, 27]))} cyc x {int(cnt[u, 27])}, "
                       f"admissions {int(cnt[u, 28])}, mixed {int(cnt[u, 29])}; admitting passes "
                       f"{100 * cnt[u, 30] / tot:.1f}% of cycles")
        print(f"  {enc} r{int(meta[u, 1])}: {tot / 1.965e6:.2f} ms @1965MHz | {parts} | {counts}")


if __name__ == "__main__":
    main()
