"""Dev tool: ranked.json materialization time, reference recipe (refdrv:
report_to_json -> parse -> dump(2), tools/plansim_main.cpp:128-131) vs the
streaming writer, on the same search result.

    python tools/report_speed.py c2
"""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, os.path.join(REPO, "tests"))

from harness import RefCase  # noqa: E402
from paper_2411_17651_b200.engine import Engine  # noqa: E402


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "c2"
    case = RefCase(key, "/tmp/psg_report_speed", out_ranked=True)
    eng = Engine(0)
    res = eng.search(case.plans, case.cluster, case.store, case.trace, case.config())
    out = "/tmp/psg_report_speed/ours_ranked.json"
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        res.write_ranked_json(out)
        best = min(best, time.perf_counter() - t0)
    size = os.path.getsize(out)
    print({"key": key, "bytes": size, "reference_recipe_s": case.line["ranked_s"],
           "streaming_writer_s": round(best, 4),
           "same_size": size == os.path.getsize(case.ranked_path)})


if __name__ == "__main__":
    main()
