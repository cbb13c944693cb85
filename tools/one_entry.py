"""Dev tool: run a search over the units of selected entries only (by plan
encoding), e.g. to capture one critical unit alone under ncu:

    PSG_SPECULATE=0 ncu --set full --import-source on -k regex:sim_kernel -c 1 \\
        python tools/one_entry.py c2 dp1:pp1:GQA-tp16x1:SwiGLU-tp4x4
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, os.path.join(REPO, "tests"))

from harness import RefCase  # noqa: E402
from paper_2411_17651_b200.engine import Engine  # noqa: E402


def main(key, encs, workdir="/tmp/psg_probe"):
    case = RefCase(key, workdir)
    F = max(1, len(case.workload.freqs))
    sub = [p * F + f for p, e in enumerate(case.plans.encodings) if e in encs for f in range(F)]
    cfg = case.config(entry_subset=sub)
    res = Engine(0).search(case.plans, case.cluster, case.store, case.trace, cfg)
    print(f"{key}: {len(sub)} entries, sim {res.ms['sim']:.3f} ms, {res.total_iterations} plan-iterations")


if __name__ == "__main__":
    main(sys.argv[1], set(sys.argv[2:]))
