import sys, time, statistics, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_2411_17651_b200.engine import Engine
from paper_2411_17651_b200.host import problem_for
from paper_2411_17651_b200.inputs import Config
from paper_2411_17651_b200.workloads import WORKLOADS
eng = Engine(0)
ws = [WORKLOADS[k] for k in (sys.argv[1:] or ["c2", "c2fp8"])]
probs = [problem_for(w) for w in ws]
jobs = [(p.plans, p.cluster, p.store, p.trace, Config(objective=w.objective, freqs=w.freqs, detail=True, rank=True)) for p, w in zip(probs, ws)]
rows = []
for i in range(8):
    t0 = time.perf_counter()
    n = len(jobs)
    res = eng.search_many(jobs, copy=False)
    t1 = time.perf_counter()
    rows.append(((t1 - t0) * 1e3, eng.last_span_ms, [r.ms for r in res]))
for w, span, ms in rows[3:]:
    print(f"wall {w:.2f} ms  span {span:.2f} ms  " + " | ".join(" ".join(f"{k}={v:.2f}" for k, v in m.items()) for m in ms))
