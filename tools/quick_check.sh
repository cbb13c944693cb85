# dev: parity subset + per-workload simulation times (tools/probe.py)
cd ${GRAFT_REPO_ROOT:-/root/repo}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fixtures.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -3
timeout 300 python tools/probe.py c1 c2 c2fp8 c4 c5_10k --reps 3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['key'], round(d['ms']['sim'],2))
"
