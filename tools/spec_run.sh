timeout 240 python -m pytest tests/test_gpu_fixtures.py -x -q 2>&1 | tail -2 || exit 1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in 1 0; do echo "SPEC=$v"; PSG_SPECULATE=$v timeout 300 python tools/probe.py c1 c2 c2fp8 c4 c5_10k --reps 3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['key'], round(d['ms']['sim'],2))
"; done
timeout 300 python tools/phase_profile.py c2 c5_10k --top 1 2>&1 | grep -v "^psg" | tail -4
