for v in 20 100 400; do echo "SLEEP=$v"; PSG_SPEC_SLEEP_NS=$v timeout 300 python tools/probe.py c2 c2fp8 c5_10k --reps 3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['key'], round(d['ms']['sim'],2))
"; done
