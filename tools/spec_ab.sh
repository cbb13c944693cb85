for v in ${SPECS:-1 2 0}; do echo "SPEC=$v"; PSG_SPECULATE=$v timeout 300 python tools/probe.py ${KEYS:-c2 c5_10k} --reps 3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['key'], round(d['ms']['sim'],2))
"; done
