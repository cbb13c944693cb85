for v in 1 0; do echo "CHAIN=$v"; PSG_CHAIN_REPLICAS=$v python tools/probe.py c1 c2 c2fp8 c4 c5_10k --reps 3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['key'], round(d['ms']['sim'],2))
"; done
