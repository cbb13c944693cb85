for v in ${SERIALS:-64 128 256 1000000000}; do echo "SERIAL=$v"; PSG_SERIAL_RUN=$v python tools/probe.py c1 c2 c3 c4 --reps 3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['key'], round(d['ms']['sim'],2), d['plan_iterations'])
"; done
