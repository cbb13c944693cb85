# dev: A/B an environment knob on tools/probe.py:  VAR=PSG_SERIAL_RUN VALS="4 8 16" bash tools/ab_env.sh
cd ${GRAFT_REPO_ROOT:-/root/repo}
KEYS=${KEYS:-"c1 c2 c2fp8 c4 c5_10k"}
for round in 1 2; do
for v in $VALS; do
  echo "== $VAR=$v"
  env $VAR=$v timeout 300 python tools/probe.py $KEYS --reps 3 2>&1 | python -c "
import sys,json
print(' '.join(f\"{d['key']}={d['ms']['sim']:.2f}\" for d in (json.loads(l) for l in sys.stdin if l.startswith('{'))))
"
done; done
