# dev: A/B several environment settings on tools/probe.py:
#   SETTINGS="A=1;A=2 B=3" KEYS="c2" bash tools/ab_envs.sh
cd ${GRAFT_REPO_ROOT:-/root/repo}
KEYS=${KEYS:-"c2 c2fp8 c5_10k"}
IFS=';' read -ra SETS <<< "$SETTINGS"
for round in 1 2; do
for st in "${SETS[@]}"; do
  echo "== $st"
  env $st timeout 300 python tools/probe.py $KEYS --reps 3 2>&1 | python -c "
import sys,json
print(' '.join(f\"{d['key']}={d['ms']['sim']:.2f}\" for d in (json.loads(l) for l in sys.stdin if l.startswith('{'))))
"
done; done
