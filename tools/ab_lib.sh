# dev: A/B two in-tree builds (PSG_LIBRARY) on tools/probe.py, interleaved
cd ${GRAFT_REPO_ROOT:-/root/repo}
KEYS=${KEYS:-"c1 c2 c2fp8 c4 c5_10k"}
for round in 1 2; do
for lib in ${LIBS:-libpsg_head.so libpsg.so}; do
  echo "== $lib"
  PSG_LIBRARY=$lib timeout 300 python tools/probe.py $KEYS --reps 3 2>&1 | python -c "
import sys,json
print(' '.join(f\"{d['key']}={d['ms']['sim']:.2f}\" for d in (json.loads(l) for l in sys.stdin if l.startswith('{'))))
"
done; done
