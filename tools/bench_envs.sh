# dev: bench.py (C2, no CPU baseline) under several environment settings
#   SETTINGS="A=1;A=2" bash tools/bench_envs.sh
cd ${GRAFT_REPO_ROOT:-/root/repo}
IFS=';' read -ra SETS <<< "$SETTINGS"
for round in 1 2; do
for st in "${SETS[@]}"; do
  printf "%-40s " "$st"
  env $st timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} 2>/dev/null | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), 'ms', round(d['value']/1e9,3), 'G plan-iter/s, e2e', round(d['full_search_ms']['e2e_median'],2), 'ms')"
done; done
