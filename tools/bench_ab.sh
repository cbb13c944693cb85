# dev: A/B environment settings on bench.py (device ms per step / end-to-end ms per step):
#   CONFIGS="c2 c5" SETTINGS="A=1;B=2" STEPS=5 bash tools/bench_ab.sh
cd ${GRAFT_REPO_ROOT:-/root/repo}
IFS=';' read -ra SETS <<< "$SETTINGS"
for round in 1 2; do
for st in "${SETS[@]}"; do
  line="== $st:"
  for c in $CONFIGS; do
    ms=$(env $st timeout 600 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); it=d['workload_stats']['plan_iterations_per_step']; print(f\"{d['ms_per_step']:.2f}/{1e3*it/d['e2e']['value']:.2f}\")")
    line="$line $c=$ms"
  done
  echo "$line"
done; done
