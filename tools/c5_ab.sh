for cfg in "1 1" "0 1" "1 0" "0 0"; do set -- $cfg; echo "SPEC=$1 CHAIN=$2"; PSG_SPECULATE=$1 PSG_CHAIN_REPLICAS=$2 timeout 300 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), 'ms', round(d['value']/1e6,1), 'M plan-iter/s')"; done
