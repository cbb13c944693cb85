# dev: parity subset, kernel durations of the table kernels, probe timings
cd ${GRAFT_REPO_ROOT:-/root/repo}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fixtures.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/probe.py ${NCU_KEYS:-c5_10k c2 c4} --reps 1 2>/dev/null | python -c "
import csv,sys
for r in csv.reader(sys.stdin):
    if len(r)>14 and r[12]=='gpu__time_duration.sum' and ('tab' in r[4] or 'sim' in r[4]): print(r[4][:22], r[8], r[14])
"
for lib in ${LIBS:-libpsg.so}; do
PSG_LIBRARY=$lib timeout 300 python tools/probe.py ${KEYS:-c1 c2 c2fp8 c4 c5_10k} --reps 3 2>&1 | grep "^{" | python -c "
import sys,json
print('$lib', ' '.join(f\"{d['key']}={d['ms']['sim']:.2f}\" for d in (json.loads(l) for l in sys.stdin)))
"
done
