# dev: every measurement behind profiles/ in one GPU session (see profiles/README.md)
#   bash tools/refresh_profiles.sh <round tag, e.g. r2>
cd ${GRAFT_REPO_ROOT:-/root/repo}
T=${1:-r2}; O=gpurun_out/refresh; mkdir -p $O
python bench.py > $O/bench_c2_$T.json 2> $O/bench_c2.err
python bench.py --config c5 --steps 5 > $O/bench_c5_$T.json 2> $O/bench_c5.err
for c in c1 c4 c3slo c2dvfs; do
  python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_${c}_$T.json 2> $O/bench_$c.err
done
python bench.py --config c5full --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c5full_$T.json 2> $O/bench_c5full.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launches_c2_$T.csv 2> $O/launches.err
PSG_PROFILE_RANGE=1 ncu --replay-mode app-range --clock-control none \
  --metrics sm__inst_issued.sum,sm__cycles_active.sum,sm__cycles_elapsed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --csv --log-file $O/range_c2_$T.csv python bench.py --steps 1 --no-cpu-baseline > $O/range.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:sim_kernel -s 6 -c 1 \
  -o $O/prof_bench_sim_c2_$T python bench.py --steps 1 --no-cpu-baseline > $O/prof.log 2>&1
ls -la $O
