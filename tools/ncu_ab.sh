# dev: warp-state / instruction stats of the simulation kernel for several in-tree builds
cd ${GRAFT_REPO_ROOT:-/root/repo}
KEY=${KEY:-c5_10k}
python tools/probe.py $KEY --reps 1 > /dev/null 2>&1   # warm the input cache
for lib in ${LIBS:-libpsg_head.so libpsg.so}; do
  echo "== $lib"
  PSG_LIBRARY=$lib timeout 600 ncu --clock-control none -k regex:sim_kernel -c 1 \
    --section WarpStateStats --section InstructionStats --section LaunchStats --section SpeedOfLight --metrics smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio --csv --page details \
    python tools/probe.py $KEY --reps 1 2>/dev/null | grep -v "^==PROF==" | python -c "
import sys,csv
for r in csv.reader(sys.stdin):
    if len(r)>14 and (r[12].startswith('smsp__average') or r[12] in ('Executed Instructions','Warp Cycles Per Issued Instruction','Registers Per Thread','Duration') or r[12].startswith('smsp__pcsamp') or 'stall' in r[12].lower()):
        print('  ', r[12], r[14])
"
done
