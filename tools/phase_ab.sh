# dev: phase profiles of the critical units for several profiler builds
cd ${GRAFT_REPO_ROOT:-/root/repo}
for lib in ${LIBS:-libpsg_headprof.so libpsg_prof.so}; do
  echo "== $lib"
  PSG_LIBRARY=$lib timeout 300 python tools/phase_profile.py ${KEYS:-c2 c5_10k} --top ${TOP:-2} 2>&1 | grep -v "^psg"
done
