# dev: parity subset on the current build, then A/B against another build
cd ${GRAFT_REPO_ROOT:-/root/repo}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fixtures.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
KEYS=${KEYS:-"c1 c2 c2fp8 c4 c5_10k"} bash tools/ab_lib.sh
