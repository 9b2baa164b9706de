# Run on the GPU box (gpurun): the GPU parity suite with per-assertion gradient statistics
# (OIT_PARITY_LOG), smoke, and compute-sanitizer memcheck / racecheck / synccheck runs, all written
# to gpurun_out/. usage: bash tools/check.sh <tag>
TAG=${1:-r02}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
OIT_PARITY_LOG=gpurun_out/${TAG}_parity_stats.jsonl timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputest.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_gputest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/san_smoke.log 2>&1; echo memcheck_smoke=$? >> gpurun_out/san_smoke.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests -m gpu -x -q -k "u8 or concurrency or maximum or degenerate or score_split or update_active or fusion or long_lists or score_subsample" > gpurun_out/san_tests.log 2>&1; echo memcheck_tests=$? >> gpurun_out/san_tests.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/race_smoke.log 2>&1; echo racecheck_smoke=$? >> gpurun_out/race_smoke.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests -m gpu -x -q -k "long_lists or bin_tiles_bitexact or score_subsample_parity" > gpurun_out/race_tests.log 2>&1; echo racecheck_tests=$? >> gpurun_out/race_tests.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/sync_smoke.log 2>&1; echo synccheck_smoke=$? >> gpurun_out/sync_smoke.log
for f in ${TAG}_gputest smoke san_smoke san_tests race_smoke race_tests sync_smoke; do echo "== $f"; tail -n 3 gpurun_out/$f.log; done
