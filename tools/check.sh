cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q -k "maximum or degenerate" > gpurun_out/t.log 2>&1; echo rc=$? >> gpurun_out/t.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/san_smoke.log 2>&1; echo memcheck_smoke=$? >> gpurun_out/san_smoke.log
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests -m gpu -x -q -k "u8 or concurrency or maximum or degenerate or score_split or update_active or fusion" > gpurun_out/san_tests.log 2>&1; echo memcheck_tests=$? >> gpurun_out/san_tests.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/race_smoke.log 2>&1; echo racecheck_smoke=$? >> gpurun_out/race_smoke.log
