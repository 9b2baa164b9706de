cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q ${TESTS:-} > gpurun_out/t.log 2>&1; echo tests=$? >> gpurun_out/t.log
timeout 400 python bench.py --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile > gpurun_out/b.log 2>&1; echo bench=$? >> gpurun_out/b.log
