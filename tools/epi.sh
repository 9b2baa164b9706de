cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q -k "bwd or fusion or c2_full" > gpurun_out/t.log 2>&1; echo rc=$? >> gpurun_out/t.log
timeout 300 python bench.py --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile --no-c3 --no-c4 > gpurun_out/fb0.log 2>&1
timeout 300 python bench.py --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile --no-c3 --no-c4 > gpurun_out/fb1.log 2>&1
