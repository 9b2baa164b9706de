cd $GRAFT_REPO_ROOT
for s in 8 10 12 14; do
  timeout 300 python bench.py --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile --no-c3 --no-c4 --no-c5 --streams $s > gpurun_out/s$s.log 2>&1
done
