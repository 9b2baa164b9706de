cd $GRAFT_REPO_ROOT
for s in 4 8 12 16; do
  timeout 300 python bench.py --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile --streams $s > gpurun_out/s$s.log 2>&1
done
