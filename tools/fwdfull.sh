cd $GRAFT_REPO_ROOT
for f in 16 24 12; do
  OIT_FWD_FULL=$f python tools/ab.py --variants 0 --rounds 4 > gpurun_out/ff_$f.log 2>&1
  OIT_FWD_FULL=$f timeout 300 python bench.py --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile --no-c3 --no-c4 > gpurun_out/fb_$f.log 2>&1
done
