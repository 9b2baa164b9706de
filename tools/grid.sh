cd $GRAFT_REPO_ROOT
B="python bench.py --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile --no-c3 --no-c4"
for cfg in "4 2" "2 1" "3 1" "2 2" "3 2" "4 3" "5 2" "3 3"; do
  set -- $cfg
  OIT_FWD_CTAS=$1 OIT_MOM_CTAS=$2 timeout 300 $B > gpurun_out/g_$1_$2.log 2>&1
done
