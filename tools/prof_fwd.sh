cd $GRAFT_REPO_ROOT
BENCH="python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile --no-graph"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_fwd_items<\(bool\)1, \(bool\)0>' -s 40 -c 1 \
    -o gpurun_out/r01b_full_k_fwd_items_base -f $BENCH > gpurun_out/r01b_full_k_fwd_items_base.log 2>&1
echo fwd=$?
