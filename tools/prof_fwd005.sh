cd $GRAFT_REPO_ROOT
BENCH="python bench.py --rho 0.05 --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile --no-graph --no-c3 --no-c4"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_fwd_items<\(bool\)1, \(bool\)0>' -s 40 -c 1 \
    -o gpurun_out/fwd005 -f $BENCH > gpurun_out/fwd005.log 2>&1
echo fwd=$?
