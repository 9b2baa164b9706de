# Run on the GPU box (gpurun): the parity tests a kernel change touches, the in-process A/B timing of
# the hot kernels (tools/ab.py) and a short bench (headline ρ only) — the loop used to accept or
# reject the kernel experiments listed in DESIGN.md §7.
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q -k "bwd or score or fusion or concurrency or c2_full or degenerate" > gpurun_out/t.log 2>&1; echo rc=$? >> gpurun_out/t.log
python tools/ab.py --variants 0 --rounds 4 > gpurun_out/ab0.log 2>&1
timeout 300 python bench.py --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile --no-c3 --no-c4 --no-c5 > gpurun_out/fb0.log 2>&1
