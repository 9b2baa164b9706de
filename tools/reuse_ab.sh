# Run on the GPU box: the score-coefficient reuse A/B (bench --coef-reuse vs the default) at rho 0.2 / 0.05,
# after the parity tests that touch it.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "score or fusion or bench" > gpurun_out/t_reuse.log 2>&1; echo rc=$? >> gpurun_out/t_reuse.log; tail -3 gpurun_out/t_reuse.log
BENCH="python bench.py --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile --no-c3 --no-c4 --no-c5"
for r in 1 2; do for rho in 0.2 0.05; do for f in "--coef-reuse" ""; do
  timeout 400 $BENCH --rho $rho $f > gpurun_out/ru.json 2> gpurun_out/ru.err || tail -5 gpurun_out/ru.err
  python -c "import json; d=json.loads(open('gpurun_out/ru.json').read().strip().splitlines()[-1]); print('$rho', '$f' or 'no-reuse', round(d['value'],1), round(d['ms_per_step'],3), d['gpu_launches'], d['segments_ms'])"
done; done; done
