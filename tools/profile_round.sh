#!/bin/bash
# Run on the GPU box (gpurun): launch list of the bench command + one ncu --set full capture per
# hot kernel, written to gpurun_out/<tag>_*. Summaries are produced here with tools/*.py.
# usage: bash tools/profile_round.sh <tag> [kernel regex ...]
set -u
TAG=${1:-r01}
shift || true
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
  $BENCH > $OUT/${TAG}_launches_bench.log 2>&1
echo "launch list rc=$?"
KS=${@:-k_fwd_items k_moments k_epilogue k_project k_bin_expand k_quad_count k_quad_scatter k_items_fused}
for k in $KS; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^${k}\$" -s 40 -c 1 \
    -o $OUT/${TAG}_full_${k} -f $BENCH --no-graph > $OUT/${TAG}_full_${k}.log 2>&1
  echo "full $k rc=$?"
done
