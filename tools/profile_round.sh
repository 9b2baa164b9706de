#!/bin/bash
# Run on the GPU box (gpurun): launch list of the bench command + one ncu --set full capture per
# hot kernel, written to gpurun_out/<tag>_*. Summaries are produced here with tools/*.py.
# usage: bash tools/profile_round.sh <tag> [kernel regex ...]
set -u
TAG=${1:-r01}
shift || true
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile --no-c3 --no-c4 --no-c5"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
  $BENCH > $OUT/${TAG}_launches_bench.log 2>&1
echo "launch list rc=$?"
# full sets: the kernels as the roofline pass launches them (one stream, full grid: --streams 1)
KS=("$@")
if [ ${#KS[@]} -eq 0 ]; then
  KS=('k_fwd_items<\(bool\)1, \(bool\)0, \(int\)2>' 'oit::k_moments\(' 'oit::k_epilogue' 'oit::k_project'
      'k_bin_expand<\(bool\)1>' 'oit::k_quad_bin' 'oit::k_items_emit' 'oit::k_tile_sort')
fi
i=0
for k in "${KS[@]}"; do
  i=$((i+1))
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$k" -s 40 -c 1 \
    -o $OUT/${TAG}_full_$i -f $BENCH --no-graph --streams 1 > $OUT/${TAG}_full_$i.log 2>&1
  echo "full $i ($k) rc=$?"
done
