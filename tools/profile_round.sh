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
# full sets: the kernels as the roofline pass launches them (one stream, full grid: --streams 1).
# Each entry: "<kernel regex>|<launches of that kernel to skip>": the bench's first 100 binning /
# projection launches build the frozen-set caches (240k slots) and the next 100 count the work; skip
# 230 to capture a training view (60k active slots) like the hot composite kernels.
KS=("$@")
if [ ${#KS[@]} -eq 0 ]; then
  KS=('k_fwd_items<\(bool\)1, \(bool\)0, \(int\)2>|40' 'oit::k_moments\(|40' 'oit::k_epilogue\(|40' 'oit::k_project|230'
      'k_bin_expand<\(bool\)1>|230' 'oit::k_quad_bin|40' 'oit::k_items_emit|40' 'oit::k_tile_sort|230'
      'oit::k_epilogue_mv|2')
fi
i=0
for ks in "${KS[@]}"; do
  k=${ks%|*}; skip=${ks##*|}
  [ "$skip" = "$ks" ] && skip=40
  i=$((i+1))
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$k" -s $skip -c 1 \
    -o $OUT/${TAG}_full_$i -f $BENCH --no-graph --streams 1 > $OUT/${TAG}_full_$i.log 2>&1
  echo "full $i ($k, skip $skip) rc=$?"
done
