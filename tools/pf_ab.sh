cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
LIB=paper_2605_13855_b200/lib/liboit.so
cp $LIB /tmp/A.so
BENCH="python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile --no-c3 --no-c4 --no-c5 --no-graph --streams 1"
for v in A pre; do
  if [ $v = A ]; then cp /tmp/A.so $LIB; else cp build/liboit_pre.so $LIB; fi; touch $LIB
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:k_epilogue|k_project" --csv $BENCH > gpurun_out/pf_$v.csv 2>/dev/null
  python - $v <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(f"gpurun_out/pf_{sys.argv[1]}.csv")) if len(r) > 10]
hdr = rows[0]; iN = hdr.index("Kernel Name"); iM = hdr.index("Metric Name"); iV = hdr.index("Metric Value"); iID = hdr.index("ID")
d = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    n = r[iN].split("(")[0]
    d[n][r[iM]].append(float(r[iV].replace(",", "")))
for n, m in d.items():
    t = m["gpu__time_duration.sum"]
    print(sys.argv[1], n, len(t), "median us", sorted(t)[len(t)//2], "sum ms", round(sum(t)/1e3, 3))
PY
done
cp /tmp/A.so $LIB
BENCH_ARGS="--rho 0.05" R=2 bash tools/ab_bench.sh build/liboit_pre.so
R=1 bash tools/ab_legs.sh build/liboit_pre.so
