# Run on the GPU box (gpurun): A/B of builds of liboit.so on the bench's headline step (C2, rho 0.2;
# other legs off), round-robin so clock drift hits all alike. Variant A is the in-tree
# lib/liboit.so as shipped; the others are the files given (e.g. build/liboit_base.so).
# usage: R=<rounds> bash tools/ab_bench.sh <B.so> [<C.so> ...]   (BENCH_ARGS: extra bench flags)
R=${R:-2}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
LIB=paper_2605_13855_b200/lib/liboit.so
cp $LIB /tmp/liboit_A.so
LIBS=(/tmp/liboit_A.so "$@")
BENCH="python bench.py --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile --no-c3 --no-c4 --no-c5 ${BENCH_ARGS:-}"
for r in $(seq 1 $R); do
  for i in "${!LIBS[@]}"; do
    cp "${LIBS[$i]}" $LIB
    touch $LIB
    timeout 400 $BENCH > gpurun_out/ab_${i}_$r.json 2> gpurun_out/ab_${i}_$r.err
    python - "$i" "$r" "${LIBS[$i]}" <<'EOF'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
except Exception as e:  # noqa: BLE001
    print(sys.argv[3], sys.argv[2], "FAILED", e); raise SystemExit
rf = d.get("roofline", {})
per = {k: (round(v.get("kernel_ms_per_step"), 3), round(v.get("frac", 0), 3)) for k, v in (rf.get("per_kernel") or {}).items()}
print(sys.argv[3], sys.argv[2], d["value"], d["ms_per_step"], per)
EOF
  done
done
cp /tmp/liboit_A.so $LIB
