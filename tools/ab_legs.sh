# Run on the GPU box (gpurun): A/B of builds of liboit.so on the bench's configs[2]/[3] legs (C3 training
# views, C4 score sweep), round-robin. Variant A = the in-tree lib as shipped; others = files given.
# usage: R=<rounds> bash tools/ab_legs.sh <B.so> [<C.so> ...]
R=${R:-1}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
LIB=paper_2605_13855_b200/lib/liboit.so
cp $LIB /tmp/liboit_A.so
LIBS=(/tmp/liboit_A.so "$@")
for r in $(seq 1 $R); do
  for i in "${!LIBS[@]}"; do
    cp "${LIBS[$i]}" $LIB; touch $LIB
    timeout 600 python bench.py --no-sweep --no-e2e --no-cpu --no-ablation --no-dssim --no-adam --no-reconcile --no-c5 \
      > gpurun_out/abl_${i}_$r.json 2> gpurun_out/abl_${i}_$r.err
    python - "$i" "$r" "${LIBS[$i]}" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/abl_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
c3 = d["c3_mip360_shaped"]; c4 = d["c4_score_sweep"]["sweep"]
print(sys.argv[3], sys.argv[2], round(d["value"], 1), "C3", round(c3["clustered"]["mpix_per_s"]), round(c3["uniform"]["mpix_per_s"]),
      "C4 ms/refresh", {k: round(v["ms_per_refresh"], 2) for k, v in c4.items()})
PY
  done
done
cp /tmp/liboit_A.so $LIB
