# Run on the GPU box: the launch list of exactly one bench step (ncu --profile-from-start off around
# bench.py --profile-once) against the step's claimed kernel count (bench.py's gpu_launches / steps).
# usage: bash tools/check_launches.sh [extra bench args, e.g. --rho 0.05]
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/one_step_launches.csv python bench.py --profile-once "$@" > gpurun_out/one_step.log 2>&1
python - <<'PY'
import csv, json, collections
rows = list(csv.reader(open("gpurun_out/one_step_launches.csv")))
hdr = next(r for r in rows if r and r[0] == "ID")
names = [dict(zip(hdr, r))["Kernel Name"] for r in rows if len(r) == len(hdr) and r[0] != "ID"]
ours = [n for n in names if "oit::" in n]
claim = json.loads([l for l in open("gpurun_out/one_step.log") if l.startswith("{")][-1])["kernel_launches_claimed_per_step"]
print(f"launch list: {len(ours)} liboit kernels in one step ({len(names)} kernels in all); claimed {claim}")
for k, v in sorted(collections.Counter(n.split("(")[0] for n in ours).items(), key=lambda x: -x[1]):
    print(f"  {v:6d}  {k}")
PY
