# Run on the GPU box (gpurun): the GPU parity suite with per-assertion gradient statistics
# (OIT_PARITY_LOG) and smoke, written to gpurun_out/. The compute-sanitizer runs this script made
# through round 2's r02e (profiles/r02e_sanitizer.txt) are gone: the GPU pool has closed
# compute-sanitizer (runs under it left GPUs needing a reset). usage: bash tools/check.sh <tag>
TAG=${1:-r02}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
OIT_PARITY_LOG=gpurun_out/${TAG}_parity_stats.jsonl timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputest.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_gputest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
for f in ${TAG}_gputest smoke; do echo "== $f"; tail -n 3 gpurun_out/$f.log; done
