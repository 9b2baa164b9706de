cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err; echo bench=$?
bash tools/check.sh r02g > gpurun_out/r02g_check.log 2>&1; echo check=$?
bash tools/profile_round.sh r02g > gpurun_out/r02g_profile.log 2>&1; echo profile=$?
bash tools/check_launches.sh --rho 0.2 > gpurun_out/r02g_launch_check.txt 2>&1
bash tools/check_launches.sh --rho 0.05 >> gpurun_out/r02g_launch_check.txt 2>&1
bash tools/check_launches.sh --rho 1.0 >> gpurun_out/r02g_launch_check.txt 2>&1
echo launches=$?
for f in gpurun_out/r02g_full_*.ncu-rep; do ncu -i $f --page source --csv --print-source sass > ${f%.ncu-rep}_src.csv 2>/dev/null; done
ls -la gpurun_out | tail -40
