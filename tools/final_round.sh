cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err; echo bench=$?
bash tools/check.sh r02i > gpurun_out/r02i_check.log 2>&1; echo check=$?
bash tools/profile_round.sh r02i "k_fwd_items<\(bool\)1, \(bool\)0, \(int\)2>|40" "oit::k_moments\(|40" "oit::k_epilogue\(|40" "oit::k_epilogue_mv|2" > gpurun_out/r02i_profile.log 2>&1; echo profile=$?
bash tools/check_launches.sh --rho 0.2 > gpurun_out/r02i_launch_check.txt 2>&1
bash tools/check_launches.sh --rho 0.05 >> gpurun_out/r02i_launch_check.txt 2>&1
bash tools/check_launches.sh --rho 1.0 >> gpurun_out/r02i_launch_check.txt 2>&1
echo launches=$?
for f in gpurun_out/r02i_full_*.ncu-rep; do ncu -i $f --page source --csv --print-source sass > ${f%.ncu-rep}_src.csv 2>/dev/null; done
ls -la gpurun_out | tail -40
