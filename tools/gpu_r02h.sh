# ncu --set full of the config-5 passes below the top two: the L2 spmv_dots (fp32 matrix, class-1 code + value
# streams) and the fp64 true-residual pass, for profiles/traffic.json
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
i=0
for k in 'k_spmv_dots<\(int\)1' 'k_residual'; do
  i=$((i+1))
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$k" --launch-skip 3 -c 1 -f -o /tmp/r02h_$i python tools/profile_solve.py --config 5 --solves 2 > gpurun_out/r02h_ncu_$i.log 2>&1
  ncu -i /tmp/r02h_$i.ncu-rep --page raw --csv > gpurun_out/r02h_ncu_c5_${i}_raw.csv 2>&1
done
echo done
