# ncu of the windowed SELL engine on config 5: Richardson + L3 spmv_dots (raw + source pages)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in k_richardson k_spmv_dots; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 20 -c 1 -f -o /tmp/r02q_c5_$k python tools/profile_solve.py --config 5 --solves 2 > gpurun_out/r02q_ncu_c5_$k.log 2>&1
  ncu -i /tmp/r02q_c5_$k.ncu-rep --page raw --csv > gpurun_out/r02q_ncu_c5_${k}_raw.csv 2>&1
  ncu -i /tmp/r02q_c5_$k.ncu-rep --page source --csv > gpurun_out/r02q_ncu_c5_${k}_source.csv 2>&1
done
echo done
