# round-2 final capture: the whole GPU suite, the default bench (config 5) with its CPU baseline, the reference
# arm, ncu captures of the two top kernels (traffic table + summaries) and the launch list of the config-5 solve
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nproc > gpurun_out/r02y_nproc.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02y_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02y_pytest.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.err
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02y_ref.json 2> gpurun_out/r02y_ref.err
for k in k_richardson k_spmv_dots; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 20 -c 1 -f -o /tmp/r02y_c5_$k python tools/profile_solve.py --config 5 --solves 2 > gpurun_out/r02y_ncu_c5_$k.log 2>&1
  ncu -i /tmp/r02y_c5_$k.ncu-rep --page raw --csv > gpurun_out/r02y_ncu_c5_${k}_raw.csv 2>&1
  ncu -i /tmp/r02y_c5_$k.ncu-rep --page source --csv > gpurun_out/r02y_ncu_c5_${k}_source.csv 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02y_launches_c5.csv python tools/profile_solve.py --config 5 --solves 2 > gpurun_out/r02y_launches_c5.log 2>&1
timeout 600 python bench.py --config 2 --partition --steps 5 --warmup 3 > gpurun_out/r02y_c2_part.json 2> gpurun_out/r02y_c2_part.err
echo done
