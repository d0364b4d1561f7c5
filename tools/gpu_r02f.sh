# round-2 closing capture on the library with class-1 streams for every replica: smoke, bench, GPU suite, reference arm, ncu + launch list
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nproc > gpurun_out/r02f_nproc.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02f_smoke.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02f_pytest.log
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02f_ref.json 2> gpurun_out/r02f_ref.err
for k in k_richardson k_spmv_dots; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 20 -c 1 -f -o /tmp/r02f_c5_$k python tools/profile_solve.py --config 5 --solves 2 > gpurun_out/r02f_ncu_c5_$k.log 2>&1
  ncu -i /tmp/r02f_c5_$k.ncu-rep --page raw --csv > gpurun_out/r02f_ncu_c5_${k}_raw.csv 2>&1
  ncu -i /tmp/r02f_c5_$k.ncu-rep --page source --csv > gpurun_out/r02f_ncu_c5_${k}_source.csv 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches_c5.csv python tools/profile_solve.py --config 5 --solves 2 > gpurun_out/r02f_launches_c5.log 2>&1
timeout 600 python bench.py --config 2 --partition --steps 5 --warmup 3 > gpurun_out/r02f_c2_part.json 2> gpurun_out/r02f_c2_part.err
echo done
