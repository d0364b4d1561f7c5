# seq-mode exactness with the glibc hypot restatement + ncu of the config-5 fp16 passes
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_seq.py tests/test_gpu_solver.py tests/test_gpu_kernels.py -m gpu -q > gpurun_out/r02b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02b_pytest.log
for k in k_richardson k_spmv_dots; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 20 -c 1 -f -o /tmp/r02b_$k python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02b_ncu_$k.log 2>&1
  ncu -i /tmp/r02b_$k.ncu-rep --page raw --csv > gpurun_out/r02b_ncu_${k}_raw.csv 2>&1
  ncu -i /tmp/r02b_$k.ncu-rep --page details --csv > gpurun_out/r02b_ncu_${k}_details.csv 2>&1
  ncu -i /tmp/r02b_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/r02b_ncu_${k}_source.csv 2>&1
  ls -la /tmp/r02b_$k.ncu-rep >> gpurun_out/r02b_ncu_$k.log
done
du -sh gpurun_out
