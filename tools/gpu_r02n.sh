# partition schedule (update phases only where the call can update) + all five configs
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_partition.py tests/test_gpu_solver.py tests/test_gpu_precond.py -m gpu -x -q > gpurun_out/r02n_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02n_pytest.log
timeout 600 python bench.py --config 2 --partition --steps 5 --warmup 3 > gpurun_out/r02n_c2_part.json 2> gpurun_out/r02n_c2_part.err
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02n_c$c.json 2> gpurun_out/r02n_c$c.err
done
echo done
