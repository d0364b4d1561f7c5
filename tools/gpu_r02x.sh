# windowed engine, unrolled z1 pre-pass: parity + config-5 bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wsell.py tests/test_gpu_seq.py tests/test_gpu_kernels.py tests/test_gpu_solver.py tests/test_gpu_krylov.py -m gpu -x -q > gpurun_out/r02x_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02x_pytest.log
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02x_c5.json 2> gpurun_out/r02x_c5.err
echo done
