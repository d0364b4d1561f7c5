# windowed SELL engine: parity, regression, config-5 A/B
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wsell.py -m gpu -x -q > gpurun_out/r02p_wsell.log 2>&1; echo "rc=$?" >> gpurun_out/r02p_wsell.log
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02p_c5.json 2> gpurun_out/r02p_c5.err
F3RG_WSELL=0 timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02p_c5_tiles.json 2> gpurun_out/r02p_c5_tiles.err
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py tests/test_gpu_seq.py -m gpu -x -q > gpurun_out/r02p_reg.log 2>&1; echo "rc=$?" >> gpurun_out/r02p_reg.log
echo done
