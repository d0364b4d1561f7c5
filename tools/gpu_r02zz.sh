# validation of the class-1 code + value streams: smoke(), the GPU suite, the default bench line (with CPU baseline),
# ncu of the L2 spmv_dots
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02zz_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02zz_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02zz_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02zz_pytest.log
timeout 1500 python bench.py > gpurun_out/r02zz_bench.json 2> gpurun_out/r02zz_bench.err
echo done
