# last check of the round on the committed library: smoke(), the GPU suite, the default bench line, INTEGRATION doc test
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02z_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02z_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02z_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02z_pytest.log
timeout 1500 python bench.py > gpurun_out/r02z_bench.json 2> gpurun_out/r02z_bench.err
for c in 1 2 3 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02z_c$c.json 2> gpurun_out/r02z_c$c.err
done
echo done
