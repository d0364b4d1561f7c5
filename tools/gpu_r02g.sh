# last check of the rebuilt library (comment-only header edits after r02f): smoke, the windowed-engine and C-ABI GPU tests,
# the default bench line, configs 1-4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02g_smoke.log
timeout 1500 python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02g_pytest.log
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02g_c$c.json 2> gpurun_out/r02g_c$c.err
done
echo done
