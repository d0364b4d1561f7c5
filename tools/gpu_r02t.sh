# round-2 validation of the windowed engine build: config-5 bench, the whole GPU suite (durations listed:
# the config-5 ILU(0) test is new), per-config lines
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02t_c5.json 2> gpurun_out/r02t_c5.err
timeout 2700 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r02t_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02t_pytest.log
for c in 1 2 3 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02t_c$c.json 2> gpurun_out/r02t_c$c.err
done
echo done
