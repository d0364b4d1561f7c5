# L2 eviction priorities: config-5 A/B over {tiles, SELL} x {hints on, off}; config 2/3 regression
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sell.py tests/test_gpu_kernels.py -m gpu -x -q > gpurun_out/r02l_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02l_pytest.log
for v in "F3RG_SELL=0" "F3RG_SELL=0 F3RG_L2HINT=0" "F3RG_SELL=1" "F3RG_SELL=1 F3RG_L2HINT=0"; do
  tag=$(echo $v | tr ' =' '_-')
  env $v timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02l_c5_$tag.json 2> gpurun_out/r02l_c5_$tag.err
done
for c in 2 3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02l_c${c}_hint.json 2> /dev/null
  F3RG_L2HINT=0 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02l_c${c}_nohint.json 2> /dev/null
done
echo done
