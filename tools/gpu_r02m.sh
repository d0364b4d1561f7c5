# round-2 capture after the L2 hints + D16 gap-1: full GPU suite, the default bench
# (config 5) with its CPU baseline, the reference arm, ncu captures for the traffic table
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nproc > gpurun_out/r02m_nproc.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02m_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02m_pytest.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r02m_bench.json 2> gpurun_out/r02m_bench.err
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02m_ref.json 2> gpurun_out/r02m_ref.err
for c in 5 2 4; do
  for k in k_richardson k_spmv_dots; do
    timeout 900 ncu --set full --clock-control none -k regex:$k --launch-skip 20 -c 1 -f -o /tmp/r02m_c${c}_$k python tools/profile_solve.py --config $c --solves 2 > gpurun_out/r02m_ncu_c${c}_$k.log 2>&1
    ncu -i /tmp/r02m_c${c}_$k.ncu-rep --page raw --csv > gpurun_out/r02m_ncu_c${c}_${k}_raw.csv 2>&1
  done
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02m_launches_c5.csv python tools/profile_solve.py --config 5 --solves 2 > gpurun_out/r02m_launches_c5.log 2>&1
echo done
