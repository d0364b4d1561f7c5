# Evidence for the block-Jacobi M (run on the GPU box): bench line with --precond ic0,
# the drop-in tests, and an ncu capture of one forward + one backward sweep.
D=gpurun_out/${1:-pc}
mkdir -p $D
timeout 600 python -m pytest tests/test_dropin.py tests/test_gpu_precond.py -q -p no:cacheprovider --timeout 300 > $D/pytest.log 2>&1; echo rc=$? >> $D/pytest.log
timeout 900 python bench.py --precond ic0 --steps 3 --warmup 3 > $D/bench_ic0.json 2> $D/bench_ic0.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $D/bench_identity.json 2> $D/bench_identity.err
timeout 200 python tools/precond_timing.py --config 2 --apply-only > $D/apply.json 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_sweep" -s 4 -c 2 -o $D/sweep \
  python tools/precond_timing.py --config 2 --apply-only > $D/ncu.log 2>&1
ncu -i $D/sweep.ncu-rep --page raw --csv > $D/sweep_raw.csv 2>/dev/null
ncu -i $D/sweep.ncu-rep --page source --csv --kernel-name regex:k_sweep_fwd --print-source sass > $D/sweep_fwd_source.csv 2>/dev/null
tail -3 $D/pytest.log; head -c 600 $D/bench_ic0.json; echo; head -c 300 $D/bench_identity.json; echo
