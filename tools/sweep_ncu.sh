# ncu capture of one forward and one backward ILU/IC sweep launch (run on the GPU box)
mkdir -p gpurun_out/p6
timeout 200 python tools/precond_timing.py --config 2 --apply-only > gpurun_out/p6/plain.json 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_sweep" -s 4 -c 2 -o gpurun_out/p6/sweep \
  python tools/precond_timing.py --config 2 --apply-only > gpurun_out/p6/ncu.log 2>&1
tail -3 gpurun_out/p6/ncu.log
ls -la gpurun_out/p6
