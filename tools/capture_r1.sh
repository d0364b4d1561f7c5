# Round-1 evidence capture (run on the GPU box from the repo root):
#   bench line, per-launch timing list of one solve, full ncu capture of the top kernels
set -x
mkdir -p gpurun_out/r1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r1/bench.json 2> gpurun_out/r1/bench.err; echo rc=$? >> gpurun_out/r1/bench.err
timeout 300 python tools/profile_solve.py --solves 2 > gpurun_out/r1/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1/launches.csv python tools/profile_solve.py --solves 2 > gpurun_out/r1/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_spmv_dots<.int.0, .int.0, .int.1|k_richardson<.int.0, .int.0, .int.1|k_cgs<.int.1|k_spmv_dots<.int.1, .int.1, .int.1" \
  -s 100 -c 6 -o gpurun_out/r1/full python tools/profile_solve.py --solves 1 > gpurun_out/r1/ncu_full.log 2>&1
echo done
