# Evidence capture for profiles/ (run on the GPU box from the repo root):
#   bash tools/capture_round.sh <tag>
# bench line (with the CPU reference sample), a per-launch timing list of one solve,
# and a full ncu capture of the top kernels. Each ncu pass runs only after the same
# command has exited 0 without ncu.
set -x
T=${1:-rNN}
D=gpurun_out/$T
mkdir -p $D
timeout 900 python bench.py --steps 5 --warmup 3 > $D/bench.json 2> $D/bench.err; echo rc=$? >> $D/bench.err
timeout 300 python tools/profile_solve.py --solves 2 > $D/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches.csv \
  python tools/profile_solve.py --solves 2 > $D/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_spmv_dots<.int.0, .int.0, .int.1|k_richardson<.int.0, .int.0, .int.1|k_cgs<.int.1|k_spmv_dots<.int.1, .int.1, .int.1" \
  -s 100 -c 4 -o $D/full python tools/profile_solve.py --solves 1 > $D/ncu_full.log 2>&1
# summaries on the box (gpurun copies back at most 64 MiB of gpurun_out/)
python tools/summarize_ncu.py launches $D/launches.csv --solve 2 > $D/launches.md 2>&1
python tools/summarize_ncu.py full $D/full.ncu-rep > $D/full.md 2>&1
ncu -i $D/full.ncu-rep --page raw --csv > $D/full_raw.csv 2>/dev/null
[ $(stat -c %s $D/full.ncu-rep 2>/dev/null || echo 0) -gt 40000000 ] && rm -f $D/full.ncu-rep
du -sh gpurun_out
echo done
