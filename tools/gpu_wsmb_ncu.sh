# ncu of the microbenchmark's kernels (full-size config 5): raw + source pages per kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "from paper_2505_20719_b200 import csr_cache; print(csr_cache.ensure(5))" > gpurun_out/wsmb_cache.log 2>&1
B=${WSMB_BIN:-build/wsell_microbench}
for k in ${WSMB_KERNELS:-kb_spmv kb_dots}; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 4 -c 1 -f -o /tmp/wsmb_$k $B /tmp/f3rg_cache/config5_20000000.csr 3 ${WSMB_ONLY:-SE} > gpurun_out/wsmb_ncu_$k.log 2>&1
  ncu -i /tmp/wsmb_$k.ncu-rep --page raw --csv > gpurun_out/wsmb_ncu_${k}_raw.csv 2>&1
  ncu -i /tmp/wsmb_$k.ncu-rep --page source --csv > gpurun_out/wsmb_ncu_${k}_source.csv 2>&1
done
echo done
