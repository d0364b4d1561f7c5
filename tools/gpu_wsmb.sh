# windowed SELL microbenchmark on the box: small config-5 sample with the row-tile cross-check, then full size
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python - <<'P' > gpurun_out/wsmb_cache.log 2>&1
from paper_2505_20719_b200 import csr_cache
print(csr_cache.ensure(5, 300000)); print(csr_cache.ensure(5))
P
for b in ${WSMB_BINS:-build/wsell_microbench}; do
  echo "== $b small" >> gpurun_out/wsmb.log
  WS_CHECK=1 timeout 300 $b /tmp/f3rg_cache/config5_300000.csr 5 >> gpurun_out/wsmb.log 2>&1; echo "rc=$?" >> gpurun_out/wsmb.log
  echo "== $b full" >> gpurun_out/wsmb.log
  WS_CHECK=${WSMB_CHECK_FULL:-1} timeout 900 $b /tmp/f3rg_cache/config5_20000000.csr 10 >> gpurun_out/wsmb.log 2>&1; echo "rc=$?" >> gpurun_out/wsmb.log
done
echo done
