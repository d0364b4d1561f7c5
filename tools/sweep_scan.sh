# sweep chunk variants (run on the GPU box)
mkdir -p gpurun_out/pv
for v in "" variants/libf3rg_chunk8.so variants/libf3rg_chunk32.so; do
  lib=""; [ -n "$v" ] && lib="$PWD/paper_2505_20719_b200/lib/$v"
  for cfg in "2" "2 --grid 16" "4"; do
    F3RG_LIB=$lib timeout 300 python tools/precond_timing.py --config $cfg --apply-only > gpurun_out/pv/t.json 2>&1
    echo "lib=${v:-default} cfg=$cfg $(python -c "import json;d=json.load(open('gpurun_out/pv/t.json'));print(round(d['apply_ms'],3), round(d['us_per_level'],3), d['sweep_levels'])")"
  done
done
