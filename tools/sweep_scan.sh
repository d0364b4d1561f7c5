# block vs global sweep modes (run on the GPU box)
mkdir -p gpurun_out/pb
timeout 600 python -m pytest tests/test_gpu_precond.py -x -q -p no:cacheprovider --timeout 300 > gpurun_out/pb/pytest.log 2>&1; echo rc=$? >> gpurun_out/pb/pytest.log; tail -3 gpurun_out/pb/pytest.log
for mode in block global; do for cfg in "2" "2 --grid 16" "1" "4"; do
F3RG_SWEEP_MODE=$mode timeout 300 python tools/precond_timing.py --config $cfg --apply-only > gpurun_out/pb/t.json 2>&1
echo "mode=$mode cfg=$cfg $(python -c "import json;d=json.load(open('gpurun_out/pb/t.json'));print(round(d['apply_ms'],3), round(d['us_per_level'],3), d['sweep_levels'])")"
done; done
for b in 1 16 148; do timeout 300 python tools/precond_timing.py --config 2 --blocks $b --apply-only > gpurun_out/pb/t.json 2>&1
echo "block-mode cfg2 blocks=$b $(python -c "import json;d=json.load(open('gpurun_out/pb/t.json'));print(round(d['apply_ms'],3), round(d['us_per_level'],3), d['sweep_levels'])")"; done
