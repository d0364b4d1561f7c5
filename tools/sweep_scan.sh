# A/B of the ILU/IC sweep knobs (run on the GPU box)
mkdir -p gpurun_out/p9
timeout 300 python -m pytest tests/test_gpu_precond.py -x -q -p no:cacheprovider --timeout 200 -k "apply or richardson" > gpurun_out/p9/pytest.log 2>&1; echo rc=$? >> gpurun_out/p9/pytest.log; tail -3 gpurun_out/p9/pytest.log
F3RG_SWEEP_POLL=1 timeout 300 python -m pytest tests/test_gpu_precond.py -x -q -p no:cacheprovider --timeout 200 -k "apply" 2>&1 | tail -1
for po in 0 1; do for ah in 4 8 32 100000; do for c in 1 2; do
F3RG_SWEEP_POLL=$po F3RG_SWEEP_AHEAD=$ah F3RG_SWEEP_CTAS=$c timeout 200 python tools/precond_timing.py --config 2 --apply-only > gpurun_out/p9/t.json 2>&1
echo "poll=$po ahead=$ah ctas=$c $(python -c "import json;d=json.load(open('gpurun_out/p9/t.json'));print(round(d['apply_ms'],3), round(d['us_per_level'],3))")"
done; done; done
for po in 0 1; do F3RG_SWEEP_POLL=$po timeout 200 python tools/precond_timing.py --config 2 --grid 16 --apply-only > gpurun_out/p9/g16.json 2>&1
echo "grid16 poll=$po $(python -c "import json;d=json.load(open('gpurun_out/p9/g16.json'));print(round(d['apply_ms'],3), round(d['us_per_level'],3))")"; done
