# Per-config bench lines (configs 1-5 of BASELINE.json, fp16-F3R, M = identity,
# 1 GPU; run on the GPU box from the repo root):  bash tools/per_config.sh <tag>
T=${1:-rNN}
D=gpurun_out/$T
mkdir -p $D
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline \
    > $D/config$c.json 2> $D/config$c.err; echo rc=$? >> $D/config$c.err
done
echo done
