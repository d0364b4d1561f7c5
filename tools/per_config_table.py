"""Markdown table of the per-config bench lines written by tools/per_config.sh:
    python tools/per_config_table.py gpurun_out/<tag> [gpurun_out/<baseline tag>]
time to solution, outer count, the top kernels and the standalone SpMV rate per
precision triple (streamed bytes / the measured copy peak)."""
import json
import os
import sys


def load(d, c):
    try:
        return json.loads(open(os.path.join(d, f"config{c}.json")).read().strip().splitlines()[-1])
    except (OSError, ValueError, IndexError):
        return None


def main():
    d = sys.argv[1]
    base = sys.argv[2] if len(sys.argv) > 2 else None
    print("| config | n / nnz | time to solution | before | outer | final residual | top kernel (share, avg us, frac of peak) |")
    print("|---|---|---|---|---|---|---|")
    for c in range(1, 6):
        x = load(d, c)
        if not x:
            continue
        b = load(base, c) if base else None
        k = x["kernels"][0]
        cfg = x["config"]
        print(f"| {c} | {cfg['n']:,} / {cfg['nnz']:,} | **{x['ms_per_step']:.2f} ms** | "
              f"{(f'{b['ms_per_step']:.2f} ms') if b else '-'} | {x['outer_iterations']} | "
              f"{x['final_true_residual']:.2e} | {k['kernel']} ({k['share']:.2f}, {k['avg_us']:.1f}, "
              f"{x['roofline']['frac']:.2f}) |")
    print()
    print("Standalone SpMV per precision triple: us per launch, streamed GB/s, fraction of the measured copy peak")
    print()
    print("| config | A f64, x f64, y f64 | A f32, x f32, y f32 | A f16, x f32, y f32 | A f16, x f16, y f16 |")
    print("|---|---|---|---|---|")
    for c in range(1, 6):
        x = load(d, c)
        if not x:
            continue
        cells = [f"{s['us']:.1f} us, {s['streamed_gbs']:.0f} GB/s, {s['frac_streamed']:.2f}"
                 for s in x["spmv_per_precision"]]
        print(f"| {c} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
