"""Tuning sweep of the tile pipeline (stages x tile size x gather chunk).

Here (CPU):   python tools/variant_sweep.py build     -> lib/variants/libf3rg_<name>.so
On the GPU:   python tools/variant_sweep.py run       -> one line per variant: time per
              config-2 solve (graph mode) and per-kernel GB/s (eager profile)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# compile-time knobs of spmv.cuh: CTAs per SM (register budget), fp16 pipeline
# depth, gather chunk (u32/D16 streams, and P16), fp16 tile size
VARIANTS = {
    "m2_s3_c16": ["F3RG_TILE_MINB=2", "F3RG_D16_STAGES=3", "F3RG_CHUNK=16"],
    "m3_s2_c16": ["F3RG_TILE_MINB=3", "F3RG_D16_STAGES=2", "F3RG_CHUNK=16"],
    "m3_s2_c8": ["F3RG_TILE_MINB=3", "F3RG_D16_STAGES=2", "F3RG_CHUNK=8", "F3RG_P16_CHUNK=8"],
    "m4_t5k": ["F3RG_TILE_MINB=4", "F3RG_TNNZ16=5120"],
    # short-row (7-point, configs 1/3/4) candidates: more CTAs per SM, one chunk per row
    "m5_c8": ["F3RG_TILE_MINB=5", "F3RG_CHUNK=8", "F3RG_P16_CHUNK=8", "F3RG_TNNZ16=3328",
              "F3RG_TNNZ32=2560", "F3RG_TNNZ64=1536"],
    "m6_c8": ["F3RG_TILE_MINB=6", "F3RG_CHUNK=8", "F3RG_P16_CHUNK=8", "F3RG_TNNZ16=2816",
              "F3RG_TNNZ32=2048", "F3RG_TNNZ64=1280"],
    "m4_c8": ["F3RG_TILE_MINB=4", "F3RG_CHUNK=8", "F3RG_P16_CHUNK=8", "F3RG_TNNZ16=4352",
              "F3RG_TNNZ32=3200", "F3RG_TNNZ64=2048"],
    # gather-heavy (config 5): smaller tiles leave more of the SM's 256 KB to L1
    "g_half": ["F3RG_TNNZ16=3584", "F3RG_TNNZ32=3456", "F3RG_TNNZ64=2048"],
    "g_quarter": ["F3RG_TNNZ16=1792", "F3RG_TNNZ32=1728", "F3RG_TNNZ64=1024"],
    "g_half_c24": ["F3RG_TNNZ16=3584", "F3RG_TNNZ32=3456", "F3RG_TNNZ64=2048", "F3RG_CHUNK=24"],
}
if os.environ.get("SWEEP"):
    VARIANTS = {k: v for k, v in VARIANTS.items() if k in os.environ["SWEEP"].split(",")}

CHILD = r"""
import os, sys, time, json, torch
sys.path.insert(0, %r)
import paper_2505_20719_b200 as f
from paper_2505_20719_b200 import problems
p = problems.problem(int(os.environ.get("SWEEP_CONFIG", "2")))
reps = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values))
s = f.build(f.parse_solver_spec("F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > identity"), reps, f.IdentityPrecond(p.n))
b = torch.from_numpy(p.b).cuda()
o = f.RunOptions(tol=1e-10)
for _ in range(2):
    s.reset(); s.run(b, o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    s.reset(); r = s.run(b, o)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
s.set_profile(True); s.reset(); s.run(b, o); s.set_profile(False)
prof = {k[0]: round(k[3] / k[2] / (k[1] / k[2] * 1e-3) / 1e9) for k in s.profile()}
tot = {k[0]: round(k[1], 2) for k in s.profile()}
print(json.dumps({"ms": round(ms, 2), "outer": r.report.outer_iterations, "gbs": prof, "kernel_ms": tot}))
""" % ROOT


def build():
    from paper_2505_20719_b200 import buildlib
    for name, defs in VARIANTS.items():
        buildlib.build_lib(defines=defs, name=name)
        print("built", name, flush=True)


def run():
    names = list(VARIANTS)
    if os.environ.get("SWEEP_DEFAULT"):
        names = ["default"] + names
    for name in names:
        lib = os.path.join(ROOT, "paper_2505_20719_b200", "lib", "variants", f"libf3rg_{name}.so")
        env = dict(os.environ, F3RG_LIB=lib) if name != "default" else dict(os.environ)
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-400:]
        print(name, line, flush=True)


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
