#!/usr/bin/env python
"""bench.py -- time-to-solution of the fp16-F3R solve (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One "step" = one complete fp16-F3R solve (F100:f64/f64 > F8:f32/f32 > F4:f16/f32 >
R2:f16,c=64, identity M) of BASELINE config 2 (27-point 128^3, n = 2,097,152,
nnz = 55,742,968, x_true ~ U[-1,1] seed 1) to relative residual 1e-10, from a
zero initial guess, inputs resident in HBM. The matrix replicas (A16 + indices
alone: 334 MB) exceed the 126 MB L2, so no explicit flush is needed between steps.

Printed JSON line (rank 0): value = mean time-to-solution (s, lower is better),
e2e = the same solve through the C ABI with host buffers (pinned b in, x out),
roofline = the dominant kernel's achieved HBM GB/s (algorithmic bytes, SURVEY.md
§8(d)) over the measured copy peak, cpu_baseline = the unmodified reference CPU
solver on this host (one outer iteration, extrapolated to the full count).

--impl reference: the reference's own CPU implementation (oracle/_ref, built from
/root/reference/proj/src) on all host threads; each step = one outer iteration
of the same config, value extrapolated to the reference's full outer count.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

SPEC = "F100:f64/f64 > F8:f32/f32 > F4:f16/f32 > R2:f16,c=64 > identity"
METRIC = "time-to-solution to rel. residual 1e-10 (s)"
TOL = 1e-10


def spec_for(args):
    """the timed nest: M = identity (the north-star path) or, with --precond, the
    reference bench's default block-Jacobi M (4 blocks, alpha 1, fp16 factors;
    include/f3r/bench.hpp:31-34, src/bench.cpp:160-177)"""
    if args.precond == "identity":
        return SPEC
    return SPEC.rsplit(">", 1)[0] + f"> {args.precond}(blocks=4,alpha=1,prec=f16)"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index=0):
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None
        self.index = index

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        try:
            rows = [r.split(", ") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in rows]
        mx = float(rows[0][1])
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 3 + i and "Active" in r[3 + i]
                          and "Not" not in r[3 + i]})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows)}


# DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) from the
# committed `ncu --set full` capture of config 2 (profiles/r01_ncu_full.md, P16 rows)
TRAFFIC = {"richardson[f16,f16,f32]": 256101120.0, "spmv_dots[f16,f16,f32]": 261074688.0}


def streams_matrix(kernel):
    return kernel.split("[")[0] in ("richardson", "spmv_dots", "spmv", "residual")


def column_stream_saving(p):
    """u32 column bytes minus D16 bytes (u16 deltas + u32 first column per row) when
    the engine uses the D16 stream (every in-row gap < 2^16, F3RG_COLUMNS unset)."""
    if os.environ.get("F3RG_COLUMNS") == "u32" or p.nnz == 0:
        return 0.0
    rp = p.row_ptr.astype(np.int64)
    gaps = np.diff(p.col_idx.astype(np.int64))
    inrow = np.ones(len(gaps), dtype=bool)
    inrow[rp[1:-1][(rp[1:-1] > 0) & (rp[1:-1] < p.nnz)] - 1] = False
    if len(gaps) and gaps[inrow].max(initial=0) > 0xFFFF:
        return 0.0
    return 4.0 * p.nnz - (2.0 * p.nnz + 4.0 * p.n)


def spmv_per_precision(f, torch, reps, p, reps_n=20):
    """The metric's second half, "SpMV HBM GB/s per precision": the standalone device
    SpMV (f3rg_spmv, reference spmv src/csr.cpp:138-147) at each precision triple of
    the path, timed with CUDA events over `reps_n` back-to-back launches (inputs
    resident; the 223-446 MB matrix streams exceed the 126 MB L2). GB/s by SURVEY
    8(d)'s algorithmic bytes nnz (sA + 4) + 4 (n + 1) + n (sx + sy) -- the reference's
    u32 CSR -- and by the bytes actually streamed (D16/P16 column streams)."""
    size = {0: 2, 1: 4, 2: 8}
    peak, _ = _peaks()
    saving = column_stream_saving(p)
    out = []
    for pa, px, py, role in ((2, 2, 2, "L1 / true residual"), (1, 1, 1, "L2"), (0, 1, 1, "L3"),
                             (0, 0, 0, "Richardson operand")):
        x = f.DenseVector(torch.rand(p.n, device="cuda", dtype=torch.float64).to(f.torch_dtype(px)))
        y = f.DenseVector(p.n, f.Precision(py))
        A = reps.at(f.Precision(pa))
        for _ in range(3):
            f.spmv(A, x, y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps_n):
            f.spmv(A, x, y)
        e1.record()
        torch.cuda.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / reps_n
        algo = p.nnz * (size[pa] + 4) + 4 * (p.n + 1) + p.n * (size[px] + size[py])
        streamed = algo - saving
        out.append({"precision": f"A f{8 * size[pa]}, x f{8 * size[px]}, y f{8 * size[py]}", "role": role,
                    "us": round(us, 2), "algorithmic_gbs": round(algo / us / 1e3, 1),
                    "streamed_gbs": round(streamed / us / 1e3, 1), "frac": round(algo / us / 1e3 / peak, 4),
                    "frac_streamed": round(streamed / us / 1e3 / peak, 4)})
    return out


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def reference_runs():
    path = os.path.join(ROOT, "tests", "golden", "reference_runs.json")
    try:
        return json.load(open(path))
    except Exception:
        return {}


def cpu_reference_sample(p, outer_full: int, threads: int, sample_outer: int = 1, args=None):
    """Times the UNMODIFIED reference solve for `sample_outer` outer iterations
    (RunOptions.max_outer_total, include/f3r/nesting.hpp:35); returns seconds per
    outer iteration and the extrapolated time-to-solution."""
    from oracle_bind import Reference
    r = Reference()
    r.set_threads(threads)
    m = r.matrix(p.row_ptr, p.col_idx, p.values)
    M = _ref_m(r, m, args)
    rep = r.solve(m, spec_for(args) if args else SPEC, p.b, tol=TOL, max_outer_total=sample_outer, want_x=False,
                  precond=M)
    per_outer = rep.wall_seconds / max(1, rep.outer_iterations)
    return per_outer, per_outer * outer_full, rep


def _ref_m(r, m, args):
    """the reference's own BlockJacobiIlu0::factorize for --precond (untimed setup, as
    the reference bench times factorisation apart, src/bench.cpp:202-207)"""
    if args is None or args.precond == "identity":
        return None
    return r.ilu(m, 4, 1.0, args.precond == "ic0", 0)


def _mode_key(args):
    return "fp16-f3r" if args.precond == "identity" else f"fp16-f3r-{args.precond}"


def run_reference_arm(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    from paper_2505_20719_b200 import problems
    p = problems.problem(args.config)
    threads = os.cpu_count()
    runs = reference_runs().get(f"config{args.config}/{_mode_key(args)}", {})
    outer_full = int(runs.get("outer_iterations", 0)) or None
    from oracle_bind import Reference, reference_available
    if not reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libf3r_ref.so not built"}))
        return
    r = Reference()
    r.set_threads(threads)
    m = r.matrix(p.row_ptr, p.col_idx, p.values)
    M = _ref_m(r, m, args)
    spec = spec_for(args)
    if outer_full is None:  # no committed full run for this config: measure it once
        full = r.solve(m, spec, p.b, tol=TOL, want_x=False, precond=M)
        outer_full = full.outer_iterations
    for _ in range(min(args.warmup, 1)):
        r.solve(m, spec, p.b, tol=TOL, max_outer_total=1, want_x=False, precond=M)
    times = []
    for _ in range(args.steps):
        rep = r.solve(m, spec, p.b, tol=TOL, max_outer_total=1, want_x=False, precond=M)
        times.append(rep.wall_seconds)
    per_outer = float(np.mean(times))
    value = per_outer * outer_full
    sample = (f"1 outer iteration (of {outer_full}) of the reference fp16-F3R solve per step, "
              f"config {args.config}; value = mean x {outer_full}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": min(args.warmup, 1), "ms_per_step": per_outer * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "mixed f64/f32/f16 (software binary16)",
        "data": "synthetic", "config": _config(args, p),
        "cpu_baseline": {"value": value, "unit": "s", "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def _config(args, p):
    mname = "identity" if args.precond == "identity" else f"block-Jacobi {args.precond}, 4 blocks, fp16 factors"
    return {"workload": f"BASELINE config {args.config}: fp16-F3R solve to 1e-10 (M = {mname})", "n": p.n,
            "nnz": p.nnz, "solver": spec_for(args), "problem": p.name, "tol": TOL,
            "l2_flush": "none: working set (A16+idx 334 MB, A32+idx 446 MB) exceeds the 126 MB L2",
            "parallelism": f"dp{args.gpus}" if args.gpus > 1 else "single GPU"}


def run_partitioned(args):
    """N > 1 (or --partition): ONE config-2 system row-block partitioned over the
    ranks: NCCL point-to-point halos + allgather of rank-local totals
    inside the solve; strong scaling (total work fixed). Timed as the max over ranks
    of CUDA-event time per solve."""
    import torch
    import torch.distributed as dist

    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import partition, problems

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("cpu:gloo,cuda:nccl", rank=rank, world_size=world)
    p = problems.problem(args.config)
    a = f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values)
    uid = [partition.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    part = partition.NcclPartition(a, SPEC, world, rank, uid[0])
    pl = part.plan
    opts = f.RunOptions(tol=TOL)
    b_own = torch.from_numpy(p.b[pl.r0:pl.r1].copy()).cuda()
    x_own = torch.zeros(pl.r1 - pl.r0, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    for _ in range(max(args.warmup, 0)):
        part.reset()
        rep = part.run(b_own, x_own, opts, sp)
    assert rep.converged and rep.final_true_residual <= TOL, rep
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            part.reset()
            rep = part.run(b_own, x_own, opts, sp)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    dist.barrier()
    # e2e: host b slice in, host x slice out, every step
    b_host = torch.from_numpy(p.b[pl.r0:pl.r1].copy()).pin_memory()
    x_host = torch.empty(pl.r1 - pl.r0, dtype=torch.float64).pin_memory()
    e2e_t = []
    for _ in range(max(1, min(args.steps, 5))):
        dist.barrier()
        t0 = time.perf_counter()
        part.reset()
        b_own.copy_(b_host, non_blocking=True)
        rep = part.run(b_own, x_own, opts, sp)
        x_host.copy_(x_own, non_blocking=True)
        torch.cuda.synchronize()
        e2e_t.append(time.perf_counter() - t0)
    e2 = torch.tensor([float(np.mean(e2e_t))], device="cuda")
    dist.all_reduce(e2, op=dist.ReduceOp.MAX)
    # per-kernel timing of one eager solve on every rank (the exchanges pair up):
    # launch count and the top kernel's roofline, rank 0's
    part.solver.set_profile(True)
    part.reset()
    part.run(b_own, x_own, opts, sp)
    part.solver.set_profile(False)
    prof = part.solver.profile()
    launches = int(sum(k[2] for k in prof))
    streaming = [k for k in prof if k[3] > 0]
    top = max(streaming, key=lambda k: k[1])
    peak, peak_kind = _peaks()
    per_launch_ms = top[1] / top[2]
    gbs = top[3] / top[2] / (per_launch_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "mixed f64/f32/f16", "data": "synthetic",
        "config": dict(_config(args, p), parallelism=f"row-block partition over {world} GPU(s), NCCL halos"),
        "outer_iterations": rep.outer_iterations, "final_true_residual": rep.final_true_residual,
        "e2e": {"value": float(e2.item()), "unit": "s", "h2d_bytes_per_step": int(p.n * 8),
                "d2h_bytes_per_step": int(p.n * 8)},
        "gpu_launches": launches * args.steps, "clocks": clk.summary(),
        "roofline": {"bound": "hbm", "kernel": top[0], "achieved": round(gbs, 1), "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": round(gbs / peak, 4), "traffic": None,
                     "bytes": "streamed bytes of rank 0's rows (its ext-layout CSR)",
                     "avg_launch_us": per_launch_ms * 1e3},
        "partition": {"rows_rank0": pl.r1 - pl.r0, "halo_rank0": pl.n_lo + pl.n_hi},
    }
    if rank == 0:
        print(json.dumps(line))
    del part
    dist.destroy_process_group()


def run_ours(args):
    import torch

    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import problems

    rank, local, world = dist_env()
    if world > 1 or args.partition:
        if args.precond != "identity":
            raise SystemExit("--precond: the row-block partition runs M = identity only (DESIGN.md section 6c)")
        return run_partitioned(args)
    torch.cuda.set_device(local)
    p = problems.problem(args.config)
    reps = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values))
    if args.precond == "identity":
        M = f.IdentityPrecond(p.n)
    else:  # factorised once, untimed (the reference bench times it apart)
        M = f.BlockJacobiIlu0.factorize(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values),
                                        f.IluConfig(4, 1.0, args.precond == "ic0", f.Precision.P16))
    solver = f.build(f.parse_solver_spec(spec_for(args)), reps, M)
    opts = f.RunOptions(tol=TOL)
    b_dev = torch.from_numpy(p.b).cuda()
    stream = torch.cuda.current_stream()

    # every step is a fresh solve: the reference's run_once builds a new
    # ComposedSolver per repeat (src/bench.cpp:210-219); reset() restores that state
    for _ in range(max(args.warmup, 0)):
        solver.reset()
        run = solver.run(b_dev, opts)
    solver.reset()
    run = solver.run(b_dev, opts)
    outer = run.report.outer_iterations
    assert run.report.converged and run.report.final_true_residual <= TOL, run.report

    # ---- timed region: K full solves, device-resident inputs ----
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            solver.reset()
            run = solver.run(b_dev, opts)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    if not (run.report.converged and run.report.final_true_residual <= TOL):
        raise SystemExit(f"timed solve did not converge: {run.report}")

    # ---- e2e: through the C ABI with host buffers (pinned b in, x out) ----
    b_host = torch.from_numpy(p.b).pin_memory().numpy()
    x_host = torch.empty(p.n, dtype=torch.float64).pin_memory().numpy()
    e2e_t = []
    # one untimed warm-up through the host-buffer entry point (its first call
    # builds the pinned-staging graph), then the timed steps
    for it in range(1 + max(1, min(args.steps, 5))):
        t0 = time.perf_counter()
        solver.reset()
        r2 = solver.run(b_host, opts, out=x_host)
        if it:
            e2e_t.append(time.perf_counter() - t0)
    e2e = float(np.mean(e2e_t))
    assert r2.report.converged

    # ---- per-kernel timing (CUDA events around every launch, eager mode) ----
    solver.set_profile(True)
    solver.reset()
    solver.run(b_dev, opts)
    solver.set_profile(False)
    prof = solver.profile()
    total_ms = sum(k[1] for k in prof)
    launches = int(sum(k[2] for k in prof))
    # roofline of the top STREAMING kernel (the ILU/IC sweeps are latency-bound:
    # reported apart, per dependency level)
    streaming = [k for k in prof if not k[0].startswith("precond_")]
    top = max(streaming, key=lambda k: k[1])
    peak, peak_kind = _peaks()
    per_launch_ms = top[1] / top[2]
    # profile bytes are what the kernel streams (D16 column stream when in use);
    # SURVEY.md 8(d)'s algorithmic unit counts the reference's u32 CSR instead
    per_launch_bytes = top[3] / top[2]
    algo_bytes = per_launch_bytes + (column_stream_saving(p) if streams_matrix(top[0]) else 0.0)
    achieved = algo_bytes / (per_launch_ms * 1e-3) / 1e9
    streamed = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
    breakdown = sorted(prof, key=lambda k: -k[1])
    kernels = [{"kernel": k[0], "share": round(k[1] / total_ms, 4), "launches": k[2],
                "avg_us": round(1e3 * k[1] / k[2], 2),
                "gbs": round(k[3] / k[2] / (k[1] / k[2] * 1e-3) / 1e9, 1)} for k in breakdown[:8]]

    line = {
        "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "mixed f64/f32/f16", "data": "synthetic", "config": _config(args, p),
        "outer_iterations": outer, "final_true_residual": run.report.final_true_residual,
        "roofline": {"bound": "hbm", "kernel": top[0], "achieved": round(achieved, 1), "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": TRAFFIC.get(top[0]), "algorithmic_bytes_per_launch": algo_bytes,
                     "streamed_bytes_per_launch": per_launch_bytes, "achieved_streamed": round(streamed, 1),
                     "frac_streamed": round(streamed / peak, 4), "avg_launch_us": per_launch_ms * 1e3},
        "kernels": kernels,
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": int(p.n * 8), "d2h_bytes_per_step": int(p.n * 8)},
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
    }
    line["spmv_per_precision"] = spmv_per_precision(f, torch, reps, p)
    pre = [k for k in prof if k[0].startswith("precond_")]
    if pre:
        lv = M.sweep_levels()
        apply_ms = pre[0][1] / pre[0][2]
        line["precond"] = {"kernel": pre[0][0], "share": round(pre[0][1] / total_ms, 4), "applies": pre[0][2],
                           "apply_ms": round(apply_ms, 4), "sweep_levels": list(lv),
                           "us_per_level": round(1e3 * apply_ms / (lv[0] + lv[1]), 3), "bound": "latency"}
    if not args.no_cpu_baseline:
        try:
            threads = os.cpu_count()
            per_outer, extrap, rep = cpu_reference_sample(p, outer, threads, args=args)
            line["cpu_baseline"] = {"value": extrap, "unit": "s", "cores": threads, "kind": "reference",
                                    "sample": f"1 outer iteration of the unmodified reference fp16-F3R solve "
                                              f"(M = {args.precond}; {per_outer:.2f} s), extrapolated "
                                              f"x{outer} outer iterations"}
        except Exception as e:  # keep the GPU line even if the CPU leg fails
            line["cpu_baseline"] = {"value": None, "unit": "s", "cores": os.cpu_count(), "kind": "reference",
                                    "sample": f"failed: {e}"}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--precond", default="identity", choices=["identity", "ic0", "ilu0"],
                    help="primary preconditioner M of the nest (default identity, the north-star path)")
    ap.add_argument("--partition", action="store_true",
                    help="use the row-block partitioned NCCL path even on one GPU")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
