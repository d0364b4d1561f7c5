#!/usr/bin/env python
"""bench.py -- time-to-solution of the fp16-F3R solve (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

One "step" = one complete fp16-F3R solve (F100:f64/f64 > F8:f32/f32 > F4:f16/f32 >
R2:f16,c=64, identity M) to relative residual 1e-10 from a zero initial guess,
inputs resident in HBM. Default workload: BASELINE config 5, the largest
configuration that fits one GPU (unstructured n = 20,000,000, ~6.0e8 entries,
seed 4); --config 1..4 select the others. Every config's matrix streams exceed the
126 MB L2 except config 1's (L2-resident), so no flush is
needed between steps. Inputs come from the binary CSR cache (csr_cache.py,
written once per host by lib/f3rg_gen), the same bytes for both arms.

Printed JSON line (rank 0): value = mean time-to-solution (s, lower is better),
e2e = the same solve through the C ABI with host buffers (pinned b in, x out),
roofline = the dominant kernel's achieved HBM GB/s (algorithmic bytes, SURVEY.md
§8(d)) over the measured copy peak, cpu_baseline = the unmodified reference CPU
solver on this host: a bounded sample (SAMPLES_PER_OUTER) scaled by its own
recorded outer count.

--impl reference: the reference's own CPU implementation (oracle/_ref, built from
/root/reference/proj/src) on all host threads, fed from the binary CSR cache
(this process never maps libf3rg.so); each step = the same bounded sample.
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


PSIZE = {0: 2, 1: 4, 2: 8}
PNAME = {"f16": 0, "f32": 1, "f64": 2}


def traffic_table():
    """measured DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
    of the top kernels, per config, from the committed `ncu --set full` captures
    (profiles/traffic.json, written by tools/summarize_ncu.py)"""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except Exception:
        return {}


def streams_matrix(kernel):
    return kernel.split("[")[0] in ("richardson", "spmv_dots", "spmv", "residual")


def column_stream_saving(reps, p, pa):
    """the reference's u32-CSR bytes of one pass over replica pa (SURVEY 8(d):
    nnz (sA + 4) + 4 (n + 1)) minus the bytes the device actually streams (its
    compressed column stream, f3rg_matrix_stream_bytes)"""
    return float(p.nnz * (PSIZE[pa] + 4) + 4 * (p.n + 1) - reps.stream_bytes(pa))


def spmv_per_precision(f, torch, reps, p, reps_n=20):
    """The metric's second half, "SpMV HBM GB/s per precision": the standalone device
    SpMV (f3rg_spmv, reference spmv src/csr.cpp:138-147) at each precision triple of
    the path, timed with CUDA events over `reps_n` back-to-back launches (inputs
    resident; the 223-446 MB matrix streams exceed the 126 MB L2). GB/s by SURVEY
    8(d)'s algorithmic bytes nnz (sA + 4) + 4 (n + 1) + n (sx + sy) -- the reference's
    u32 CSR -- and by the bytes actually streamed (D16/P16 column streams)."""
    size = PSIZE
    peak, _ = _peaks()
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
        streamed = algo - column_stream_saving(reps, p, pa)
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


# Reference CPU sample per step, sized so one step is ~5-15 s on the box's cores:
# a full outer iteration (configs 1-2), one L2 Arnoldi step = 1/8 of an outer
# iteration (configs 3-4: one F4 > R2 invocation below it), or one L3 Arnoldi step
# = 1/32 (config 5: one Richardson call plus its fp16-matrix SpMV and Gram-Schmidt).
# Each sample is a ComposedSolver::run of the unmodified reference with the
# nest's lower levels as its levels and max_outer_total = 1 (include/f3r/nesting.hpp:35).
SAMPLES_PER_OUTER = {1: 1, 2: 1, 3: 8, 4: 8, 5: 32}


def sample_spec(args, per_outer):
    levels = [t.strip() for t in spec_for(args).split(">")]
    return " > ".join(levels[{1: 0, 8: 1, 32: 2}[per_outer]:])


def sample_desc(per_outer):
    return {1: "1 outer iteration", 8: "1 L2 Arnoldi step (1/8 of an outer iteration)",
            32: "1 innermost-FGMRES Arnoldi step (1/32 of an outer iteration: one fp16 Richardson call, "
                "one fp16-matrix SpMV and its Gram-Schmidt)"}[per_outer]


class ReferenceSampler:
    """the UNMODIFIED reference (oracle/_ref/libf3r_ref.so) on this host's cores,
    fed from the binary CSR cache (csr_cache: this process never maps libf3rg.so)"""

    def __init__(self, args, p, threads):
        from oracle_bind import Reference
        self.r = Reference()
        self.r.set_threads(threads)
        self.m = self.r.matrix(p.row_ptr, p.col_idx, p.values)
        self.M = _ref_m(self.r, self.m, args)
        self.b = np.ascontiguousarray(p.b)
        self.per_outer = SAMPLES_PER_OUTER.get(args.config, 1)
        self.spec = sample_spec(args, self.per_outer)

    def step(self):
        rep = self.r.solve(self.m, self.spec, self.b, tol=TOL, max_outer_total=1, want_x=False, precond=self.M)
        return rep.wall_seconds

    def full(self, args):
        return self.r.solve(self.m, spec_for(args), self.b, tol=TOL, want_x=False, precond=self.M)


def _ref_m(r, m, args):
    """the reference's own BlockJacobiIlu0::factorize for --precond (untimed setup, as
    the reference bench times factorisation apart, src/bench.cpp:202-207)"""
    if args is None or args.precond == "identity":
        return None
    return r.ilu(m, 4, 1.0, args.precond == "ic0", 0)


def _mode_key(args):
    return "fp16-f3r" if args.precond == "identity" else f"fp16-f3r-{args.precond}"


def cpu_context(args):
    """the reference's recorded full runs of the three F3R modes (src/nesting.cpp:359-386)
    for this config: SURVEY 8(d)'s context beside the fp16-F3R baseline"""
    runs = reference_runs()
    out = {}
    for mode in ("fp16-f3r", "fp32-f3r", "fp64-f3r"):
        r = runs.get(f"config{args.config}/{mode}")
        if r:
            out[mode] = {"seconds": r["wall_seconds"], "outer": r["outer_iterations"], "threads": r["threads"],
                         "where": "full run in the build container (tests/golden/reference_runs.json)"}
    return out


def reference_outer(args, smp):
    """the reference's own outer count for this config (recorded full run); None if
    there is none and the sample is sub-outer (a full run would take too long)"""
    runs = reference_runs().get(f"config{args.config}/{_mode_key(args)}", {})
    outer_full = int(runs.get("outer_iterations", 0)) or None
    if outer_full is None and smp.per_outer == 1:
        outer_full = smp.full(args).outer_iterations  # small config: measure the count once
    return outer_full


def run_reference_arm(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    from oracle_bind import reference_available

    from paper_2505_20719_b200 import csr_cache  # reads the cache; never loads libf3rg.so
    if not reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libf3r_ref.so not built"}))
        return
    p = csr_cache.load(args.config)
    threads = os.cpu_count()
    smp = ReferenceSampler(args, p, threads)
    outer_full = reference_outer(args, smp)
    if outer_full is None:
        print(json.dumps({"impl": "reference", "unavailable": f"no recorded full reference run for config "
                          f"{args.config} ({_mode_key(args)}) to scale the sample by"}))
        return
    warm = min(args.warmup, 1)
    for _ in range(warm):
        smp.step()
    times = [smp.step() for _ in range(args.steps)]
    per_step = float(np.mean(times))
    value = per_step * smp.per_outer * outer_full
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": warm, "ms_per_step": per_step * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "mixed f64/f32/f16 (software binary16)",
        "data": "synthetic", "config": _config(args, p),
        "cpu_baseline": {"value": value, "unit": "s", "cores": threads, "kind": "reference",
                         "sample": sample_text(args, smp, outer_full)},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "inputs": f"binary CSR cache {os.path.basename(p.path)} (lib/f3rg_gen)",
    }
    print(json.dumps(line))


def sample_text(args, smp, outer_full):
    return (f"{sample_desc(smp.per_outer)} of the unmodified reference fp16-F3R solve per step "
            f"(ComposedSolver::run of '{smp.spec}', max_outer_total 1), config {args.config}; "
            f"value = mean x {smp.per_outer} x {outer_full} outer iterations (the reference's own count)")


def l2_note(p):
    a16 = p.nnz * 6 + 4 * (p.n + 1)  # fp16 values + u32 indices + row pointers
    if a16 > 126e6:
        return (f"none: every pass streams a matrix replica of >= {a16 / 1e6:.0f} MB (fp16 + u32 indices), "
                f"larger than the 126 MB L2")
    return f"none: the {a16 / 1e6:.0f} MB fp16 replica is L2-resident (config 1 caveat, SURVEY 8(d))"


def _config(args, p):
    mname = "identity" if args.precond == "identity" else f"block-Jacobi {args.precond}, 4 blocks, fp16 factors"
    return {"workload": f"BASELINE config {args.config}: fp16-F3R solve to 1e-10 (M = {mname})", "n": p.n,
            "nnz": p.nnz, "solver": spec_for(args), "problem": p.name, "tol": TOL,
            "l2_flush": l2_note(p),
            "parallelism": f"dp{args.gpus}" if args.gpus > 1 else "single GPU"}


def run_partitioned(args):
    """N > 1 (or --partition): ONE config-2 system row-block partitioned over the
    ranks: NCCL point-to-point halos + allgather of rank-local totals
    inside the solve; strong scaling (total work fixed). Timed as the max over ranks
    of CUDA-event time per solve."""
    import torch
    import torch.distributed as dist

    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import csr_cache, partition

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("cpu:gloo,cuda:nccl", rank=rank, world_size=world)
    p = csr_cache.load(args.config)
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
    halos, reds = part.solver.collectives()
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
        "partition": {"rows_rank0": pl.r1 - pl.r0, "halo_rank0": pl.n_lo + pl.n_hi,
                      "collectives_per_outer": {"halo_exchanges": halos / max(1, rep.outer_iterations),
                                                "reductions": reds / max(1, rep.outer_iterations)}},
    }
    if rank == 0:
        print(json.dumps(line))
    del part
    dist.destroy_process_group()


def run_ours(args):
    import torch

    import paper_2505_20719_b200 as f
    from paper_2505_20719_b200 import csr_cache

    rank, local, world = dist_env()
    if world > 1 or args.partition:
        if args.precond != "identity":
            raise SystemExit("--precond: the row-block partition runs M = identity only (DESIGN.md section 6c)")
        return run_partitioned(args)
    torch.cuda.set_device(local)
    p = csr_cache.load(args.config)  # the same bytes the reference arm reads
    reps = f.make_replicas(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values))
    if args.precond == "identity":
        M = f.IdentityPrecond(p.n)
    else:  # factorised once, untimed (the reference bench times it apart)
        M = f.BlockJacobiIlu0.factorize(f.SparseCsr(p.n, p.row_ptr, p.col_idx, p.values),
                                        f.IluConfig(4, 1.0, args.precond == "ic0", f.Precision.P16))
    solver = f.build(f.parse_solver_spec(spec_for(args)), reps, M)
    opts = f.RunOptions(tol=TOL)
    b_dev = torch.from_numpy(np.array(p.b)).cuda()
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
    b_host = torch.from_numpy(np.array(p.b)).pin_memory().numpy()
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
    top_pa = PNAME.get(top[0].split("[")[1].split(",")[0], 2) if "[" in top[0] else 2
    algo_bytes = per_launch_bytes + (column_stream_saving(reps, p, top_pa) if streams_matrix(top[0]) else 0.0)
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
                     "traffic": traffic_table().get(f"config{args.config}", {}).get(top[0]),
                     "algorithmic_bytes_per_launch": algo_bytes,
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
        try:  # the unmodified reference on this host's cores, a bounded sample (SAMPLES_PER_OUTER)
            threads = os.cpu_count()
            smp = ReferenceSampler(args, p, threads)
            outer_ref = reference_outer(args, smp)
            smp.step()  # warm-up (page faults, thread pool)
            per_step = float(np.mean([smp.step() for _ in range(2)]))
            line["cpu_baseline"] = {"value": per_step * smp.per_outer * (outer_ref or outer), "unit": "s",
                                    "cores": threads, "kind": "reference",
                                    "sample": sample_text(args, smp, outer_ref or outer) + f"; {per_step:.2f} s/step",
                                    "context_modes": cpu_context(args)}
        except Exception as e:  # keep the GPU line even if the CPU leg fails
            line["cpu_baseline"] = {"value": None, "unit": "s", "cores": os.cpu_count(), "kind": "reference",
                                    "sample": f"failed: {e}"}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5,
                    help="BASELINE config (default 5: the largest single-GPU configuration)")
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
