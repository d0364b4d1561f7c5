"""Quick look at an `ncu --page source --csv` (SASS) dump + its raw page: headline
metrics, stall mix, opcode histogram of the hot instructions, top sampled lines.
    python tools/ncu_hot.py gpurun_out/wsmb_ncu_kb_spmv [hot_threshold]
"""
import collections
import csv
import sys

base = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
rows = list(csv.reader(open(base + "_raw.csv")))
h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
H, U, V = rows[h], rows[h + 1], rows[h + 2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "smsp__warps_eligible.avg.per_cycle_active"]
print(V[H.index("Kernel Name")][:70])
for w in want:
    if w in H:
        print(f"  {w:70s} {V[H.index(w)]} {U[H.index(w)]}")
rows = list(csv.reader(open(base + "_source.csv")))
H = rows[1]
ie, ss = H.index("Instructions Executed"), H.index("# Samples")
body = [r for r in rows[2:] if len(r) > ie and r[ie].isdigit()]
tot = sum(int(r[ie]) for r in body)
ts = sum(int(r[ss]) for r in body)
mx = max(int(r[ie]) for r in body)
stall_cols = [i for i, x in enumerate(H) if x.startswith("stall_") and "Not Issued" not in x]
agg = {H[i]: sum(int(r[i]) for r in body if r[i].isdigit()) for i in stall_cols}
t = sum(agg.values()) or 1
print("  stalls:", {a[6:]: round(v / t * 100, 1) for a, v in sorted(agg.items(), key=lambda kv: -kv[1])[:9]})
hot = [r for r in body if int(r[ie]) > thr * mx]
print(f"  total warp-inst {tot/1e6:.1f}M; hot (> {thr} of max count {mx/1e6:.2f}M): {len(hot)} instrs, "
      f"{sum(int(r[ie]) for r in hot)/1e6:.1f}M inst, {sum(int(r[ss]) for r in hot)/ts*100:.1f}% of samples")
ops = collections.Counter()
for r in hot:
    op = [o for o in r[1].split() if not o.startswith("@")][0]
    ops[op.split(".")[0]] += int(r[ie])
print("  hot opcodes:", ", ".join(f"{o} {c/1e6:.1f}M" for o, c in ops.most_common(18)))
print("  top sampled:")
for r in sorted(body, key=lambda r: -int(r[ss]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 14]:
    print(f"    s={int(r[ss]):6d} ({int(r[ss])/ts*100:4.1f}%) n={int(r[ie])/1e6:6.2f}M {r[1].strip()[:90]}")
