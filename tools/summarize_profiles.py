#!/usr/bin/env python
"""Turns the ncu artefacts of tools/profile_round.sh (gpurun_out/) into the tracked summaries under profiles/:
   <tag>_launches.csv (raw launch list), <tag>_launch_summary.md, <tag>_ncu_top_kernels.csv (selected metrics)."""
import collections, csv, re, shutil, subprocess, sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r1b"
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
           "smsp__average_warp_latency_per_inst_issued.ratio", "smsp__thread_inst_executed_per_inst_executed.ratio",
           "sm__warps_active.avg.per_cycle_active", "smsp__warps_active.avg.per_cycle_active",
           "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio", "lts__t_sector_hit_rate.pct"]

shutil.copy("gpurun_out/launches.csv", f"profiles/{tag}_launches.csv")
rows = list(csv.reader(open("gpurun_out/launches.csv")))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
iK, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= iV:
        continue
    name = re.sub(r"\(.*", "", r[iK]).replace("void temo_b200::<unnamed>::", "").replace("void temo_b200::", "")
    try:
        v = float(r[iV].replace(",", ""))
    except ValueError:
        continue
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v for _, v in agg.values())
with open(f"profiles/{tag}_launch_summary.md", "w") as fh:
    fh.write("| kernel | launches | total ms | avg us | share |\n|---|---:|---:|---:|---:|\n")
    for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:16]:
        fh.write(f"| `{k}` | {n} | {v / 1e6:.3f} | {v / n / 1e3:.1f} | {100 * v / tot:.1f}% |\n")

out = []
for rep in ("prof_k1", "prof_assoc"):
    raw = subprocess.run(["ncu", "-i", f"gpurun_out/{rep}.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h, units = rr[0], rr[1]
    for vals in rr[2:]:
        d = dict(zip(h, vals))
        if not out:
            out.append(["Kernel Name"] + METRICS)
            out.append([""] + [dict(zip(h, units)).get(m, "") for m in METRICS])
        out.append([d.get("Kernel Name", "")[:90]] + [d.get(m, "") for m in METRICS])
with open(f"profiles/{tag}_ncu_top_kernels.csv", "w", newline="") as fh:
    csv.writer(fh).writerows(out)
print(open(f"profiles/{tag}_launch_summary.md").read())
print(open(f"profiles/{tag}_ncu_top_kernels.csv").read())
