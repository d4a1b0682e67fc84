# developer: stall / pipe metrics of the pair kernel at a given shape: tools/k1_stalls_shape.sh TAG <k1_check.py args>
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio,smsp__average_warps_issue_stalled_membar_per_issue_active.ratio,smsp__average_warp_latency_per_inst_issued.ratio,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
tag=$1; shift
ncu --metrics $M --clock-control none -k regex:reproduce_pairs -s ${SKIP:-3} -c ${COUNT:-2} --csv --log-file gpurun_out/stalls_$tag.csv python tools/k1_check.py --no-hash --gens 3 --reps 1 "$@" > gpurun_out/stalls_$tag.log 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/stalls_$tag.csv")) if len(r)>10 and r[0].isdigit()]
by={}
for r in rows: by.setdefault(r[0]+" "+r[4][:40],{})[r[-3].replace("smsp__average_warps_issue_stalled_","st_").replace("_per_issue_active.ratio","")]=r[-1]
for k,v in by.items():
    print(k); [print("   ",a,b) for a,b in v.items()]
PY
