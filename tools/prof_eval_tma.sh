M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio,smsp__average_warps_issue_stalled_membar_per_issue_active.ratio,smsp__average_warps_issue_stalled_selected_per_issue_active.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio
ncu --metrics $M --clock-control none -k regex:"eval_lsmop1_tma|eval_tma_kernel" -c 3 --csv --log-file gpurun_out/lsmop_tma.csv python tools/k1_check.py --no-hash --gens 1 --reps 1 --problem $1 --pop 131072 --dim 5000 --obj 3 > gpurun_out/lsmop_tma.log 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/lsmop_tma.csv")) if len(r)>10 and r[0].isdigit()]
by={}
for r in rows: by.setdefault(r[0]+" "+r[4][:60],{})[r[-3].replace("smsp__average_warps_issue_stalled_","st_").replace("_per_issue_active.ratio","")]=r[-1]
for k,v in list(by.items())[:1]:
    print(k); [print("   ",a,b) for a,b in v.items()]
PY
