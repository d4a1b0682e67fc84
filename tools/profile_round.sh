# Round profile artefacts (run under gpurun): launch list of the bench command + one full capture of the dominant kernel.
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 12 --warmup 3 --no-cpu-baseline --stage-reps 1 > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:reproduce_pairs -s 6 -c 1 -f -o gpurun_out/prof_k1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --stage-reps 1 > gpurun_out/ncu_k1.log 2>&1
ncu --set full --clock-control none -k regex:assoc_indexed -s 6 -c 1 -f -o gpurun_out/prof_assoc python bench.py --steps 3 --warmup 3 --no-cpu-baseline --stage-reps 1 > gpurun_out/ncu_assoc.log 2>&1
ls -la gpurun_out
