# developer: --set full capture of the pair kernel at pop 32768 -> gpurun_out/prof_k1full.ncu-rep
ncu --set full --clock-control none --import-source on -k regex:reproduce_pairs -s 1 -c 1 -f -o gpurun_out/prof_k1full python tools/k1_check.py --pop 32768 --gens 2 --reps 1 --no-hash > gpurun_out/ncu_k1full.log 2>&1; tail -2 gpurun_out/ncu_k1full.log
