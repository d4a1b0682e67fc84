# BASELINE.json configs 2-5 on one GPU (bench.py with explicit shapes; the JSON lines go to gpurun_out/config_sweep.jsonl)
out=gpurun_out/config_sweep.jsonl; : > $out
run() { echo "== $*" >&2; python bench.py --no-cpu-baseline --steps 12 --warmup 3 --stage-reps 2 "$@" >> $out 2>> gpurun_out/config_sweep.err; }
run --problem dtlz2 --obj 3 --dim 500 --pop 10000                 # C2
run --problem lsmop1 --obj 3 --dim 5000 --pop 131072              # C3
run --problem dtlz3 --obj 10 --dim 1000 --pop 65536               # C4
for p in 16384 32768 65536 131072 262144 524288 1048576; do run --problem dtlz2 --obj 3 --dim 5000 --pop $p; done   # C5, one GPU
python - <<'PY'
import json
for l in open("gpurun_out/config_sweep.jsonl"):
    d = json.loads(l); c = d["config"]; s = d["stages_ms"]
    print(f'{c["problem"]:7s} m={c["obj"]:2d} d={c["dim"]:5d} pop={c["pop"]:8d} R={c["ref_vectors"]:8d}  gens/s={d["value"]:9.2f}  e2e={d["e2e"]["value"]:9.2f}  ms: gen={s["generation"]:.3f} repro={s["reproduce"]:.3f} eval={s["evaluate"]:.3f} select={s["select"]:.3f} adapt={s["adapt"]:.3f}  K1 frac={d["roofline"]["frac"]:.3f}')
PY
