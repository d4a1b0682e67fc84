#!/usr/bin/env python
"""The reference's `scale` sub-command (temo.cpp:239-282) with the device-resident run in the `tensor` column.

    python tools/scale.py --pops 32,64,...,16384 --dim 100 --out out_dir

Per point (series population: n varies at d = --dim; series dimension: d varies at n = --pop): DTLZ1, GA, track_archive
off, --gens generations (default 20), seed 42; tensor_ms = median per-generation duration of temo_b200's rvea_run,
oracle_ms = the same for the UNMODIFIED reference's rvea_run on this box's host cores (oracle/_ref, all threads; the
scalar loop oracle with --scalar-oracle like the reference's own column), speedup = oracle_ms / tensor_ms. Writes
out_dir/scale.csv in the reference's format (io.hpp:38-59)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_01159_b200 as tb
from paper_2404_01159_b200 import harness

ap = argparse.ArgumentParser()
ap.add_argument("--pops", default="")
ap.add_argument("--dims", default="")
ap.add_argument("--pop", type=int, default=100)
ap.add_argument("--dim", type=int, default=100)
ap.add_argument("--obj", type=int, default=3)
ap.add_argument("--gens", type=int, default=20)
ap.add_argument("--seed", type=int, default=42)
ap.add_argument("--out", default="gpurun_out/scale")
ap.add_argument("--scalar-oracle", action="store_true", help="oracle column = oracle_rvea_run (single thread), as in the reference")
ap.add_argument("--max-cpu-rows-x-dim", type=float, default=2.0e8, help="skip the CPU column above this n*d (time)")
a = ap.parse_args()

from oracle.pyoracle import Ref  # the CPU column is the checker's job (bench-side use of oracle/, like bench.py's baseline)
ref = Ref()
tb.init(0)
os.makedirs(a.out, exist_ok=True)
points = [("population", int(n), a.dim) for n in a.pops.split(",") if n] + [("dimension", a.pop, int(d)) for d in a.dims.split(",") if d]
echo = {"command": "scale", "seed": str(a.seed), "threads": str(ref.num_threads()), "obj": str(a.obj), "generations": str(a.gens),
        "tensor": "temo_b200 (B200)", "oracle": "oracle_rvea_run" if a.scalar_oracle else "reference rvea_run (all host threads)"}
with harness.scale_csv(os.path.join(a.out, "scale.csv"), echo) as csv:
    for series, n, d in points:
        prob = tb.make_problem("dtlz1", d, a.obj)
        cfg = tb.RunConfig(pop=n, generations=a.gens, seed=a.seed)
        tb.rvea_run(prob, tb.RunConfig(pop=n, generations=2, seed=a.seed))  # library warm-up (context, kernels)
        rec = tb.rvea_run(prob, cfg)
        tensor_ms = harness.median_generation_ms([r.elapsed_ms for r in rec.rows])
        oracle_ms, status = 0.0, "ok"
        if float(n) * d <= a.max_cpu_rows_x_dim:
            out = ref.rvea_run("dtlz1", n, d, a.obj, a.gens, seed=a.seed, scalar=a.scalar_oracle, want_x=False)
            oracle_ms = harness.median_generation_ms(out["elapsed_ms"])
        else:
            status = "cpu_skipped"
        csv.row(harness.scale_row(series, n, d, a.obj, a.gens, tensor_ms, oracle_ms, status))
        print(f"scale {series} n={n} d={d}: tensor {tensor_ms:.3f} ms, oracle {oracle_ms:.3f} ms", file=sys.stderr)
