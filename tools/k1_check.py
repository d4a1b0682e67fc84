#!/usr/bin/env python
"""Developer tool: checksum of a short run + isolated K1 timings (A/B of the two K1 paths:
TEMO_B200_GENERIC_K1=1 forces the generic kernel)."""
import argparse, hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2404_01159_b200 as tb

ap = argparse.ArgumentParser()
ap.add_argument("--problem", default="dtlz2"); ap.add_argument("--pop", type=int, default=1 << 17)
ap.add_argument("--dim", type=int, default=5000); ap.add_argument("--obj", type=int, default=3)
ap.add_argument("--gens", type=int, default=3); ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--no-fuse", action="store_true"); ap.add_argument("--rng", default="splitmix64")
ap.add_argument("--no-hash", action="store_true")
a = ap.parse_args()
tb.init(0)
kw = {}
if a.rng != "splitmix64":
    kw["rng_mode"] = tb.RNG_PHILOX
cfg = tb.RunConfig(problem=a.problem, pop=a.pop, dim=a.dim, obj=a.obj, generations=100, seed=42, fuse_eval=not a.no_fuse, **kw)
with tb.RveaRun(cfg) as run:
    pops = [run.step() for _ in range(a.gens)]
    out = {"pops": pops, "generic": os.environ.get("TEMO_B200_GENERIC_K1", "0")}
    if not a.no_hash:
        st = run.download()
        out["x"] = hashlib.sha256(np.ascontiguousarray(st["x"]).tobytes()).hexdigest()[:16]
        out["f"] = hashlib.sha256(np.ascontiguousarray(st["f"]).tobytes()).hexdigest()[:16]
    out["k1_ms"] = run.time_stage(1, a.reps)
    out["eval_ms"] = run.time_stage(2, a.reps)
    if not a.no_fuse:
        try:
            out["k1_fused_ms"] = run.time_stage(3, a.reps)
        except ValueError:
            pass
    print(json.dumps(out))
