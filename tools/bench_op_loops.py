#!/usr/bin/env python
"""Developer tool: generations/s of the device-resident loop with every reproduction operator (RunConfig::op) at one shape."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2404_01159_b200 as tb

ap = argparse.ArgumentParser()
ap.add_argument("--pop", type=int, default=1 << 17); ap.add_argument("--dim", type=int, default=5000)
ap.add_argument("--steps", type=int, default=12); ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
tb.init(0)
out = {}
for op in ("ga", "de", "pso", "cso", "random"):
    cfg = tb.RunConfig(problem="dtlz2", op=op, pop=a.pop, dim=a.dim, obj=3, generations=100, seed=42)
    with tb.RveaRun(cfg) as run:
        for _ in range(a.warmup):
            run.step()
        t0 = time.perf_counter()
        ms = []
        for _ in range(a.steps):
            run.step()
            ms.append(run.timings())
        dt = time.perf_counter() - t0
    out[op] = {"generations/s": a.steps / dt, "reproduce_ms": float(np.mean([m["reproduce"] for m in ms])),
               "evaluate_ms": float(np.mean([m["evaluate"] for m in ms])), "select_ms": float(np.mean([m["select"] for m in ms]))}
print(json.dumps(out))
