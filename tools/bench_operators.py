#!/usr/bin/env python
"""Developer benchmark of the DE / PSO / CSO operator kernels: device time (CUDA events inside the C-ABI call) and achieved
HBM bandwidth on algorithmic bytes, host buffers in / out (the PCIe copies are outside the timed region)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2404_01159_b200 as tb

n, d = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (16384, 5000)))
tb.init(0)
rng = np.random.default_rng(0)
lo, hi = np.zeros(d), np.ones(d)
x = rng.random((n, d))
sc = rng.random(n)
out = {"n": n, "d": d}
best = lambda f: min(f() for _ in range(4))
def de():
    t = {}; tb.de_reproduce(x, tb.RngStream(1, 0), tb.DeParams(), lo, hi, timing=t); return t["kernel_ms"]
def pso():
    t = {}; st = tb.SwarmState(np.zeros_like(x), x * 0.5, sc + 0.25); tb.pso_reproduce(x, st, sc, tb.RngStream(1, 0), tb.PsoParams(), lo, hi, timing=t); return t["kernel_ms"]
def cso():
    t = {}; st = tb.make_swarm_state(x, sc); tb.cso_reproduce(x, sc, tb.RngStream(1, 0), tb.CsoParams(), lo, hi, st, timing=t); return t["kernel_ms"]
nd = float(n) * d
for name, fn, bytes_per_gene in (("de", de, 8 * (2 * 0.9 + 2)), ("pso", pso, 40.0), ("cso", cso, 40.0)):
    ms = best(fn)
    out[name] = {"kernel_ms": round(ms, 4), "algorithmic_GB": round(bytes_per_gene * nd / 1e9, 3), "GB/s": round(bytes_per_gene * nd / ms / 1e6, 1)}
print(json.dumps(out))
