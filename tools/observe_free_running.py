"""Developer tool: prints what the free-running tests observe (used to pin their assertions)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_01159_b200 as tb
from oracle.pyoracle import Ref
tb.init(0)
chk = Ref()
rec = tb.rvea_run(tb.make_problem("dtlz1", 12, 3), tb.RunConfig(pop=105, lattice_h=13, generations=100, seed=42))
exp = chk.rvea_run("dtlz1", 105, 12, 3, 100, seed=42, lattice_h=13)
pops = np.array([r.pop_size for r in rec.rows])
same = pops == exp["pop_size"]
agree = int(np.argmax(~same)) if not same.all() else len(pops)
print("C1 agree", agree, "mean|dpop|", np.abs(pops.astype(float) - exp["pop_size"]).mean(),
      "x equal", rec.final_x.shape == exp["x"].shape and np.array_equal(rec.final_x, exp["x"]),
      "f maxrel", (np.abs(rec.final_f - exp["f"]) / np.abs(exp["f"])).max() if rec.final_f.shape == exp["f"].shape else None)
ex, ef = exp["x"], exp["f"]
print("shapes", rec.final_x.shape, ex.shape, "rows equal", int((rec.final_x == ex[:rec.final_x.shape[0]]).all(axis=1).sum()),
      "max|dx|", np.abs(rec.final_x - ex[:rec.final_x.shape[0]]).max(), "max|df|", np.abs(rec.final_f - ef[:rec.final_f.shape[0]]).max())
a = {r.tobytes() for r in rec.final_x}; b = {r.tobytes() for r in ex[:rec.final_x.shape[0]]}
print("rows in common as sets", len(a & b), "of", len(a))
g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "nsga2.npz"))
rec = tb.nsga2_run(tb.make_problem("dtlz2", 9, 3), tb.RunConfig(pop=40, generations=12, seed=3))
print("nsga2 x equal", np.array_equal(rec.final_x, g["r0_x"]), "mean sum rel", abs(rec.final_f.sum(axis=1).mean() - g["r0_f"].sum(axis=1).mean()) / g["r0_f"].sum(axis=1).mean())
g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "metrics.npz"))
rec = tb.rvea_run(tb.make_problem("dtlz2", 10, 3), tb.RunConfig(pop=60, generations=15, seed=6),
                  tb.MetricContext(pf_ref=g["a_pf"], hv_ref=np.full(3, 1.1)))
pops = np.array([r.pop_size for r in rec.rows])
same = pops == g["run_pop"]
print("metrics agree", int(np.argmax(~same)) if not same.all() else len(pops), "of", len(pops),
      "igd maxabs", max(abs(rec.rows[t].igd_value - g["run_igd"][t]) for t in range(len(pops))),
      "hv maxabs", max(abs(rec.rows[t].hv_value - g["run_hv"][t]) for t in range(len(pops))))
g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "pipeline_ops.npz"))
for op in ("de", "pso", "cso", "random"):
    rec = tb.rvea_run(tb.make_problem("dtlz2", 9, 3), tb.RunConfig(op=op, pop=40, generations=12, seed=3))
    pops = np.array([r.pop_size for r in rec.rows]); e = g[f"{op}_a_pop"]; same = pops == e
    print(op, "agree", int(np.argmax(~same)) if not same.all() else len(pops), "x equal", rec.final_x.shape == g[f"{op}_a_x"].shape and np.array_equal(rec.final_x, g[f"{op}_a_x"]))
