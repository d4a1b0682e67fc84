"""Developer tool: per-step stage times of a short headline run (first-use hiccups, adaptation steps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_01159_b200 as tb
tb.init(0)
cfg = tb.RunConfig(problem="dtlz2", pop=1 << 17, dim=5000, obj=3, generations=100, seed=42)
with tb.RveaRun(cfg) as run:
    for _ in range(3): run.step()
    run.timing_history(reset=True)
    for _ in range(40): run.step()
    h = run.timing_history()
    print([round(x["adapt"], 3) for x in h])
    print([round(x["generation"], 2) for x in h])
    print([round(x["select"], 3) for x in h])
    print("rep", [round(x["reproduce"], 2) for x in h][:12])
    print("ada", [round(x["adapt"], 2) for x in h][:12])
    print("prep", [round(x["prep"], 3) for x in h][:12])
    print("eval", [round(x["evaluate"], 3) for x in h][:12])
    print("ada-all", [round(x["adapt"], 2) for x in h if x["adapt"] > 0.01])
