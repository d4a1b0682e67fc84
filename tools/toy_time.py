import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_2404_01159_b200 as tb
from oracle.pyoracle import Ref
tb.init(0)
ref = Ref()
rng = np.random.default_rng(1)
for n in (10000, 131072):
    p = rng.uniform(-1, 1, (n, 114))
    tb.env_rollout(p[:64], 100, 3)
    t = time.perf_counter(); tb.env_rollout(p, 100, 3); dt = time.perf_counter() - t
    t = time.perf_counter(); ref.env_rollout(p[:10000], 100, 3); dc = time.perf_counter() - t
    print("n", n, "gpu ms incl copies", round(dt * 1e3, 2), " cpu (10000 rows) ms", round(dc * 1e3, 2))
cfg = tb.RunConfig(problem="toy3", pop=10000, generations=30, seed=1)
with tb.RveaRun(cfg) as run:
    for _ in range(5): run.step()
    t = time.perf_counter()
    for _ in range(20): run.step()
    print("toy3 pop 10000 generation ms", (time.perf_counter() - t) / 20 * 1e3, run.timings())
