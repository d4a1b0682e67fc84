"""TEST INFRASTRUCTURE — regenerate tests/golden/*.npz from the UNMODIFIED reference.

Run in the build container (needs /root/reference mounted so that oracle/Makefile can
compile oracle/_ref/libtemo_ref.so):

    python -m oracle.gen_golden

Every array stored here is an input to, or an output of, the reference's own functions
(called through oracle/ref_wrap.cpp). The instance generators mirror the reference's
verification suites (verify.hpp:41-47,53-76,83-103: master seed + instance number, all
randomness from RngStream) so a fixture can be re-derived from (seed, instance) alone.
The fixtures are what pins the C restatement (and the CUDA path) on machines where the
reference is not mounted.
"""
from __future__ import annotations

import os

import numpy as np

from .pyoracle import Ref

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


class Stream:
    """RngStream (rng.hpp:34-52) driven through the reference's value_at."""

    def __init__(self, ref, seed, counter=0):
        self.ref, self.seed, self.counter = ref, seed, counter

    def next(self):
        v = self.ref.value_at(self.seed, self.counter)
        self.counter += 1
        return v

    def pick(self, lo, hi):  # verify.hpp:33-35
        return lo + int(self.next() * float(hi - lo + 1))

    def tensor(self, rows, cols):
        out = self.ref.uniform(self.seed, self.counter, rows * cols).reshape(rows, cols)
        self.counter += rows * cols
        return out


def operator_instance(ref, g, n_min, n_max, d_max):
    """verify.hpp:83-103 random_operator_instance."""
    n = g.pick(n_min, n_max)
    d = g.pick(1, d_max)
    lower, upper = np.empty(d), np.empty(d)
    for j in range(d):
        lower[j] = -1.0 - g.next()
        upper[j] = lower[j] + 0.5 + 2.0 * g.next()
    x = g.tensor(n, d)
    x = lower + x * (upper - lower)
    return n, d, lower, upper, x


def toyenv_fixture(ref):
    """MLP policy + toy control environment (problems.hpp:105-241) and short RVEA runs on toy2 / toy3 (a second-round
    fixture, written by `python -m oracle.gen_golden toyenv` without touching the others)."""
    te = {}
    g = Stream(ref, 9400)
    p = g.tensor(40, 114) * 2.0 - 1.0
    p[7, 3] = np.nan        # problems.hpp:224-230: non-finite parameters score -1e9
    p[9, 113] = np.inf
    te["params"] = p
    for T, m in ((100, 2), (100, 3), (1, 2), (37, 3)):
        te[f"ret_T{T}_m{m}"] = ref.env_rollout(p, T, m)
    p64 = g.tensor(6, 4 * 64 + 64 + 2 * 64 + 2) * 6.0 - 3.0   # the widest network env_rollout accepts, saturating tanh
    te["params_h64"] = p64
    te["ret_h64"] = ref.env_rollout(p64, 50, 3, hidden=64)
    obs = g.tensor(40, 4) * 4.0 - 2.0
    ok = np.isfinite(p).all(axis=1)
    te["obs"] = obs
    te["act"] = ref.mlp_forward(np.where(np.isfinite(p), p, 0.0), obs)
    te["f_toy2"] = ref.evaluate("toy2", p[ok], 2)              # make_problem's evaluate: the negated returns
    te["f_toy3_T20"] = ref.evaluate("toy3", p[ok], 3, horizon=20)
    for tag, (problem, m, n, gens, seed) in (("run2", ("toy2", 2, 40, 12, 5)), ("run3", ("toy3", 3, 66, 10, 8))):
        rr = ref.rvea_run(problem, n, 114, m, gens, seed=seed)
        te[f"{tag}_pop"] = rr["pop_size"]
        te[f"{tag}_x"] = rr["x"]
        te[f"{tag}_f"] = rr["f"]
    np.savez(os.path.join(OUT, "toyenv.npz"), **te)


def main():
    import sys
    ref = Ref()
    os.makedirs(OUT, exist_ok=True)
    if sys.argv[1:] == ["toyenv"]:
        toyenv_fixture(ref)
        return

    # ---- rng -----------------------------------------------------------------------
    seeds = np.array([0, 7, 42, 99, 2**63 + 12345], dtype=np.uint64)
    draws = np.array([[ref.value_at(int(s), k) for k in range(24)] for s in seeds])
    far = np.array([ref.value_at(42, k) for k in (10**6, 2**32 + 5, 2**40 + 17, 2**63)])
    perm20, c20 = ref.shuffle_indices(42, 0, 20)
    perm257, c257 = ref.shuffle_indices(5, 1000, 257)
    pool, cpool = ref.parent_pool_indices(77, 105, 42, 5000)
    np.savez(os.path.join(OUT, "rng.npz"), seeds=seeds, draws=draws, far=far,
             far_k=np.array([10**6, 2**32 + 5, 2**40 + 17, 2**63], dtype=np.uint64),
             perm20=perm20, c20=c20, perm257=perm257, c257=c257, pool=pool, cpool=cpool)

    # ---- operators (verify.hpp:117-182 instance recipe; test_operators.cpp:63-114 seeds)
    ops = {}
    for tag, seed, nmin, nmax, dmax in (("a", 37, 8, 8, 5), ("b", 7002, 2, 16, 8), ("c", 7003, 2, 16, 8),
                                        ("odd", 8101, 9, 9, 7), ("wide", 8102, 12, 12, 40)):
        g = Stream(ref, seed)
        n, d, lower, upper, x = operator_instance(ref, g, nmin, nmax, dmax)
        sseed = seed ^ 0x5EED
        sbx, c1 = ref.sbx(x, sseed, 0, lower, upper)
        pm, c2 = ref.polynomial_mutation(x, sseed, 0, lower, upper)
        ga, c3 = ref.ga_reproduce(x, sseed, 0, lower, upper)
        # a high mutation rate instance so the pow branch of PM is exercised on many genes
        pm_hot, _ = ref.polynomial_mutation(x, sseed, 11, lower, upper, ga=(1.0, 20.0, float(d) * 0.6, 20.0))
        ga_pc, _ = ref.ga_reproduce(x, sseed, 3, lower, upper, ga=(0.5, 15.0, 2.0, 10.0))
        for k, v in dict(x=x, lower=lower, upper=upper, sbx=sbx, pm=pm, ga=ga, pm_hot=pm_hot, ga_pc=ga_pc,
                         counters=np.array([c1, c2, c3], dtype=np.uint64),
                         seed=np.array([sseed], dtype=np.uint64)).items():
            ops[f"{tag}_{k}"] = v
    rr, crr = ref.random_reproduce(5, 7, 42, 3, np.linspace(-1, 0, 7), np.linspace(1, 3, 7))
    ops["rr"] = rr
    ops["rr_counter"] = np.array([crr], dtype=np.uint64)
    np.savez(os.path.join(OUT, "operators.npz"), **ops)

    # ---- DE / PSO / CSO (verify.hpp:117-182, ops 2..4: instance k of master seed 7002; two chained steps each)
    sw = {}
    for tag, op, k in (("de0", 2, 0), ("de1", 2, 17), ("pso0", 3, 0), ("pso1", 3, 41), ("cso0", 4, 0), ("cso1", 4, 63)):
        seed = 7002 + op * 1000003 + k
        g = Stream(ref, seed)
        n, d, lower, upper, x = operator_instance(ref, g, 4 if op == 2 else 2, 16, 8)
        scores = g.tensor(n, 1).reshape(-1)
        sseed = seed ^ 0xabcdef
        rec = dict(x=x, lower=lower, upper=upper, scores=scores, seed=np.array([sseed], dtype=np.uint64))
        if op == 2:
            y1, c1 = ref.de_reproduce(x, sseed, 0, lower, upper)
            y2, c2 = ref.de_reproduce(y1, sseed, c1, lower, upper, p=(0.8, 0.4))
            rec.update(y1=y1, y2=y2, counters=np.array([c1, c2], dtype=np.uint64))
        elif op == 3:
            vel, pbx, pbs = np.zeros_like(x), x * 0.5, scores + 0.25
            y1, c1, v1, px1, ps1 = ref.pso_reproduce(x, scores, sseed, 0, lower, upper, vel, pbx, pbs)
            y2, c2, v2, px2, ps2 = ref.pso_reproduce(y1, scores[::-1].copy(), sseed, c1, lower, upper, v1, px1, ps1)
            rec.update(y1=y1, y2=y2, v1=v1, v2=v2, px2=px2, ps2=ps2, counters=np.array([c1, c2], dtype=np.uint64))
        else:
            y1, c1, v1 = ref.cso_reproduce(x, scores, sseed, 0, lower, upper, np.zeros_like(x))
            y2, c2, v2 = ref.cso_reproduce(y1, scores[::-1].copy(), sseed, c1, lower, upper, v1)
            rec.update(y1=y1, y2=y2, v1=v1, v2=v2, counters=np.array([c1, c2], dtype=np.uint64))
        for key, val in rec.items():
            sw[f"{tag}_{key}"] = val
    np.savez(os.path.join(OUT, "swarm.npz"), **sw)

    # ---- problems ------------------------------------------------------------------
    pr = {}
    g = Stream(ref, 9100)
    for m, d in ((3, 12), (2, 7), (5, 30), (10, 25)):
        x = g.tensor(9, d)
        x[0, :] = 0.5          # test_problems.cpp:8-33 slices
        x[1, :] = 0.0
        x[2, :] = 1.0
        pr[f"x_m{m}"] = x
        for pid in (1, 2, 3, 4):
            pr[f"f{pid}_m{m}"] = ref.evaluate(f"dtlz{pid}", x, m)
    np.savez(os.path.join(OUT, "problems.npz"), **pr)

    # ---- refvec --------------------------------------------------------------------
    rv = {}
    for m, H in ((3, 4), (2, 9), (3, 13), (5, 4), (10, 2)):
        v0, gamma = ref.make_ref_set(m, H)
        g = Stream(ref, 9200 + m * 100 + H)
        zmin = g.tensor(1, m)[0]
        zmax = zmin + 0.1 + 5.0 * g.tensor(1, m)[0]
        v1, g1 = ref.adapt(v0, v0, gamma, zmin, zmax)
        zbad = zmax.copy()
        zbad[m - 1] = zmin[m - 1]
        v2, g2 = ref.adapt(v0, v1, g1, zmin, zbad)  # degenerate range: untouched
        rv.update({f"v0_{m}_{H}": v0, f"gamma_{m}_{H}": gamma, f"zmin_{m}_{H}": zmin, f"zmax_{m}_{H}": zmax,
                   f"v1_{m}_{H}": v1, f"g1_{m}_{H}": g1, f"v2_{m}_{H}": v2, f"g2_{m}_{H}": g2})
    rv["density"] = np.array([[m, n, ref.lattice_density_for(m, n)] for m, n in
                              ((3, 105), (3, 10000), (3, 16384), (3, 131072), (3, 1048576), (10, 65536), (2, 50), (5, 1000))],
                             dtype=np.uint64)
    np.savez(os.path.join(OUT, "refvec.npz"), **rv)

    # ---- selection (verify.hpp:53-76 recipe, master seed 7001) ------------------------
    se = {}
    count = 0
    for k in range(40):
        g = Stream(ref, 7001 + k)
        n = g.pick(1, 64)
        m = g.pick(2, 3)
        H = g.pick(1, 14) if m == 2 else g.pick(1, 4)
        t_max = g.pick(1, 200)
        t = g.pick(0, t_max)
        v0, gamma = ref.make_ref_set(m, H)
        f = g.tensor(n, m) * 10.0
        s = ref.rv_select(f, v0, gamma, t, t_max, 2.0)
        s2 = ref.rv_select(f, v0, gamma, t, t_max, 2.0, set_form=True)
        assert np.array_equal(s.elite, s2.elite) and np.array_equal(s.validity, s2.validity)
        se.update({f"f_{k}": f, f"mh_{k}": np.array([m, H, t, t_max], dtype=np.uint64), f"elite_{k}": s.elite,
                   f"valid_{k}": s.validity, f"assoc_{k}": s.assoc, f"theta_{k}": s.theta, f"apd_{k}": s.apd})
        count += 1
    se["count"] = np.array([count])
    # crafted: duplicates (exact APD ties -> lowest row), a row at the ideal point, adapted vectors
    v0, gamma = ref.make_ref_set(3, 5)
    g = Stream(ref, 9300)
    f = g.tensor(30, 3)
    f[7] = f[3]
    f[21] = f[3]
    f[12] = f.min(axis=0)  # exactly at the ideal point -> nf == 0 -> vector 0, apd 0
    v1, g1 = ref.adapt(v0, v0, gamma, np.array([0.0, 0.1, 0.2]), np.array([3.0, 1.0, 0.7]))
    s = ref.rv_select(f, v1, g1, 37, 100, 2.0)
    se.update(dict(crafted_f=f, crafted_v=v1, crafted_gamma=g1, crafted_elite=s.elite, crafted_valid=s.validity,
                   crafted_assoc=s.assoc, crafted_apd=s.apd))
    np.savez(os.path.join(OUT, "selection.npz"), **se)

    # ---- whole pipeline (SURVEY.md §8c goldens; test_algorithms.cpp:198-210 seed 77) ----
    c1 = ref.rvea_run("dtlz1", 105, 12, 3, 100, seed=42, lattice_h=13)
    s77 = ref.rvea_run("dtlz2", 12, 8, 3, 10, seed=77, lattice_h=3)
    s77o = ref.rvea_run("dtlz2", 12, 8, 3, 10, seed=77, lattice_h=3, scalar=True)
    assert np.array_equal(s77["f"], s77o["f"]) and np.array_equal(s77["x"], s77o["x"])
    d3 = ref.rvea_run("dtlz3", 64, 20, 4, 30, seed=5)
    d4 = ref.rvea_run("dtlz4", 50, 10, 2, 25, seed=11)
    np.savez(os.path.join(OUT, "pipeline.npz"),
             c1_x=c1["x"], c1_f=c1["f"], c1_pop=c1["pop_size"],
             s77_x=s77["x"], s77_f=s77["f"], s77_pop=s77["pop_size"],
             d3_x=d3["x"], d3_f=d3["f"], d3_pop=d3["pop_size"],
             d4_x=d4["x"], d4_f=d4["f"], d4_pop=d4["pop_size"])
    # ---- the run loop with the other operators (algorithms.hpp:253-268) ----
    po = {}
    for op in ("de", "pso", "cso", "random"):
        for tag, (problem, n, d, m, H, gens, seed) in (("a", ("dtlz2", 40, 9, 3, 0, 12, 3)), ("b", ("dtlz1", 33, 15, 2, 0, 20, 8)),
                                                        ("c", ("dtlz3", 64, 20, 4, 0, 15, 5))):
            rr = ref.rvea_run_op(op, problem, n, d, m, gens, seed=seed, lattice_h=H)
            po.update({f"{op}_{tag}_x": rr["x"], f"{op}_{tag}_f": rr["f"], f"{op}_{tag}_pop": rr["pop_size"]})
    np.savez(os.path.join(OUT, "pipeline_ops.npz"), **po)
    # ---- quality indicators (metrics.hpp:21-44, 76-124) ----
    me = {}
    for tag, (n, m, n_ref, samples, seed) in (("a", (40, 3, 91, 2048, 9001)), ("b", (300, 5, 126, 1000, 17)), ("c", (7, 2, 11, 500, 3)),
                                               ("d", (1, 4, 35, 257, 5))):
        g = Stream(ref, 8800 + n)
        f = g.tensor(n, m) * 1.5
        pf = ref.dtlz_pf_reference(2, m, {3: 12, 5: 5, 2: 10, 4: 4}[m])[:n_ref]
        rp = np.full(m, 1.2)
        lo = np.full(m, 0.05)
        me.update({f"{tag}_f": f, f"{tag}_pf": pf, f"{tag}_ref": rp, f"{tag}_lo": lo, f"{tag}_samples": np.array([samples, seed]),
                   f"{tag}_igd": np.array([ref.igd(f, pf)]), f"{tag}_hv_box": np.array(ref.hv_mc_box(f, lo, rp, samples, seed)),
                   f"{tag}_hv": np.array(ref.hv_mc_box(f, None, rp, samples, seed))})
    tr = ref.rvea_run_metrics("dtlz2", 60, 10, 3, 15, pf_ref=ref.dtlz_pf_reference(2, 3, 12), hv_ref=np.full(3, 1.1), seed=6)
    me.update(run_pop=tr["pop_size"], run_igd=tr["igd"], run_hv=tr["hv"])
    # Archive::insert / crowding_distance (algorithms.hpp:72-144, selection.hpp:289-312): coarse objective grids give exact
    # duplicates and many dominance relations; two successive insertions, the second one capped
    for tag, (n0, n1, n2, d, m, q, cap) in (("ar0", (30, 40, 35, 4, 3, 5.0, 12)), ("ar1", (0, 25, 60, 3, 2, 8.0, 5)),
                                             ("ar2", (50, 50, 50, 2, 4, 3.0, 20))):
        g = Stream(ref, 5100 + n1)
        xs = [g.tensor(k, d) if k else np.empty((0, d)) for k in (n0, n1, n2)]
        fs = [np.floor(g.tensor(k, m) * q) / q if k else np.empty((0, m)) for k in (n0, n1, n2)]
        a0 = ref.archive_insert(None, None, xs[0], fs[0]) if n0 else (None, None)
        a1 = ref.archive_insert(a0[0], a0[1], xs[1], fs[1])
        a2 = ref.archive_insert(a1[0], a1[1], xs[2], fs[2], cap)
        me.update({f"{tag}_x{k}": xs[k] for k in range(3)})
        me.update({f"{tag}_f{k}": fs[k] for k in range(3)})
        me.update({f"{tag}_cap": np.array([cap]), f"{tag}_a1x": a1[0], f"{tag}_a1f": a1[1], f"{tag}_a2x": a2[0], f"{tag}_a2f": a2[1],
                   f"{tag}_crowd": ref.crowding_distance(a1[1])})
    np.savez(os.path.join(OUT, "metrics.npz"), **me)
    # ---- NSGA-II baseline (selection.hpp:251-346, algorithms.hpp:301-369) ----
    ns = {}
    for tag, (n, m, q) in (("s0", (60, 3, 6.0)), ("s1", (200, 2, 50.0)), ("s2", (120, 5, 3.0)), ("s3", (1, 3, 2.0))):
        g = Stream(ref, 7300 + n)
        f = np.floor(g.tensor(n, m) * q) / q
        ns.update({f"{tag}_f": f, f"{tag}_rank": ref.nondominated_sort(f), f"{tag}_sel_half": ref.nsga2_select(f, n // 2),
                   f"{tag}_sel_third": ref.nsga2_select(f, (n + 2) // 3), f"{tag}_sel_all": ref.nsga2_select(f, n)})
    for tag, (problem, n, d, m, gens, seed) in (("r0", ("dtlz2", 40, 9, 3, 12, 3)), ("r1", ("dtlz1", 33, 15, 2, 15, 8))):
        rr = ref.nsga2_run(problem, n, d, m, gens, seed=seed)
        ns.update({f"{tag}_x": rr["x"], f"{tag}_f": rr["f"]})
    np.savez(os.path.join(OUT, "nsga2.npz"), **ns)
    toyenv_fixture(ref)
    total = sum(os.path.getsize(os.path.join(OUT, f)) for f in os.listdir(OUT))
    print(f"wrote {OUT}: {total/1024:.1f} KiB")


if __name__ == "__main__":
    main()
