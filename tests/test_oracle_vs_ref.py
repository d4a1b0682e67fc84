"""CPU: the C restatement against the UNMODIFIED reference compiled into
oracle/_ref/libtemo_ref.so, on the reference's own randomized suites (verify.hpp master
seeds 7001/7002). Everything is compared bit-for-bit. Skipped when _ref is not built."""
import numpy as np
import pytest

from conftest import Stream, operator_instance


def test_rng_stream(oracle, ref):
    for seed in (0, 1, 7, 42, 2**64 - 1):
        assert np.array_equal(oracle.uniform(seed, 123456789, 4096), ref.uniform(seed, 123456789, 4096))
    for n in (1, 2, 3, 64, 1000):
        a, ca = oracle.shuffle_indices(11, 17, n)
        b, cb = ref.shuffle_indices(11, 17, n)
        assert np.array_equal(a, b) and ca == cb == 17 + n - 1


def test_rv_select_suite_7001(oracle, ref):
    """verify.hpp:53-76 instance generator, 200 instances; also the set-form oracle of the reference."""
    for k in range(200):
        g = Stream(ref, 7001 + k)
        n, m = g.pick(1, 64), g.pick(2, 3)
        H = g.pick(1, 14) if m == 2 else g.pick(1, 4)
        t_max = g.pick(1, 200)
        t = g.pick(0, t_max)
        v0, gamma = ref.make_ref_set(m, H)
        f = g.tensor(n, m) * 10.0
        a = oracle.rv_select(f, v0, gamma, t, t_max, 2.0)
        b = ref.rv_select(f, v0, gamma, t, t_max, 2.0)
        c = ref.rv_select(f, v0, gamma, t, t_max, 2.0, set_form=True)
        assert np.array_equal(a.elite, b.elite) and np.array_equal(a.validity, b.validity), k
        assert np.array_equal(a.elite, c.elite) and np.array_equal(a.validity, c.validity), k
        assert np.array_equal(a.assoc, b.assoc) and np.array_equal(a.theta, b.theta) and np.array_equal(a.apd, b.apd), k


@pytest.mark.parametrize("op", [0, 1])
def test_operator_suite_7002(oracle, ref, op):
    """verify.hpp:117-182: seed 7002 + op*1000003 + k, n<=16, d<=8, random per-gene bounds."""
    for k in range(100):
        seed = 7002 + op * 1000003 + k
        g = Stream(ref, seed)
        n, d, lo, hi, x = operator_instance(g, 2, 16, 8)
        s = seed ^ 0x5EED
        if op == 0:
            a, ca = oracle.sbx(x, s, 0, lo, hi)
            b, cb = ref.sbx(x, s, 0, lo, hi)
            c, _ = ref.sbx(x, s, 0, lo, hi, scalar=True)
        else:
            a, ca = oracle.polynomial_mutation(x, s, 0, lo, hi)
            b, cb = ref.polynomial_mutation(x, s, 0, lo, hi)
            c, _ = ref.polynomial_mutation(x, s, 0, lo, hi, scalar=True)
        assert np.array_equal(a, b) and np.array_equal(a, c) and ca == cb, (op, k)
        a, ca = oracle.ga_reproduce(x, s, 5, lo, hi)
        b, cb = ref.ga_reproduce(x, s, 5, lo, hi)
        assert np.array_equal(a, b) and ca == cb, (op, k)


def test_dtlz_random(oracle, ref):
    g = Stream(ref, 9400)
    for m, d in ((2, 2), (3, 7), (3, 500), (6, 41), (10, 1000)):
        x = g.tensor(13, d)
        for pid in (1, 2, 3, 4):
            assert np.array_equal(oracle.evaluate(f"dtlz{pid}", x, m), ref.evaluate(f"dtlz{pid}", x, m)), (pid, m, d)


def test_refvec_streaming_gamma_matches_dense(oracle, ref):
    """the streamed gamma equals the reference's dense R x R form, also after
    an anisotropic adaptation."""
    for m, H in ((3, 40), (10, 4), (2, 50), (4, 9)):
        v0, g0 = oracle.make_ref_set(m, H)
        rv0, rg0 = ref.make_ref_set(m, H)
        assert np.array_equal(v0, rv0) and np.array_equal(g0, rg0), (m, H)
        zmin = np.linspace(0.0, 0.3, m)
        zmax = zmin + np.linspace(0.2, 7.0, m)
        a = oracle.adapt(v0, v0, g0, zmin, zmax)
        b = ref.adapt(v0, v0, g0, zmin, zmax)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), (m, H)


@pytest.mark.parametrize("cfg", [("dtlz2", 40, 9, 3, 0, 12, 3), ("dtlz1", 33, 15, 2, 0, 20, 8), ("dtlz4", 105, 12, 3, 13, 25, 1)])
def test_pipeline_and_lockstep(oracle, ref, cfg):
    """Free-running runs agree bit-for-bit, and so does a generation stepped on explicit state."""
    problem, n, d, m, H, gens, seed = cfg
    a = oracle.rvea_run(problem, n, d, m, gens, seed=seed, lattice_h=H)
    b = ref.rvea_run(problem, n, d, m, gens, seed=seed, lattice_h=H)
    assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["f"], b["f"]) and np.array_equal(a["pop_size"], b["pop_size"])
    # lock-step
    Hh = H or oracle.lattice_density_for(m, n)
    v0, gamma = oracle.make_ref_set(m, Hh)
    lo, hi = oracle.problem_bounds(problem, d, m)
    x, c = oracle.random_reproduce(n, d, seed, 0, lo, hi)
    f = oracle.evaluate(problem, x, m)
    adapt_every = max(1, int(np.ceil(0.1 * gens)))
    so = dict(x=x, f=f, v=v0, gamma=gamma, counter=c)
    sr = dict(so)
    for t in range(gens):
        so = oracle.generation(problem, n, m, seed, so["counter"], lo, hi, t, gens, 2.0, adapt_every, v0, so["v"], so["gamma"], so["x"], so["f"])
        sr = ref.generation(problem, n, m, seed, sr["counter"], lo, hi, t, gens, 2.0, adapt_every, v0, sr["v"], sr["gamma"], sr["x"], sr["f"])
        for key in ("x", "f", "v", "gamma", "offspring", "f_off", "elite"):
            assert np.array_equal(so[key], sr[key]), (t, key)
        assert so["counter"] == sr["counter"]
    assert np.array_equal(so["x"], a["x"]) and np.array_equal(so["f"], a["f"])


@pytest.mark.parametrize("op", ["de", "pso", "cso", "random"])
def test_pipeline_other_operators(oracle, ref, op):
    """The run loop with the other operators (algorithms.hpp:253-268): the C restatement's free run, and a run stepped
    generation by generation on explicit state (the form the GPU lock-step tests use), against the reference's rvea_run."""
    for problem, n, d, m, H, gens, seed in (("dtlz2", 40, 9, 3, 0, 12, 3), ("dtlz4", 57, 11, 3, 0, 10, 4)):
        a = oracle.rvea_run_op(op, problem, n, d, m, gens, seed=seed, lattice_h=H)
        b = ref.rvea_run_op(op, problem, n, d, m, gens, seed=seed, lattice_h=H)
        assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["f"], b["f"]) and np.array_equal(a["pop_size"], b["pop_size"])
        for chk in (oracle, ref):
            v0, gamma = chk.make_ref_set(m, H or chk.lattice_density_for(m, n))
            lo, hi = chk.problem_bounds(problem, d, m)
            x, c = chk.random_reproduce(n, d, seed, 0, lo, hi)
            st = dict(x=x, f=chk.evaluate(problem, x, m), v=v0, gamma=gamma, counter=c, swarm=None)
            adapt_every = max(1, int(np.ceil(0.1 * gens)))
            for t in range(gens):
                st = chk.generation_op(op, problem, n, m, seed, st["counter"], lo, hi, t, gens, 2.0, adapt_every, v0, st["v"],
                                       st["gamma"], st["x"], st["f"], st["swarm"])
                assert st["x"].shape[0] == b["pop_size"][t]
            assert np.array_equal(st["x"], b["x"]) and np.array_equal(st["f"], b["f"]) and st["counter"] == a["counter"]


def test_metrics_against_reference(oracle, ref):
    """igd and the Monte-Carlo hypervolume of the C restatement against metrics.hpp on random instances."""
    from conftest import Stream
    for k in range(12):
        g = Stream(ref, 4400 + k)
        n, m, n_ref = g.pick(1, 80), g.pick(2, 6), g.pick(1, 50)
        f, pf = g.tensor(n, m) * 2.0, g.tensor(n_ref, m)
        rp, lo = np.full(m, 1.5), np.full(m, 0.1 * (k % 3))
        assert oracle.igd(f, pf) == ref.igd(f, pf)
        assert oracle.hv_mc_box(f, lo, rp, 300 + k, 77 + k) == ref.hv_mc_box(f, lo, rp, 300 + k, 77 + k)
        assert oracle.hv_mc_box(f, None, rp, 300 + k, 77 + k) == ref.hv_mc_box(f, None, rp, 300 + k, 77 + k)


def test_archive_against_reference(oracle, ref):
    from conftest import Stream
    for k in range(10):
        g = Stream(ref, 6600 + k)
        n0, n1, d, m = g.pick(0, 40), g.pick(1, 60), g.pick(1, 5), g.pick(2, 5)
        q = float(g.pick(2, 9))
        x0, x1 = (g.tensor(n0, d) if n0 else np.empty((0, d))), g.tensor(n1, d)
        f0, f1 = (np.floor(g.tensor(n0, m) * q) / q if n0 else np.empty((0, m))), np.floor(g.tensor(n1, m) * q) / q
        a = ref.archive_insert(None, None, x0, f0) if n0 else (None, None)
        b = oracle.archive_insert(None, None, x0, f0) if n0 else (None, None)
        for cap in (0, 7):
            ra, rb = ref.archive_insert(a[0], a[1], x1, f1, cap), oracle.archive_insert(b[0], b[1], x1, f1, cap)
            assert np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1], rb[1]), (k, cap)
        assert np.array_equal(ref.crowding_distance(f1), oracle.crowding_distance(f1))


def test_nsga2_against_reference(oracle, ref):
    rng = np.random.default_rng(2)
    for n, m, q in ((50, 3, 6.0), (200, 2, 50.0), (120, 5, 3.0), (1, 3, 2.0), (2, 2, 2.0), (90, 4, 1000.0)):
        f = np.floor(rng.random((n, m)) * q) / q
        assert np.array_equal(oracle.nondominated_sort(f), ref.nondominated_sort(f)), (n, m)
        for t in (0, n // 3, n // 2, n):
            assert np.array_equal(oracle.nsga2_select(f, t), ref.nsga2_select(f, t)), (n, m, t)
    for problem, n, d, m, gens, seed in (("dtlz2", 41, 9, 3, 10, 3), ("dtlz3", 64, 20, 4, 8, 5)):
        a, b = oracle.nsga2_run(problem, n, d, m, gens, seed=seed), ref.nsga2_run(problem, n, d, m, gens, seed=seed)
        assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["f"], b["f"])
        # the generation stepped on explicit state (what the GPU lock-step test uses) reproduces the free run
        lo, hi = oracle.problem_bounds(problem, d, m)
        x, c = oracle.random_reproduce(n, d, seed, 0, lo, hi)
        st = dict(x=x, f=oracle.evaluate(problem, x, m), counter=c)
        for _ in range(gens):
            st = oracle.nsga2_generation(problem, m, seed, st["counter"], lo, hi, st["x"], st["f"])
        assert np.array_equal(st["x"], b["x"]) and np.array_equal(st["f"], b["f"]) and st["counter"] == a["counter"]


def test_swarm_operators_suite_7002(oracle, ref):
    """DE / PSO / CSO: the C restatement against the compiled reference, batched and
    scalar-oracle forms, on the reference's own operator_suite instances (verify.hpp:117-182: master seed 7002,
    ops 2..4, 100 instances each) - outputs, updated swarm state and draw counters bit for bit."""
    from conftest import Stream, swarm_instance
    for op in (2, 3, 4):
        for k in range(100):
            seed = 7002 + op * 1000003 + k
            g = Stream(ref, seed)
            n, d, lo, hi, x, scores = swarm_instance(g, 4 if op == 2 else 2, 16, 8)
            s = seed ^ 0xabcdef
            if op == 2:
                got, c = oracle.de_reproduce(x, s, 0, lo, hi)
                for scalar in (False, True):
                    exp, ce = ref.de_reproduce(x, s, 0, lo, hi, scalar=scalar)
                    assert c == ce and np.array_equal(got, exp), (k, scalar)
            elif op == 3:
                vel, pbx, pbs = np.zeros_like(x), x * 0.5, scores + 0.25  # verify.hpp:157-160
                got = oracle.pso_reproduce(x, scores, s, 0, lo, hi, vel, pbx, pbs)
                for scalar in (False, True):
                    exp = ref.pso_reproduce(x, scores, s, 0, lo, hi, vel, pbx, pbs, scalar=scalar)
                    assert got[1] == exp[1] and all(np.array_equal(a, b) for a, b in zip(got[::2] + got[3:4], exp[::2] + exp[3:4])), (k, scalar)
            else:
                vel = np.zeros_like(x)
                got = oracle.cso_reproduce(x, scores, s, 0, lo, hi, vel)
                for scalar in (False, True):
                    exp = ref.cso_reproduce(x, scores, s, 0, lo, hi, vel, scalar=scalar)
                    assert got[1] == exp[1] and np.array_equal(got[0], exp[0]) and np.array_equal(got[2], exp[2]), (k, scalar)


def test_swarm_operators_multi_step_and_contracts(oracle, ref):
    """Several chained steps (the state carries over), larger shapes, ties in the scores, and de_reproduce's n >= 4."""
    rng = np.random.default_rng(3)
    n, d = 37, 23
    lo, hi = -rng.random(d) - 1.0, rng.random(d) + 0.5
    x = lo + rng.random((n, d)) * (hi - lo)
    scores = np.round(rng.random(n), 1)  # many ties
    vo, pxo, pso_ = np.zeros_like(x), x.copy(), scores.copy()
    vr, pxr, psr = vo.copy(), pxo.copy(), pso_.copy()
    xo, xr, co, cr = x.copy(), x.copy(), 11, 11
    for step in range(4):
        sc = np.round(rng.random(n), 1)
        xo, co, vo, pxo, pso_ = oracle.pso_reproduce(xo, sc, 5, co, lo, hi, vo, pxo, pso_)
        xr, cr, vr, pxr, psr = ref.pso_reproduce(xr, sc, 5, cr, lo, hi, vr, pxr, psr)
        assert co == cr and np.array_equal(xo, xr) and np.array_equal(vo, vr) and np.array_equal(pxo, pxr) and np.array_equal(pso_, psr)
    vo = vr = np.zeros_like(x)
    xo, xr, co, cr = x.copy(), x.copy(), 3, 3
    for step in range(4):
        sc = np.round(rng.random(n), 1)
        xo, co, vo = oracle.cso_reproduce(xo, sc, 8, co, lo, hi, vo)
        xr, cr, vr = ref.cso_reproduce(xr, sc, 8, cr, lo, hi, vr)
        assert co == cr and np.array_equal(xo, xr) and np.array_equal(vo, vr)
    a, ca = oracle.de_reproduce(x, 9, 100, lo, hi, p=(0.7, 0.3))
    b, cb = ref.de_reproduce(x, 9, 100, lo, hi, p=(0.7, 0.3))
    assert ca == cb == 100 + 4 * n + n * d and np.array_equal(a, b)
    with pytest.raises(ValueError):
        oracle.de_reproduce(x[:3], 1, 0, lo, hi)
    with pytest.raises(Exception):
        ref.de_reproduce(x[:3], 1, 0, lo, hi)
