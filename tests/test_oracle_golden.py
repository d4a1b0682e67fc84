"""CPU: the C restatement (oracle/temo_oracle.c) against the committed golden fixtures
(generated from the unmodified reference by oracle/gen_golden.py) and against the known
answers in the reference's own unit tests. Bit-exact unless stated."""
import math

import numpy as np
import pytest

from conftest import golden


def test_rng_golden(oracle):
    g = golden("rng")
    for s, row in zip(g["seeds"], g["draws"]):
        assert [oracle.value_at(int(s), k) for k in range(24)] == list(row)
    assert [oracle.value_at(42, int(k)) for k in g["far_k"]] == list(g["far"])
    # SURVEY.md §8c recorded values
    assert oracle.value_at(42, 0) == 0.5934224109845303
    assert oracle.value_at(42, 1) == 0.59611887183020762
    perm, c = oracle.shuffle_indices(42, 0, 20)
    assert np.array_equal(perm, g["perm20"]) and c == int(g["c20"]) == 19  # test_rng.cpp:37-54
    perm, c = oracle.shuffle_indices(5, 1000, 257)
    assert np.array_equal(perm, g["perm257"]) and c == int(g["c257"])
    pool, c = oracle.parent_pool_indices(77, 105, 42, 5000)
    assert np.array_equal(pool, g["pool"]) and c == int(g["cpool"]) == 5105
    ident, c = oracle.parent_pool_indices(105, 105, 42, 5000)  # algorithms.hpp:214-217
    assert np.array_equal(ident, np.arange(105)) and c == 5000


def test_rng_kat_reference_tests(oracle):
    # test_rng.cpp:29-35: blocks are disjoint subsequences of one stream
    assert list(oracle.uniform(7, 0, 6)) == [oracle.value_at(7, i) for i in range(6)]
    # test_rng.cpp:16-27
    u = oracle.uniform(1234, 0, 100000)
    assert u.min() >= 0.0 and u.max() < 1.0 and abs(u.mean() - 0.5) < 0.01
    perm, c = oracle.shuffle_indices(3, 0, 1)
    assert list(perm) == [0] and c == 0


@pytest.mark.parametrize("tag", ["a", "b", "c", "odd", "wide"])
def test_operators_golden(oracle, tag):
    g = golden("operators")
    x, lo, hi = g[f"{tag}_x"], g[f"{tag}_lower"], g[f"{tag}_upper"]
    seed = int(g[f"{tag}_seed"][0])
    c = g[f"{tag}_counters"]
    n, d = x.shape
    out, cc = oracle.sbx(x, seed, 0, lo, hi)
    assert np.array_equal(out, g[f"{tag}_sbx"]) and cc == int(c[0]) == 3 * (n // 2) * d + n // 2
    out, cc = oracle.polynomial_mutation(x, seed, 0, lo, hi)
    assert np.array_equal(out, g[f"{tag}_pm"]) and cc == int(c[1]) == 2 * n * d
    out, cc = oracle.ga_reproduce(x, seed, 0, lo, hi)
    assert np.array_equal(out, g[f"{tag}_ga"]) and cc == int(c[2]) == (n - 1) + 3 * (n // 2) * d + n // 2 + 2 * n * d
    out, _ = oracle.polynomial_mutation(x, seed, 11, lo, hi, ga=(1.0, 20.0, float(d) * 0.6, 20.0))
    assert np.array_equal(out, g[f"{tag}_pm_hot"])
    out, _ = oracle.ga_reproduce(x, seed, 3, lo, hi, ga=(0.5, 15.0, 2.0, 10.0))
    assert np.array_equal(out, g[f"{tag}_ga_pc"])


def test_operator_kats(oracle):
    g = golden("operators")
    rr, c = oracle.random_reproduce(5, 7, 42, 3, np.linspace(-1, 0, 7), np.linspace(1, 3, 7))
    assert np.array_equal(rr, g["rr"]) and c == int(g["rr_counter"][0]) == 38
    # test_operators.cpp:73-84: delta(0.5)=0, u->0 drives to lower, u->1 to upper
    assert oracle.polynomial_delta(0.5, 0.3, 0.0, 1.0, 20.0) == 0.0
    assert abs(0.3 + oracle.polynomial_delta(1e-300, 0.3, 0.0, 1.0, 20.0) - 0.0) < 1e-9
    assert abs(0.3 + oracle.polynomial_delta(1.0 - 1e-16, 0.3, 0.0, 1.0, 20.0) - 1.0) < 1e-2
    # test_operators.cpp:43-50: pc = 0 copies parents; :86-102 pm = 0 is the identity
    x = g["a_x"]
    out, _ = oracle.sbx(x, 1, 0, g["a_lower"], g["a_upper"], ga=(0.0, 20.0, 1.0, 20.0))
    assert np.array_equal(out, x)
    out, _ = oracle.polynomial_mutation(x, 1, 0, g["a_lower"], g["a_upper"], ga=(1.0, 20.0, 0.0, 20.0))
    assert np.array_equal(out, x)
    # test_operators.cpp:52-61: odd row passes through
    xo = g["odd_x"]
    out, _ = oracle.sbx(xo, 9, 0, g["odd_lower"], g["odd_upper"])
    assert np.array_equal(out[-1], xo[-1])


@pytest.mark.parametrize("m", [3, 2, 5, 10])
def test_problems_golden(oracle, m):
    g = golden("problems")
    x = g[f"x_m{m}"]
    for pid in (1, 2, 3, 4):
        f = oracle.evaluate(f"dtlz{pid}", x, m)
        assert np.array_equal(f, g[f"f{pid}_m{m}"]), pid
    # test_problems.cpp:8-33: at x = 0.5 the g term vanishes
    f1 = oracle.evaluate("dtlz1", x[:1], m)
    assert abs(f1.sum() - 0.5) < 1e-9
    f2 = oracle.evaluate("dtlz2", x[:1], m)
    assert abs((f2 ** 2).sum() - 1.0) < 1e-12
    # batch == row by row (test_problems.cpp:35-47)
    rows = np.vstack([oracle.evaluate("dtlz3", x[i:i + 1], m) for i in range(x.shape[0])])
    assert np.array_equal(rows, oracle.evaluate("dtlz3", x, m))


def test_problem_contract(oracle):
    with pytest.raises(ValueError):
        oracle.evaluate("dtlz2", np.zeros((2, 2)), 3)  # d < m (problems.hpp:72)


@pytest.mark.parametrize("mh", [(3, 4), (2, 9), (3, 13), (5, 4), (10, 2)])
def test_refvec_golden(oracle, mh):
    m, H = mh
    g = golden("refvec")
    v0, gamma = oracle.make_ref_set(m, H)
    assert np.array_equal(v0, g[f"v0_{m}_{H}"]) and np.array_equal(gamma, g[f"gamma_{m}_{H}"])
    v1, g1 = oracle.adapt(v0, v0, gamma, g[f"zmin_{m}_{H}"], g[f"zmax_{m}_{H}"])
    assert np.array_equal(v1, g[f"v1_{m}_{H}"]) and np.array_equal(g1, g[f"g1_{m}_{H}"])
    zbad = g[f"zmax_{m}_{H}"].copy()
    zbad[m - 1] = g[f"zmin_{m}_{H}"][m - 1]
    v2, g2 = oracle.adapt(v0, v1, g1, g[f"zmin_{m}_{H}"], zbad)
    assert np.array_equal(v2, g[f"v2_{m}_{H}"]) and np.array_equal(g2, g[f"g2_{m}_{H}"])
    assert np.array_equal(v2, v1)  # degenerate range leaves the set untouched (refvec.hpp:136-137)


def test_refvec_kats(oracle):
    g = golden("refvec")
    for m, n, h in g["density"]:
        assert oracle.lattice_density_for(int(m), int(n)) == int(h)
    # test_refvec.cpp:24-38
    lat = oracle.simplex_lattice(3, 13)
    assert lat.shape == (105, 3) and np.allclose(lat.sum(axis=1), 1.0, atol=1e-12)
    assert np.array_equal(oracle.simplex_lattice(2, 1), [[1.0, 0.0], [0.0, 1.0]])
    for m in range(2, 6):
        for h in range(1, 21):
            assert oracle.lattice_count(m, h) == math.comb(h + m - 1, m - 1)
    # test_refvec.cpp:62-85
    assert np.allclose(oracle.min_vector_angles(np.eye(2)), math.pi / 2, rtol=1e-14)
    inv = 1.0 / math.sqrt(2.0)
    assert np.allclose(oracle.min_vector_angles([[1, 0], [0, 1], [inv, inv]]), math.pi / 4, rtol=1e-12)
    with pytest.raises(ValueError):
        oracle.min_vector_angles([[1.0, 0.0], [1.0, 0.0]])
    with pytest.raises(ValueError):
        oracle.min_vector_angles([[1.0, 0.0]])
    with pytest.raises(ValueError):
        oracle.normalize_to_unit(np.zeros((1, 2)))
    # test_refvec.cpp:87-113: unit(2,1)
    out, _ = oracle.adapt([[inv, inv], [1, 0]], [[inv, inv], [1, 0]], [0.5, 0.5], [0.0, 0.0], [2.0, 1.0])
    assert np.allclose(out[0], [2 / math.sqrt(5), 1 / math.sqrt(5)], rtol=1e-12)


def test_selection_golden(oracle):
    g = golden("selection")
    for k in range(int(g["count"][0])):
        m, H, t, t_max = (int(v) for v in g[f"mh_{k}"])
        v0, gamma = oracle.make_ref_set(m, H)
        s = oracle.rv_select(g[f"f_{k}"], v0, gamma, t, t_max, 2.0)
        assert np.array_equal(s.elite, g[f"elite_{k}"]), k
        assert np.array_equal(s.validity, g[f"valid_{k}"]), k
        assert np.array_equal(s.assoc, g[f"assoc_{k}"]), k
        assert np.array_equal(s.theta, g[f"theta_{k}"]), k
        assert np.array_equal(s.apd, g[f"apd_{k}"]), k
    s = oracle.rv_select(g["crafted_f"], g["crafted_v"], g["crafted_gamma"], 37, 100, 2.0)
    assert np.array_equal(s.elite, g["crafted_elite"]) and np.array_equal(s.validity, g["crafted_valid"])
    assert np.array_equal(s.assoc, g["crafted_assoc"]) and np.array_equal(s.apd, g["crafted_apd"])
    assert s.assoc[12] == 0 and s.apd[12] == 0.0  # row at the ideal point (selection.hpp:167-169)
    assert 7 not in s.elite and 21 not in s.elite   # exact ties resolve to the lowest row (3)


def test_selection_kats(oracle):
    # test_selection.cpp:85-111 restated through rv_select: t = 0 -> APD is the translated norm
    v = np.eye(2)
    gamma = np.array([0.7, 0.7])
    f = np.array([[3.0, 4.0], [0.0, 0.0]])
    s = oracle.rv_select(f, v, gamma, 0, 10, 2.0)
    assert s.apd[0] == 5.0 and s.apd[1] == 0.0
    assert oracle.apd_penalty(2, 10, 10, 2.0) == 2.0 and oracle.apd_penalty(3, 0, 10, 2.0) == 0.0
    with pytest.raises(ValueError):
        oracle.rv_select(f, v, np.zeros(2), 0, 10, 2.0)  # gamma must be positive
    # test_selection.cpp:157-171: rows on distinct vectors all survive; smaller norm wins
    v0, g3 = oracle.make_ref_set(2, 2)
    s = oracle.rv_select(2.0 * v0 + 1.0, v0, g3, 0, 10, 2.0)
    assert len(s.elite) == 3
    s = oracle.rv_select([[2, 2], [3, 3], [1, 9], [9, 1]], v0, g3, 5, 10, 2.0)
    assert 1 not in s.elite


def test_pipeline_golden(oracle):
    g = golden("pipeline")
    r = oracle.rvea_run("dtlz1", 105, 12, 3, 100, seed=42, lattice_h=13)
    assert np.array_equal(r["x"], g["c1_x"]) and np.array_equal(r["f"], g["c1_f"])
    assert np.array_equal(r["pop_size"], g["c1_pop"])
    assert list(r["pop_size"][::10]) == [69, 88, 102, 86, 83, 85, 78, 88, 76, 79]
    assert r["f"][0, 0] == 11.214396312698408 and r["x"].shape[0] == 103
    r = oracle.rvea_run("dtlz2", 12, 8, 3, 10, seed=77, lattice_h=3)  # test_algorithms.cpp:198-210
    assert np.array_equal(r["x"], g["s77_x"]) and np.array_equal(r["f"], g["s77_f"])
    r = oracle.rvea_run("dtlz3", 64, 20, 4, 30, seed=5)
    assert np.array_equal(r["x"], g["d3_x"]) and np.array_equal(r["pop_size"], g["d3_pop"])
    r = oracle.rvea_run("dtlz4", 50, 10, 2, 25, seed=11)
    assert np.array_equal(r["x"], g["d4_x"]) and np.array_equal(r["f"], g["d4_f"])


OPS_CASES = {"a": ("dtlz2", 40, 9, 3, 0, 12, 3), "b": ("dtlz1", 33, 15, 2, 0, 20, 8), "c": ("dtlz3", 64, 20, 4, 0, 15, 5)}


@pytest.mark.parametrize("op", ["de", "pso", "cso", "random"])
def test_pipeline_other_operators_golden(oracle, op):
    """rvea_run with RunConfig::op = de / pso / cso / random (algorithms.hpp:253-268): the C restatement against
    fixtures recorded from the compiled reference (oracle/gen_golden.py)."""
    g = golden("pipeline_ops")
    for tag, (problem, n, d, m, H, gens, seed) in OPS_CASES.items():
        r = oracle.rvea_run_op(op, problem, n, d, m, gens, seed=seed, lattice_h=H)
        assert np.array_equal(r["x"], g[f"{op}_{tag}_x"]) and np.array_equal(r["f"], g[f"{op}_{tag}_f"]), (op, tag)
        assert np.array_equal(r["pop_size"], g[f"{op}_{tag}_pop"]), (op, tag)


def test_metrics_golden(oracle):
    """igd / hv_mc_box / hv_mc (metrics.hpp:21-44, 76-124): the C restatement against values recorded from the compiled
    reference, bit for bit (the hypervolume is an integer hit count times the box volume)."""
    g = golden("metrics")
    for tag in "abcd":
        f, pf, rp, lo = g[f"{tag}_f"], g[f"{tag}_pf"], g[f"{tag}_ref"], g[f"{tag}_lo"]
        samples, seed = (int(v) for v in g[f"{tag}_samples"])
        assert oracle.igd(f, pf) == g[f"{tag}_igd"][0], tag
        assert oracle.hv_mc_box(f, lo, rp, samples, seed) == tuple(g[f"{tag}_hv_box"]), tag
        assert oracle.hv_mc_box(f, None, rp, samples, seed) == tuple(g[f"{tag}_hv"]), tag
    assert oracle.hv_mc_box(g["a_f"], g["a_ref"], g["a_lo"], 100, 1) == (0.0, 0.0)  # empty box (metrics.hpp:85)
    with pytest.raises(ValueError):
        oracle.igd(np.zeros((0, 3)), g["a_pf"])


def test_archive_golden(oracle):
    """Archive::insert with duplicates, dominated rows and a crowding-distance cap (algorithms.hpp:72-144)."""
    from conftest import _archive_case
    g = golden("metrics")
    for tag in ("ar0", "ar1", "ar2"):
        _archive_case(lambda xo, fo, xn, fn, cap: oracle.archive_insert(xo, fo, xn, fn, cap), oracle.crowding_distance, g, tag)


def test_nsga2_golden(oracle):
    """nondominated_sort, nsga2_select and nsga2_run of the C restatement against the recorded reference."""
    g = golden("nsga2")
    for tag in ("s0", "s1", "s2", "s3"):
        f = g[f"{tag}_f"]
        n = f.shape[0]
        assert np.array_equal(oracle.nondominated_sort(f), g[f"{tag}_rank"]), tag
        assert np.array_equal(oracle.nsga2_select(f, n // 2), g[f"{tag}_sel_half"]), tag
        assert np.array_equal(oracle.nsga2_select(f, (n + 2) // 3), g[f"{tag}_sel_third"]), tag
        assert np.array_equal(oracle.nsga2_select(f, n), g[f"{tag}_sel_all"]), tag
    for tag, (problem, n, d, m, gens, seed) in (("r0", ("dtlz2", 40, 9, 3, 12, 3)), ("r1", ("dtlz1", 33, 15, 2, 15, 8))):
        r = oracle.nsga2_run(problem, n, d, m, gens, seed=seed)
        assert np.array_equal(r["x"], g[f"{tag}_x"]) and np.array_equal(r["f"], g[f"{tag}_f"]), tag


def test_lsmop1_restatement_self_checks(oracle):
    """LSMOP1 is not in the reference (parity unpinned): check the restatement against an
    independent numpy transcription of the published definition and its basic properties."""
    d, m, nk = 64, 3, 5
    rng = np.random.default_rng(3)
    lo, hi = oracle.problem_bounds("lsmop1", d, m)
    assert list(lo) == [0.0] * d and list(hi) == [1.0] * (m - 1) + [10.0] * (d - m + 1)
    x = lo + rng.random((7, d)) * (hi - lo)
    f = oracle.evaluate("lsmop1", x, m)
    c = [3.8 * 0.1 * 0.9]
    for _ in range(m - 1):
        c.append(3.8 * c[-1] * (1 - c[-1]))
    sub = np.floor(np.array(c) / sum(c) * (d - m + 1) / nk).astype(int)
    start = np.concatenate([[0], np.cumsum(sub * nk)])
    j1 = np.arange(m, d + 1)  # 1-based gene numbers of the tail
    y = (1.0 + j1 / d) * x[:, m - 1:] - 10.0 * x[:, :1]
    G = np.stack([(y[:, start[i]:start[i + 1]] ** 2).sum(axis=1) / sub[i] / nk for i in range(m)], axis=1)
    shape = np.fliplr(np.cumprod(np.hstack([np.ones((7, 1)), x[:, :m - 1]]), axis=1)) * \
        np.hstack([np.ones((7, 1)), 1.0 - x[:, m - 2::-1]])
    assert np.allclose(f, (1.0 + G) * shape, rtol=1e-13)
    # on the Pareto set (tail genes solve the linkage) the front is the unit simplex
    xs = x.copy()
    xs[:, m - 1:] = 10.0 * xs[:, :1] / (1.0 + j1 / d)
    assert np.allclose(oracle.evaluate("lsmop1", xs, m).sum(axis=1), 1.0, atol=1e-9)


def _swarm_cases():
    g = golden("swarm")
    for tag in ("de0", "de1", "pso0", "pso1", "cso0", "cso1"):
        yield tag, {k[len(tag) + 1:]: g[k] for k in g.files if k.startswith(tag + "_")}


def test_swarm_operators_golden(oracle):
    """DE / PSO / CSO restatements against fixtures generated from the compiled reference (two chained steps each)."""
    for tag, c in _swarm_cases():
        x, lo, hi, sc, seed = c["x"], c["lower"], c["upper"], c["scores"], int(c["seed"][0])
        c1, c2 = (int(v) for v in c["counters"])
        if tag.startswith("de"):
            y1, k1 = oracle.de_reproduce(x, seed, 0, lo, hi)
            y2, k2 = oracle.de_reproduce(y1, seed, k1, lo, hi, p=(0.8, 0.4))
            assert (k1, k2) == (c1, c2) and np.array_equal(y1, c["y1"]) and np.array_equal(y2, c["y2"]), tag
        elif tag.startswith("pso"):
            y1, k1, v1, px1, ps1 = oracle.pso_reproduce(x, sc, seed, 0, lo, hi, np.zeros_like(x), x * 0.5, sc + 0.25)
            y2, k2, v2, px2, ps2 = oracle.pso_reproduce(y1, sc[::-1].copy(), seed, k1, lo, hi, v1, px1, ps1)
            assert (k1, k2) == (c1, c2), tag
            for a, b in ((y1, "y1"), (y2, "y2"), (v1, "v1"), (v2, "v2"), (px2, "px2"), (ps2, "ps2")):
                assert np.array_equal(a, c[b]), (tag, b)
        else:
            y1, k1, v1 = oracle.cso_reproduce(x, sc, seed, 0, lo, hi, np.zeros_like(x))
            y2, k2, v2 = oracle.cso_reproduce(y1, sc[::-1].copy(), seed, k1, lo, hi, v1)
            assert (k1, k2) == (c1, c2), tag
            for a, b in ((y1, "y1"), (y2, "y2"), (v1, "v1"), (v2, "v2")):
                assert np.array_equal(a, c[b]), (tag, b)
