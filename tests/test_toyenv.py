"""Neuroevolution evaluator: mlp_forward / env_rollout / make_problem("toy2" | "toy3")
(problems.hpp:105-294) and the scale-format CSV writer (io.hpp:18-76, temo.cpp:229-246).

CPU: the C restatement against the fixtures recorded from the unmodified reference (tests/golden/toyenv.npz) and
against the compiled reference itself. GPU: the device evaluator against the same — bit for bit (tanh follows the host
libm's operation sequence, sin / cos of the phase come from the host libm) — and RVEA runs on the toy problems in lock-step."""
import os

import numpy as np
import pytest

from conftest import golden


def _finite(p):
    return np.isfinite(p).all(axis=1)


# ------------------------------------------------------------------------------------------------ oracle (CPU)
def test_oracle_toyenv_against_golden(checkers):
    g = golden("toyenv")
    p = g["params"]
    for chk in checkers:
        for T, m in ((100, 2), (100, 3), (1, 2), (37, 3)):
            assert np.array_equal(chk.env_rollout(p, T, m), g[f"ret_T{T}_m{m}"]), (type(chk).__name__, T, m)
        assert np.array_equal(chk.env_rollout(g["params_h64"], 50, 3, hidden=64), g["ret_h64"])
        assert np.array_equal(chk.mlp_forward(np.where(np.isfinite(p), p, 0.0), g["obs"]), g["act"])
        assert np.array_equal(chk.evaluate("toy2", p[_finite(p)], 2), g["f_toy2"])
        lo, hi = chk.problem_bounds("toy3", 114, 3)
        assert np.all(lo == -1.0) and np.all(hi == 1.0)
    # known answers: non-finite parameters score -1e9 in every objective (problems.hpp:224-230); actions lie in (-1, 1);
    # the control return is minus a sum of squares; one step from rest gives fwd = 0.1 a1
    assert np.all(g["ret_T100_m3"][7] == -1e9) and np.all(g["ret_T100_m2"][9] == -1e9)
    assert np.all(np.abs(g["act"]) < 1.0)
    ok = _finite(p)
    assert np.all(g["ret_T100_m2"][ok, 1] <= 0.0) and np.all(g["ret_T100_m2"][ok, 1] >= -200.0)
    obs0 = np.tile(np.array([0.0, 1.0, 0.0, 1.0]), (int(ok.sum()), 1))
    a = checkers[0].mlp_forward(p[ok], obs0)
    assert np.array_equal(g["ret_T1_m2"][ok, 0], 0.9 * 0.0 + 0.1 * a[:, 0])


def test_oracle_toy_runs_against_golden(oracle):
    """Whole RVEA runs on toy2 / toy3 through the C restatement reproduce the reference's runs bit for bit."""
    g = golden("toyenv")
    for tag, (problem, m, n, gens, seed) in (("run2", ("toy2", 2, 40, 12, 5)), ("run3", ("toy3", 3, 66, 10, 8))):
        out = oracle.rvea_run(problem, n, 114, m, gens, seed=seed)
        assert np.array_equal(out["pop_size"], g[f"{tag}_pop"])
        assert np.array_equal(out["x"], g[f"{tag}_x"]) and np.array_equal(out["f"], g[f"{tag}_f"])


# ------------------------------------------------------------------------------------------------ product (GPU)
@pytest.mark.gpu
def test_device_env_rollout_bit_exact(tb, checkers):
    g = golden("toyenv")
    p = g["params"]
    for T, m in ((100, 2), (100, 3), (1, 2), (37, 3)):
        assert np.array_equal(tb.env_rollout(p, T, m), g[f"ret_T{T}_m{m}"]), (T, m)
    assert np.array_equal(tb.env_rollout(g["params_h64"], 50, 3, hidden=64), g["ret_h64"])
    assert np.array_equal(tb.mlp_forward(np.where(np.isfinite(p), p, 0.0), g["obs"]), g["act"])
    ok = _finite(p)
    assert np.array_equal(tb.evaluate("toy2", p[ok], 2), g["f_toy2"])
    assert np.array_equal(tb.evaluate("toy3", p[ok], 3, horizon=20), g["f_toy3_T20"])
    # a larger random batch (several CTAs, a partial last one) against the live checker
    chk = checkers[-1]
    rng = np.random.default_rng(12)
    big = rng.uniform(-1.0, 1.0, (3001, 114))
    big[rng.integers(0, 3001, 7), rng.integers(0, 114, 7)] = np.nan
    assert np.array_equal(tb.env_rollout(big, 60, 3), chk.env_rollout(big, 60, 3))
    prob = tb.make_problem("toy2", toy_horizon=33)
    assert prob.dim == 114 and prob.num_obj == 2 and prob.maximization and np.all(prob.lower == -1.0) and np.all(prob.upper == 1.0)
    assert np.array_equal(prob.evaluate(big[:100]), -chk.env_rollout(big[:100], 33, 2))
    with pytest.raises(ValueError):
        tb.make_problem("toy3", dim=100)            # problems.hpp:284
    with pytest.raises(ValueError):
        tb.env_rollout(np.zeros((2, 100)))          # problems.hpp:213


@pytest.mark.gpu
@pytest.mark.parametrize("case", [("toy2", 2, 40, 12, 5), ("toy3", 3, 66, 10, 8)])
def test_toy_runs_lockstep_and_free_running(tb, checkers, case):
    """RVEA on the toy problems: lock-step generations (offspring, objectives and survivor sets bit-identical: there is
    no libm difference left on this path), then the free-running device run against the recorded reference run."""
    from test_gpu_parity import _lockstep
    problem, m, n, gens, seed = case
    _lockstep(tb, checkers[-1], problem, n, 114, m, gens, seed)
    g = golden("toyenv")
    tag = "run2" if problem == "toy2" else "run3"
    rec = tb.rvea_run(tb.make_problem(problem), tb.RunConfig(pop=n, generations=gens, seed=seed))
    assert np.array_equal(np.array([r.pop_size for r in rec.rows]), g[f"{tag}_pop"])
    assert np.array_equal(rec.final_x, g[f"{tag}_x"]) and np.array_equal(rec.final_f, g[f"{tag}_f"])


# ------------------------------------------------------------------------------------------------ CSV / harness formats
def test_csv_writer_and_scale_format(tmp_path):
    from paper_2404_01159_b200 import harness
    assert harness.fmt(0.1) == "0.10000000000000001" and harness.fmt(3) == "3" and harness.fmt(1e300) == "1.0000000000000001e+300"
    assert harness.fmt(float("nan")) == "nan" and harness.fmt(2.5) == "2.5"
    assert harness.median([3.0, 1.0, 2.0]) == 2.0 and harness.median([4.0, 1.0, 2.0, 3.0]) == 2.5 and np.isnan(harness.median([]))
    assert harness.iqr([1.0, 2.0, 3.0, 4.0, 5.0]) == 3.0 and harness.iqr([7.0]) == 0.0   # quartiles = medians of the halves
    path = tmp_path / "scale.csv"
    w = harness.scale_csv(path, {"threads": "8", "command": "scale", "seed": "42"})
    w.row(harness.scale_row("population", 4096, 100, 3, 20, 1.5, 30.0, "ok"))
    w.row(harness.scale_row("dimension", 100, 512, 3, 20, 0.0, 0.0, "skipped"))
    w.close()
    lines = path.read_text().splitlines()
    assert lines[0] == "# version=0.1.0"
    assert lines[1] == "# config: command=scale seed=42 threads=8"          # keyed and ordered (std::map)
    assert lines[2] == "series,n,d,m,generations,tensor_ms,oracle_ms,speedup,status"
    assert lines[3] == "population,4096,100,3,20,1.5,30,20,ok"
    assert lines[4] == "dimension,100,512,3,20,0,0,0,skipped"
    # median per-generation duration from cumulative elapsed_ms (temo.cpp:229-237)
    assert harness.median_generation_ms([10.0, 12.0, 17.0, 19.0]) == 3.5
