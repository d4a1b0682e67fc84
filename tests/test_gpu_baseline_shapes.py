"""GPU parity at the shapes BASELINE.json's configs actually run.

The reference-vector sets of the headline configuration (m = 3, H = 510: R = 130 816) and of the top of the
population sweep (N = 2^20: H = 1447, R = 1 049 076) make the direction index (csrc/vecindex.cu) three and four
levels deep; config #4's set (m = 10, H = 9: R = 48 620) takes the fp32-filtered scan in eight chunks. None of
the oracle-sized tests in test_gpu_parity.py reaches those code paths, so they are compared here with the CPU
checkers on SAMPLED rows / vectors: the oracle's scan of a row is O(R), so 8192 rows against the full set cost
seconds while the vector set — the thing that selects the code path — is the real one.

reference: detail::rv_core / rv_select (selection.hpp:148-224), min_vector_angles (refvec.hpp:81-100),
adapt_vectors (refvec.hpp:119-131), the generation loop (algorithms.hpp:246-292).
"""
import numpy as np
import pytest

from conftest import ulp_diff
from test_gpu_parity import _check_selection, _lockstep

pytestmark = pytest.mark.gpu


def _unit_lattice(oracle, m, H):
    return oracle.normalize_to_unit(oracle.simplex_lattice(m, H))


def _anisotropic(oracle, v0):
    """adapt_vectors with a 400:1 objective range: the patches of the index become long and thin."""
    m = v0.shape[1]
    zmin = np.linspace(0.0, 0.2, m)
    zmax = zmin + np.geomspace(0.05, 20.0, m)
    return oracle.adapt_vectors(v0, zmin, zmax)


def _sample_rows(v, n, seed):
    """Objective rows that stress the pruned search: random directions, rows exactly on a vector, rows midway
    between two neighbouring vectors (cosines equal up to rounding: the first-strict-maximum rule decides), rows an
    ulp-scale step off a vector, duplicates, the ideal point itself, a NaN row."""
    rng = np.random.default_rng(seed)
    r, m = v.shape
    base = np.linspace(0.3, 0.7, m)
    f = rng.random((n, m)) * np.linspace(1.0, 4.0, m) + 1e-3
    q = n // 8
    j = rng.integers(0, r, size=q)
    f[q:2 * q] = v[j] * rng.uniform(0.5, 3.0, size=(q, 1))                       # on a vector
    j = rng.integers(0, r - 1, size=q)
    f[2 * q:3 * q] = (v[j] + v[j + 1]) * rng.uniform(0.5, 3.0, size=(q, 1))      # between lexicographic neighbours
    j = rng.integers(0, r, size=q)
    f[3 * q:4 * q] = v[j] * (1.0 + 1e-13 * rng.standard_normal((q, m))) * 2.0    # an ulp-scale step off a vector
    j = rng.integers(0, r, size=(q, 3))
    f[4 * q:5 * q] = v[j[:, 0]] + v[j[:, 1]] + v[j[:, 2]]                        # far from every lattice point
    f += base
    f[0] = base                       # the ideal point (nf == 0: vector 0, angle 0)
    f[1] = f[q + 5]                   # an exact duplicate of an on-vector row (APD tie: lowest row wins)
    f[2, 0] = np.nan                  # a NaN row
    f[3] = base + v[0] * 2.0          # the first and the last vector of the set
    f[4] = base + v[r - 1] * 2.0
    return f


def _rows_budget(chk):
    return 8192 if chk.name == "reference" else 4096


@pytest.mark.parametrize("m,H,levels", [(3, 510, 3), (3, 1447, 4)])
@pytest.mark.parametrize("adapted", [False, True])
def test_rv_select_at_baseline_vector_sets(tb, oracle, checkers, m, H, levels, adapted):
    """rv_select against the real R = 130 816 (headline, index depth 3) and R = 1 049 076 (N = 2^20, depth 4)
    sets, isotropic and after an anisotropic adaptation: association, validity, elites bit-exact."""
    chk = checkers[-1]
    v0 = _unit_lattice(oracle, m, H)
    r = v0.shape[0]
    depth, cnt = 0, r
    while True:  # VecIndex::alloc (vecindex.cu): levels of the 32-ary tree
        cnt = (cnt + 31) // 32
        depth += 1
        if cnt <= 32:
            break
    assert depth == levels, (r, depth)
    v = _anisotropic(oracle, v0) if adapted else v0
    gamma = tb.min_vector_angles(v)  # shared input of both sides; checked on its own below
    assert np.all(gamma > 0.0)
    n = _rows_budget(chk) // (2 if levels == 4 else 1)
    f = _sample_rows(v, n, 1000 + H + int(adapted))
    got = tb.rv_select(f, tb.RefVectorSet(v0, v, gamma), 33, 100, 2.0)
    exp = chk.rv_select(f, v, gamma, 33, 100, 2.0)
    _check_selection(got, exp)
    assert got.assoc[3] == 0 and got.assoc[4] == r - 1


@pytest.mark.parametrize("m,H", [(3, 510), (3, 1447), (10, 9)])
@pytest.mark.parametrize("adapted", [False, True])
def test_gamma_at_baseline_vector_sets(tb, oracle, m, H, adapted):
    """min_vector_angles on the full BASELINE sets (the reference's own dense R x R matrix would need 137 GB /
    8.8 TB, refvec.hpp:83): sampled vectors against the oracle's full-j maximum, including the corners of the
    simplex, the first / last positions and a stride that hits every residue of the 32-wide groups."""
    v0 = _unit_lattice(oracle, m, H)
    r = v0.shape[0]
    v = _anisotropic(oracle, v0) if adapted else v0
    gamma = tb.min_vector_angles(v)
    k = 4096 if r < 500000 else 2048
    rng = np.random.default_rng(77 + H)
    rows = np.unique(np.concatenate([[0, 1, 31, 32, 33, 1023, 1024, 1025, r - 2, r - 1],
                                     np.arange(0, r, max(1, r // (k // 2)) | 1)[: k // 2],
                                     rng.integers(0, r, size=k // 2)])).astype(np.uint64)
    exp = oracle.min_vector_angles_rows(v, rows)
    assert ulp_diff(gamma[rows.astype(np.int64)], exp).max() <= 2, (m, H, adapted)
    if not adapted:  # through make_ref_set as well (the entry point the run's initialisation mirrors)
        refs = tb.make_ref_set(m, H)
        assert np.array_equal(refs.v0, v0) and np.array_equal(refs.gamma, gamma)


@pytest.mark.parametrize("adapted", [False, True])
def test_rv_select_at_config4_vector_set(tb, oracle, checkers, adapted):
    """BASELINE config #4's own set: m = 10, H = 9, R = 48 620 (fp32-filtered exact scan, 8 vector chunks)."""
    chk = checkers[-1]
    m, H = 10, 9
    v0 = _unit_lattice(oracle, m, H)
    assert v0.shape[0] == 48620
    v = _anisotropic(oracle, v0) if adapted else v0
    gamma = tb.min_vector_angles(v)
    f = _sample_rows(v, _rows_budget(chk), 4000 + int(adapted))
    _check_selection(tb.rv_select(f, tb.RefVectorSet(v0, v, gamma), 70, 100, 2.0), chk.rv_select(f, v, gamma, 70, 100, 2.0))


def test_lockstep_sweep_floor_shape(tb, ref):
    """Config #5's smallest point (DTLZ2 m = 3, d = 5000, N = 2^14; R = 16 471) against the UNMODIFIED reference:
    two lock-step generations (about 7 s of CPU each): offspring / survivor sets / survivors bit-exact, objectives 1e-12."""
    _lockstep(tb, ref, "dtlz2", 1 << 14, 5000, 3, 2, 42)


def test_lockstep_lsmop1_full_width(tb, oracle):
    """Config #3's decision width (LSMOP1, d = 5000: two-segment bounds inside a run) for one generation.
    LSMOP1 is not in the reference: the checker is the restatement only (parity unpinned)."""
    _lockstep(tb, oracle, "lsmop1", 1 << 12, 5000, 3, 1, 5)
