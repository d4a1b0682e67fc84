"""pytest configuration: registers the `gpu` marker and provides the CPU checkers.

`-m "not gpu"`: oracle vs golden fixtures / vs the compiled reference, host logic, C-ABI
symbol checks (no compute). `-m gpu`: parity of the CUDA path (called through the C-ABI)
against the oracle, the compiled reference and the golden fixtures.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run with -m gpu on the B200 box)")


@pytest.fixture(scope="session")
def tb():
    """The product package bound to cuda:0 (GPU tests only; there is no CPU fallback)."""
    import paper_2404_01159_b200 as tb
    assert tb.device_count() >= 1, "GPU tests need a CUDA device"
    tb.init(0)
    return tb


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.pyoracle import Ref
    if not Ref.available():
        pytest.skip("oracle/_ref/libtemo_ref.so not built (reference not mounted)")
    return Ref()


@pytest.fixture(scope="session")
def checkers(oracle):
    """Every CPU checker available here: the C restatement, plus the real reference if built."""
    from oracle.pyoracle import Ref
    out = [oracle]
    if Ref.available():
        out.append(Ref())
    return out


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


class Stream:
    """RngStream (rng.hpp:34-52) on top of a checker's value_at; mirrors verify.hpp's generators."""

    def __init__(self, chk, seed, counter=0):
        self.chk, self.seed, self.counter = chk, seed, counter

    def next(self):
        v = self.chk.value_at(self.seed, self.counter)
        self.counter += 1
        return v

    def pick(self, lo, hi):  # verify.hpp:33-35
        return lo + int(self.next() * float(hi - lo + 1))

    def tensor(self, rows, cols):
        out = self.chk.uniform(self.seed, self.counter, rows * cols).reshape(rows, cols)
        self.counter += rows * cols
        return out


def operator_instance(g, n_min, n_max, d_max):
    """verify.hpp:83-103."""
    n = g.pick(n_min, n_max)
    d = g.pick(1, d_max)
    lower, upper = np.empty(d), np.empty(d)
    for j in range(d):
        lower[j] = -1.0 - g.next()
        upper[j] = lower[j] + 0.5 + 2.0 * g.next()
    x = g.tensor(n, d)
    x = lower + x * (upper - lower)
    return n, d, lower, upper, x


def swarm_instance(g, n_min, n_max, d_max):
    """verify.hpp:83-103 including the scores the swarm operators use (drawn after x)."""
    n, d, lower, upper, x = operator_instance(g, n_min, n_max, d_max)
    scores = g.tensor(n, 1).reshape(-1)
    return n, d, lower, upper, x, scores


def ulp_diff(a, b):
    """Distance in units in the last place between two finite fp64 arrays."""
    a = np.ascontiguousarray(a, dtype=np.float64).view(np.int64)
    b = np.ascontiguousarray(b, dtype=np.float64).view(np.int64)
    a = np.where(a < 0, np.int64(-2**63) - a, a)
    b = np.where(b < 0, np.int64(-2**63) - b, b)
    return np.abs(a - b)


def _archive_case(ins, crowd, g, tag):
    """Two successive Archive::insert calls (the second capped) and crowding_distance against the recorded reference."""
    xs, fs = [g[f"{tag}_x{k}"] for k in range(3)], [g[f"{tag}_f{k}"] for k in range(3)]
    cap = int(g[f"{tag}_cap"][0])
    a = ins(None, None, xs[0], fs[0], 0) if fs[0].shape[0] else (None, None)
    a = ins(a[0], a[1], xs[1], fs[1], 0)
    assert np.array_equal(a[0], g[f"{tag}_a1x"]) and np.array_equal(a[1], g[f"{tag}_a1f"]), tag
    assert np.array_equal(crowd(a[1]), g[f"{tag}_crowd"]), tag
    a = ins(a[0], a[1], xs[2], fs[2], cap)
    assert np.array_equal(a[0], g[f"{tag}_a2x"]) and np.array_equal(a[1], g[f"{tag}_a2f"]), tag
    assert a[1].shape[0] <= cap
