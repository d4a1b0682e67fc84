"""The libm-exact pow (paper_2404_01159_b200/csrc/glibc_pow.cuh) against the live C library.

CPU (not gpu): the host twin of the device function — same source, same operation sequence —
must reproduce this host's libm pow bit for bit on every domain the generation loop uses, and
the generated constant header must match the installed libm. GPU: the device kernel must do
the same (the oracle / reference call exactly that libm pow)."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT


def libm_pow(x, y):
    libm = ctypes.CDLL("libm.so.6")
    libm.pow.restype = ctypes.c_double
    libm.pow.argtypes = [ctypes.c_double, ctypes.c_double]
    return np.array([libm.pow(float(a), float(b)) for a, b in zip(x, y)])


def domains(n, seed):
    rng = np.random.default_rng(seed)
    m = rng.random(n)
    e21 = 1.0 / 21.0
    xs = [np.where(m <= 0.5, 2.0 * m, 2.0 - 2.0 * m)]          # SBX spreads (operators.hpp:85-86)
    ys = [np.where(m <= 0.5, e21, -e21)]
    dist, u = rng.random(n), rng.random(n)
    p = np.power(dist, 21.0)
    xs += [dist, 2.0 * u + (1.0 - 2.0 * u) * p, dist]            # PM (operators.hpp:115-118), DTLZ4 (problems.hpp:79)
    ys += [np.full(n, 21.0), np.full(n, e21), np.full(n, 100.0)]
    xs += [dist * 1e-3, np.exp((rng.random(n) - 0.5) * 1400.0), rng.random(n) * 2.0**-1022]  # exp tails, subnormal x
    ys += [np.full(n, 21.0), (rng.random(n) - 0.5) * 4.0, (rng.random(n) - 0.5) * 2.0]
    xs += [np.exp((rng.random(n) - 0.5) * 40.0), np.array([1.0, 0.0, 0.5, 2.0, 1.0 - 2**-53, 1.0 + 2**-52, 2**-52, 4.9e-324])]
    ys += [(rng.random(n) - 0.5) * 30.0, np.array([e21, e21, -e21, 21.0, e21, -e21, e21, e21])]
    return np.concatenate(xs), np.concatenate(ys)


def test_generated_constants_match_installed_libm():
    rc = subprocess.call([sys.executable, os.path.join(ROOT, "tools", "gen_glibc_pow_tables.py"), "--check"])
    assert rc == 0, "installed libm carries different pow tables: regenerate glibc_pow_data.h"


def test_host_twin_is_bit_exact_with_libm():
    import paper_2404_01159_b200 as tb
    x, y = domains(40000, 1)
    got = tb.pow_like_host(x, y, on_device=False)
    exp = libm_pow(x, y)
    assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))


@pytest.mark.gpu
def test_device_pow_is_bit_exact_with_libm():
    import paper_2404_01159_b200 as tb
    x, y = domains(200000, 2)
    got = tb.pow_like_host(x, y, on_device=True)
    exp = libm_pow(x, y)
    bad = got.view(np.uint64) != exp.view(np.uint64)
    assert not bad.any(), (x[bad][:5], y[bad][:5], got[bad][:5], exp[bad][:5])
