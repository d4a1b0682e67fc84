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


# ---- tanh (csrc/glibc_tanh.cuh): the toy environment's policy network chains 18 of them per step
def libm_tanh(x):
    libm = ctypes.CDLL("libm.so.6")
    libm.tanh.restype = ctypes.c_double
    libm.tanh.argtypes = [ctypes.c_double]
    return np.array([libm.tanh(float(a)) for a in x])


def tanh_domain(n, seed):
    rng = np.random.default_rng(seed)
    u = rng.uniform(-1.0, 1.0, (5, n))
    special = np.array([0.0, -0.0, 1.0, -1.0, 22.0, -22.0, 21.999999, 0.34657359027997264, 1.0397207708399179, 19.4, 38.9, 1e-300,
                        5e-324, 1e300, np.inf, -np.inf, 0.25, -0.25, 0.125, 2.0**-55, 2.0**-54, 0.5493061443340549])
    return np.concatenate([u[0] * 25.0, u[1], u[2] * 0.35, u[3] * 3.0, np.ldexp(u[4], rng.integers(-60, 20, n)), special])


def test_tanh_host_twin_is_bit_exact_with_libm():
    import paper_2404_01159_b200 as tb
    x = tanh_domain(60000, 3)
    got, exp = tb.tanh_like_host(x, on_device=False), libm_tanh(x)
    assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))


@pytest.mark.gpu
def test_device_tanh_is_bit_exact_with_libm():
    import paper_2404_01159_b200 as tb
    x = tanh_domain(100000, 4)
    got, exp = tb.tanh_like_host(x, on_device=True), libm_tanh(x)
    bad = got.view(np.uint64) != exp.view(np.uint64)
    assert not bad.any(), (x[bad][:5], got[bad][:5], exp[bad][:5])
