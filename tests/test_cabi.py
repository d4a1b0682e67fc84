"""CPU: the C-ABI shared library loads and exports every symbol include/temo_b200.h declares,
the ctypes table binds exactly that set, host-only entry points work without a GPU, and the
compute entry points fail loudly (no CPU fallback) when no device is present."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "temo_b200.h")


@pytest.fixture(scope="module")
def lib():
    so = os.path.join(ROOT, "paper_2404_01159_b200", "libtemo_b200.so")
    if not os.path.exists(so):
        subprocess.check_call(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2404_01159_b200", "csrc")])
    from paper_2404_01159_b200 import _lib
    return _lib.load()


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(temo_b200_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_are_exported_and_bound(lib):
    from paper_2404_01159_b200 import _lib
    names = declared_symbols()
    assert len(names) >= 35
    assert sorted(_lib.SIGNATURES) == names
    exported = subprocess.check_output(["nm", "-D", "--defined-only", _lib.LIB_PATH], text=True)
    for n in names:
        assert re.search(rf"\bT {n}\b", exported), f"{n} not exported"
        getattr(lib, n)
    # no torch / C++ types in the ABI: only temo_b200_* are exported from our translation units
    assert not re.search(r"\bT _ZN9temo_b200.*capi", exported)


def test_header_compiles_as_plain_c(tmp_path):
    src = tmp_path / "probe.c"
    src.write_text('#include "temo_b200.h"\nint main(void){temo_b200_run_config c; temo_b200_ga_params g; (void)c; (void)g; return 0;}\n')
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-pedantic", "-I", os.path.join(ROOT, "include"), "-c", str(src), "-o", str(tmp_path / "probe.o")])


def test_struct_layout_matches_header(lib):
    from paper_2404_01159_b200._lib import GaParamsC, RunConfigC
    assert C.sizeof(GaParamsC) == 32
    assert C.sizeof(RunConfigC) == 8 + 6 * 8 + 3 * 8 + 32 + 8 + 6 * 8 + 8
    cfg = RunConfigC()
    lib.temo_b200_default_run_config(C.byref(cfg))
    assert cfg.horizon == 100  # algorithms.hpp:35
    # reference defaults: RunConfig (algorithms.hpp:21-41), GaParams (operators.hpp:22-27)
    assert (cfg.pop, cfg.generations, cfg.seed, cfg.obj, cfg.alpha, cfg.fr) == (105, 100, 42, 3, 2.0, 0.1)
    assert (cfg.ga.pc, cfg.ga.eta, cfg.ga.pm, cfg.ga.xi) == (1.0, 20.0, 1.0, 20.0)
    # op = ga; DeParams / PsoParams / CsoParams defaults (operators.hpp:28-41)
    assert cfg.op == 0
    assert (cfg.opp.de_f, cfg.opp.de_cr, cfg.opp.pso_inertia, cfg.opp.pso_c1, cfg.opp.pso_c2, cfg.opp.cso_phi) == (0.5, 0.9, 0.4, 1.5, 1.5, 0.1)


def test_host_side_entry_points_without_gpu(lib, oracle):
    import paper_2404_01159_b200 as tb
    for m, n in ((3, 105), (3, 131072), (10, 65536), (2, 50)):
        assert tb.lattice_density_for(m, n) == oracle.lattice_density_for(m, n)
    assert np.array_equal(tb.simplex_lattice(3, 13), oracle.simplex_lattice(3, 13))
    assert np.array_equal(tb.simplex_lattice(5, 3), oracle.simplex_lattice(5, 3))
    st = tb.RngStream(42, 0)
    assert np.array_equal(tb.shuffle_indices(st, 20), oracle.shuffle_indices(42, 0, 20)[0]) and st.counter == 19
    st = tb.RngStream(42, 5000)
    assert np.array_equal(tb.parent_pool_indices(77, 105, st), oracle.parent_pool_indices(77, 105, 42, 5000)[0])
    assert tb.apd_penalty(3, 7, 100, 2.0) == oracle.apd_penalty(3, 7, 100, 2.0)
    p = tb.make_problem("lsmop1", 50, 3)
    lo, hi = oracle.problem_bounds("lsmop1", 50, 3)
    assert np.array_equal(p.lower, lo) and np.array_equal(p.upper, hi)
    with pytest.raises(ValueError):
        tb.simplex_lattice(1, 4)


def test_compute_fails_loudly_without_gpu(lib):
    import paper_2404_01159_b200 as tb
    if tb.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(tb.TemoB200Error) as e:
        tb.dtlz_eval(2, np.full((2, 5), 0.5), 3)
    assert e.value.code == 3 and "no CPU fallback" in str(e.value)
    with pytest.raises(tb.TemoB200Error):
        tb.RveaRun(tb.RunConfig(pop=8, dim=5))


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2404_01159_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, fn)).read()
                assert "pyoracle" not in text and "temo_oracle" not in text and "libtemo_ref" not in text, fn
