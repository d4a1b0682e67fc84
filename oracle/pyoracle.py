"""TEST INFRASTRUCTURE — ctypes front-ends for the two CPU checkers.

``Oracle``  : oracle/libtemo_oracle.so, our plain-C restatement (temo_oracle.c).
``Ref``     : oracle/_ref/libtemo_ref.so, the UNMODIFIED reference headers compiled by
              oracle/Makefile through ref_wrap.cpp (present only if it was built in the
              container that has /root/reference; it travels to the GPU box prebuilt).

Both expose the same numpy-level methods so a parity test can be parametrised over them.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libtemo_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtemo_ref.so")

u64 = C.c_uint64
f64p = C.POINTER(C.c_double)
u64p = C.POINTER(C.c_uint64)
u8p = C.POINTER(C.c_ubyte)

PROBLEM_IDS = {"dtlz1": 1, "dtlz2": 2, "dtlz3": 3, "dtlz4": 4, "lsmop1": 101, "toy2": 201, "toy3": 202}
GA_DEFAULT = (1.0, 20.0, 1.0, 20.0)  # pc, eta, pm, xi — operators.hpp:22-27
OPP_DEFAULT = (0.5, 0.9, 0.4, 1.5, 1.5, 0.1)  # de.f, de.cr, pso.inertia, pso.c1, pso.c2, cso.phi — operators.hpp:28-41


def build(force: bool = False) -> None:
    """Compile the C restatement (always) and the reference shim (when mounted)."""
    if force or not os.path.exists(ORACLE_SO) or (
        os.path.getmtime(ORACLE_SO) < os.path.getmtime(os.path.join(HERE, "temo_oracle.c"))
    ):
        subprocess.check_call(["make", "-s", "-C", HERE, "libtemo_oracle.so"])
    ref_src = os.path.join(HERE, "ref_wrap.cpp")
    if os.path.isdir("/root/reference/proj/include") and (
        force or not os.path.exists(REF_SO) or os.path.getmtime(REF_SO) < os.path.getmtime(ref_src)
    ):
        subprocess.check_call(["make", "-s", "-C", HERE, "_ref/libtemo_ref.so"])


def _f(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a, typ=f64p):
    return None if a is None else a.ctypes.data_as(typ)


@dataclass
class Selection:
    elite: np.ndarray      # merged-row index per valid vector, ascending vector index
    validity: np.ndarray   # uint8[r]
    assoc: np.ndarray | None = None
    theta: np.ndarray | None = None
    apd: np.ndarray | None = None


class _Base:
    name = "base"

    # ---- shared numpy-level helpers -------------------------------------------------
    def take_generation(self, *a, **k):  # pragma: no cover - overridden
        raise NotImplementedError

    def _archive(self, fn_insert, x_old, f_old, x_new, f_new, cap):
        x_new, f_new = _f(x_new), _f(f_new)
        d, m = x_new.shape[1], f_new.shape[1]
        x_old = np.empty((0, d)) if x_old is None else _f(x_old).reshape(-1, d)
        f_old = np.empty((0, m)) if f_old is None else _f(f_old).reshape(-1, m)
        n_old, n_new = f_old.shape[0], f_new.shape[0]
        xo, fo = np.empty((n_old + n_new, d)), np.empty((n_old + n_new, m))
        rows = u64(0)
        rc = fn_insert(_p(x_old) if n_old else None, _p(f_old) if n_old else None, u64(n_old), _p(x_new), _p(f_new), u64(n_new),
                       u64(d), u64(m), u64(cap), _p(xo), _p(fo), C.byref(rows))
        if rc:
            raise RuntimeError(f"archive_insert rc={rc}")
        return xo[: rows.value].copy(), fo[: rows.value].copy()

    def pool_scores(self, f, v, gamma, t, t_max, alpha):
        """apd_scores (selection.hpp:228-234): rv_core's apd column."""
        return self.rv_select(f, v, gamma, t, t_max, alpha).apd

    def generation_op(self, op, problem, n, m, seed, counter, lower, upper, t, t_max, alpha, adapt_every,
                      v0, v, gamma, x, f, swarm=None, ga=GA_DEFAULT, opp=OPP_DEFAULT):
        """algorithms.hpp:246-281 for any operator of :250-271, composed from this checker's own stage functions.
        `swarm` is the SwarmState dict {vel, pb_x, pb_score} (None = empty, created on first use like
        make_swarm_state, operators.hpp:58-60); the updated one is returned under "swarm"."""
        x, f = _f(x), _f(f)
        P = x.shape[0]
        pool_idx, c = self.parent_pool_indices(P, n, seed, counter)
        idx = pool_idx.astype(np.int64)
        pool = x[idx]
        scores = None
        if op in ("pso", "cso"):
            scores = self.pool_scores(f[idx], v, gamma, t, t_max, alpha)
            if swarm is None:
                swarm = dict(vel=np.zeros_like(pool), pb_x=pool.copy(), pb_score=scores.copy())
        if op == "ga":
            off, c = self.ga_reproduce(pool, seed, c, lower, upper, ga)
        elif op == "de":
            off, c = self.de_reproduce(pool, seed, c, lower, upper, opp[0:2])
        elif op == "pso":
            off, c, vel, pbx, pbs = self.pso_reproduce(pool, scores, seed, c, lower, upper, swarm["vel"], swarm["pb_x"],
                                                       swarm["pb_score"], opp[2:5])
            swarm = dict(vel=vel, pb_x=pbx, pb_score=pbs)
        elif op == "cso":
            off, c, vel = self.cso_reproduce(pool, scores, seed, c, lower, upper, swarm["vel"], opp[5:6])
            swarm = dict(swarm, vel=vel)
        elif op == "random":
            off, c = self.random_reproduce(n, pool.shape[1], seed, c, lower, upper)
        else:
            raise ValueError(f"rvea_run: unknown operator '{op}'")
        f_off = self.evaluate(problem, off, m)
        mx, mf = np.vstack([x, off]), np.vstack([f, f_off])
        sel = self.rv_select(mf, v, gamma, t, t_max, alpha)
        e = sel.elite.astype(np.int64)
        nx, nf = mx[e], mf[e]
        v, gamma = _f(v).copy(), _f(gamma).copy()
        if (t + 1) % adapt_every == 0:
            v, gamma = self.adapt(v0, v, gamma, nf.min(axis=0), nf.max(axis=0))
        return dict(x=nx, f=nf, v=v, gamma=gamma, counter=c, offspring=off, f_off=f_off, elite=sel.elite, swarm=swarm,
                    scores=scores)


OPERATOR_IDS = {"ga": 0, "de": 1, "pso": 2, "cso": 3, "random": 4}


class Oracle(_Base):
    """Plain-C restatement (oracle/temo_oracle.c)."""

    name = "oracle"

    def __init__(self):
        build()
        self.lib = C.CDLL(ORACLE_SO)
        L = self.lib
        L.to_value_at.restype = C.c_double
        L.to_value_at.argtypes = [u64, u64]
        L.to_polynomial_delta.restype = C.c_double
        L.to_polynomial_delta.argtypes = [C.c_double] * 5
        L.to_apd_penalty.restype = C.c_double
        L.to_apd_penalty.argtypes = [u64, u64, u64, C.c_double]
        L.to_lattice_count.restype = u64
        L.to_lattice_count.argtypes = [u64, u64]
        L.to_lattice_density_for.restype = u64
        L.to_lattice_density_for.argtypes = [u64, u64]

    # rng
    def value_at(self, seed, k):
        return self.lib.to_value_at(seed, k)

    def uniform(self, seed, counter, count):
        out = np.empty(count)
        self.lib.to_uniform_fill(u64(seed), u64(counter), _p(out), u64(count))
        return out

    def shuffle_indices(self, seed, counter, n):
        out = np.empty(n, dtype=np.uint64)
        c = u64(counter)
        self.lib.to_shuffle_indices(u64(seed), C.byref(c), u64(n), _p(out, u64p))
        return out, c.value

    def parent_pool_indices(self, current, n, seed, counter):
        out = np.empty(n, dtype=np.uint64)
        c = u64(counter)
        self.lib.to_parent_pool_indices(u64(current), u64(n), u64(seed), C.byref(c), _p(out, u64p))
        return out, c.value

    # operators
    def _op(self, fn, x, seed, counter, ga, lower, upper):
        x = _f(x)
        n, d = x.shape
        out = np.empty_like(x)
        c = u64(counter)
        g = _f(ga)
        rc = fn(_p(x), u64(n), u64(d), u64(seed), C.byref(c), _p(g), _p(_f(lower)), _p(_f(upper)), _p(out))
        if rc not in (0, None):
            raise RuntimeError(f"oracle operator failed rc={rc}")
        return out, c.value

    def sbx(self, x, seed, counter, lower, upper, ga=GA_DEFAULT):
        self.lib.to_sbx.restype = None
        return self._op(self.lib.to_sbx, x, seed, counter, ga, lower, upper)

    def polynomial_mutation(self, x, seed, counter, lower, upper, ga=GA_DEFAULT):
        self.lib.to_polynomial_mutation.restype = None
        return self._op(self.lib.to_polynomial_mutation, x, seed, counter, ga, lower, upper)

    def ga_reproduce(self, x, seed, counter, lower, upper, ga=GA_DEFAULT):
        self.lib.to_ga_reproduce.restype = C.c_int
        return self._op(self.lib.to_ga_reproduce, x, seed, counter, ga, lower, upper)

    # ---- DE / PSO / CSO (operators.hpp:166-284); states are copied in and returned
    def de_reproduce(self, x, seed, counter, lower, upper, p=(0.5, 0.9)):
        x = _f(x)
        n, d = x.shape
        out, c = np.empty_like(x), u64(counter)
        rc = self.lib.to_de_reproduce(_p(x), u64(n), u64(d), u64(seed), C.byref(c), _p(_f(p)), _p(_f(lower)), _p(_f(upper)), _p(out))
        if rc:
            raise ValueError("de_reproduce: needs at least four rows")
        return out, c.value

    def pso_reproduce(self, x, scores, seed, counter, lower, upper, vel, pb_x, pb_score, p=(0.4, 1.5, 1.5)):
        x = _f(x)
        n, d = x.shape
        vel, pb_x, pb_score = _f(vel).copy(), _f(pb_x).copy(), _f(pb_score).reshape(-1).copy()
        out, c = np.empty_like(x), u64(counter)
        self.lib.to_pso_reproduce(_p(x), _p(_f(scores)), u64(n), u64(d), u64(seed), C.byref(c), _p(_f(p)), _p(vel), _p(pb_x),
                                  _p(pb_score), _p(_f(lower)), _p(_f(upper)), _p(out))
        return out, c.value, vel, pb_x, pb_score

    def cso_reproduce(self, x, scores, seed, counter, lower, upper, vel, p=(0.1,)):
        x = _f(x)
        n, d = x.shape
        vel = _f(vel).copy()
        out, c = np.empty_like(x), u64(counter)
        rc = self.lib.to_cso_reproduce(_p(x), _p(_f(scores)), u64(n), u64(d), u64(seed), C.byref(c), _p(_f(p)), _p(vel),
                                       _p(_f(lower)), _p(_f(upper)), _p(out))
        if rc:
            raise MemoryError("cso_reproduce")
        return out, c.value, vel

    def random_reproduce(self, n, d, seed, counter, lower, upper):
        out = np.empty((n, d))
        c = u64(counter)
        self.lib.to_random_reproduce(u64(n), u64(d), u64(seed), C.byref(c), _p(_f(lower)), _p(_f(upper)), _p(out))
        return out, c.value

    def polynomial_delta(self, u, x, lo, hi, xi):
        return self.lib.to_polynomial_delta(u, x, lo, hi, xi)

    # problems
    def evaluate(self, problem, x, m):
        x = _f(x)
        n, d = x.shape
        f = np.empty((n, m))
        pid = PROBLEM_IDS[problem]
        if pid == 101:
            rc = self.lib.to_lsmop1_eval(_p(x), u64(n), u64(d), u64(m), _p(f))
        elif pid in (201, 202):
            rc = self.lib.to_toy_eval(C.c_int(pid), _p(x), u64(n), u64(d), u64(m), u64(100), _p(f))
        else:
            rc = self.lib.to_dtlz_eval(C.c_int(pid), _p(x), u64(n), u64(d), u64(m), _p(f))
        if rc:
            raise ValueError(f"evaluate({problem}) rejected its arguments rc={rc}")
        return f

    def problem_bounds(self, problem, d, m):
        lo, hi = np.empty(d), np.empty(d)
        self.lib.to_problem_bounds(C.c_int(PROBLEM_IDS[problem]), u64(d), u64(m), _p(lo), _p(hi))
        return lo, hi

    def env_rollout(self, params, horizon=100, num_obj=2, hidden=16):
        """env_rollout (problems.hpp:211-241): returns in maximisation orientation."""
        params = _f(params)
        f = np.empty((params.shape[0], num_obj))
        if self.lib.to_env_rollout(_p(params), u64(params.shape[0]), u64(params.shape[1]), u64(hidden), u64(horizon), u64(num_obj), _p(f)):
            raise ValueError("env_rollout: parameter length mismatch")
        return f

    def mlp_forward(self, params, obs, hidden=16):
        params, obs = _f(params), _f(obs)
        act = np.empty((params.shape[0], 2))
        for i in range(params.shape[0]):
            self.lib.to_mlp_forward(_p(params[i]), u64(hidden), _p(obs[i]), _p(act[i : i + 1]))
        return act

    # refvec
    def lattice_count(self, m, H):
        return self.lib.to_lattice_count(m, H)

    def lattice_density_for(self, m, target):
        return self.lib.to_lattice_density_for(m, target)

    def simplex_lattice(self, m, H):
        out = np.empty((self.lattice_count(m, H), m))
        self.lib.to_simplex_lattice(u64(m), u64(H), _p(out))
        return out

    def normalize_to_unit(self, v):
        v = _f(v)
        out = np.empty_like(v)
        if self.lib.to_normalize_to_unit(_p(v), u64(v.shape[0]), u64(v.shape[1]), _p(out)):
            raise ValueError("normalize_to_unit: zero row")
        return out

    def min_vector_angles(self, v):
        v = _f(v)
        g = np.empty(v.shape[0])
        rc = self.lib.to_min_vector_angles(_p(v), u64(v.shape[0]), u64(v.shape[1]), _p(g))
        if rc:
            raise ValueError(f"min_vector_angles rc={rc}")
        return g

    def min_vector_angles_rows(self, v, rows, want_cos=False):
        """gamma of the vectors `rows` against the full set (refvec.hpp:81-100 per sampled vector)."""
        v = _f(v)
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        g, c = np.empty(rows.size), np.empty(rows.size)
        rc = self.lib.to_min_vector_angles_rows(_p(v), u64(v.shape[0]), u64(v.shape[1]), _p(rows, u64p), u64(rows.size), _p(g), _p(c))
        if rc:
            raise ValueError(f"min_vector_angles_rows rc={rc}")
        return (g, c) if want_cos else g

    def adapt_vectors(self, v0, zmin, zmax):
        """adapt_vectors (refvec.hpp:119-131) without the gamma recomputation."""
        v0 = _f(v0)
        v = v0.copy()
        rc = self.lib.to_adapt_vectors(_p(v0), _p(v), u64(v0.shape[0]), u64(v0.shape[1]), _p(_f(zmin)), _p(_f(zmax)))
        if rc < 0:
            raise ValueError(f"adapt_vectors rc={rc}")
        return v

    def make_ref_set(self, m, H):
        r = self.lattice_count(m, H)
        v0, g = np.empty((r, m)), np.empty(r)
        rc = self.lib.to_make_ref_set(u64(m), u64(H), _p(v0), _p(g))
        if rc:
            raise ValueError(f"make_ref_set rc={rc}")
        return v0, g

    def adapt(self, v0, v, gamma, zmin, zmax):
        v0 = _f(v0)
        v, gamma = _f(v).copy(), _f(gamma).copy()
        rc = self.lib.to_adapt(_p(v0), _p(v), _p(gamma), u64(v0.shape[0]), u64(v0.shape[1]), _p(_f(zmin)), _p(_f(zmax)))
        if rc:
            raise ValueError(f"adapt rc={rc}")
        return v, gamma

    # selection
    def apd_penalty(self, m, t, t_max, alpha):
        return self.lib.to_apd_penalty(m, t, t_max, alpha)

    def rv_select(self, f, v, gamma, t, t_max, alpha=2.0):
        f, v, gamma = _f(f), _f(v), _f(gamma)
        n, m = f.shape
        r = v.shape[0]
        elite = np.empty(max(r, 1), dtype=np.uint64)
        valid = np.empty(r, dtype=np.uint8)
        assoc = np.empty(n, dtype=np.uint64)
        theta, apd = np.empty(n), np.empty(n)
        ne = u64(0)
        rc = self.lib.to_rv_select(_p(f), u64(n), u64(m), _p(v), _p(gamma), u64(r), u64(t), u64(t_max),
                                   C.c_double(alpha), _p(elite, u64p), C.byref(ne), _p(valid, u8p),
                                   _p(assoc, u64p), _p(theta), _p(apd))
        if rc:
            raise ValueError(f"rv_select contract violation rc={rc}")
        return Selection(elite[: ne.value].copy(), valid, assoc, theta, apd)

    def archive_insert(self, x_old, f_old, x_new, f_new, cap=0):
        """Archive::insert (algorithms.hpp:72-144) -> (x, f) of the updated archive."""
        return self._archive(self.lib.to_archive_insert, x_old, f_old, x_new, f_new, cap)

    def crowding_distance(self, front):
        front = _f(front)
        out = np.empty(front.shape[0])
        if self.lib.to_crowding_distance(_p(front), u64(front.shape[0]), u64(front.shape[1]), _p(out)):
            raise ValueError("crowding_distance: empty front")
        return out

    # ---- NSGA-II baseline (selection.hpp:251-346, algorithms.hpp:301-369)
    def nondominated_sort(self, f):
        f = _f(f)
        rank = np.zeros(f.shape[0], dtype=np.uint64)
        if self.lib.to_nondominated_sort(_p(f), u64(f.shape[0]), u64(f.shape[1]), _p(rank, u64p)):
            raise MemoryError("nondominated_sort")
        return rank

    def nsga2_select(self, f, target):
        f = _f(f)
        sel = np.zeros(target, dtype=np.uint64)
        if self.lib.to_nsga2_select(_p(f), u64(f.shape[0]), u64(f.shape[1]), u64(target), _p(sel, u64p)):
            raise ValueError("nsga2_select: target exceeds population")
        return sel

    def nsga2_generation(self, problem, m, seed, counter, lower, upper, x, f, ga=GA_DEFAULT):
        """One generation of nsga2_run on explicit state -> dict(x, f, counter, offspring, f_off, sel, pool_idx)."""
        x, f = _f(x).copy(), _f(f).copy()
        n, d = x.shape
        off, f_off = np.empty((n, d)), np.empty((n, m))
        sel, pool_idx = np.zeros(n, dtype=np.uint64), np.zeros(n, dtype=np.uint64)
        c = u64(counter)
        rc = self.lib.to_nsga2_generation(C.c_int(PROBLEM_IDS[problem]), u64(n), u64(d), u64(m), u64(seed), C.byref(c), _p(_f(ga)),
                                          _p(_f(lower)), _p(_f(upper)), _p(x), _p(f), _p(off), _p(f_off), _p(sel, u64p),
                                          _p(pool_idx, u64p))
        if rc:
            raise RuntimeError(f"nsga2_generation rc={rc}")
        return dict(x=x, f=f, counter=c.value, offspring=off, f_off=f_off, sel=sel, pool_idx=pool_idx)

    def nsga2_run(self, problem, n, d, m, generations, seed=42, ga=GA_DEFAULT):
        x, f = np.empty((n, d)), np.empty((n, m))
        c = u64(0)
        rc = self.lib.to_nsga2_run(C.c_int(PROBLEM_IDS[problem]), u64(n), u64(d), u64(m), u64(generations), u64(seed), _p(_f(ga)),
                                   _p(x), _p(f), C.byref(c))
        if rc:
            raise RuntimeError(f"nsga2_run rc={rc}")
        return dict(x=x, f=f, counter=c.value)

    # ---- metrics.hpp
    def igd(self, f, pf):
        f, pf = _f(f), _f(pf)
        out = C.c_double(0)
        if self.lib.to_igd(_p(f), u64(f.shape[0]), u64(f.shape[1]), _p(pf), u64(pf.shape[0]), C.byref(out)):
            raise ValueError("igd: empty set")
        return out.value

    def hv_mc_box(self, f, lo, ref, samples, seed):
        """(value, std_error); lo=None -> hv_mc (box from col_min(f))."""
        f, ref = _f(f), _f(ref)
        out = np.zeros(2)
        if lo is None:
            rc = self.lib.to_hv_mc(_p(f), u64(f.shape[0]), u64(f.shape[1]), _p(ref), u64(samples), u64(seed), _p(out))
        else:
            rc = self.lib.to_hv_mc_box(_p(f), u64(f.shape[0]), u64(f.shape[1]), _p(_f(lo)), _p(ref), u64(samples), u64(seed), _p(out))
        if rc:
            raise ValueError("hv_mc: bad arguments")
        return out[0], out[1]

    # algorithms
    def generation(self, problem, n, m, seed, counter, lower, upper, t, t_max, alpha, adapt_every,
                   v0, v, gamma, x, f, ga=GA_DEFAULT):
        """One generation on explicit state. Returns dict with new x, f, v, gamma, counter,
        offspring, f_off, elite (merged indices)."""
        x, f = _f(x), _f(f)
        P, d = x.shape
        v0, v, gamma = _f(v0), _f(v).copy(), _f(gamma).copy()
        r = v0.shape[0]
        cap = max(P, r, n)
        xb = np.zeros((cap, d)); xb[:P] = x
        fb = np.zeros((cap, m)); fb[:P] = f
        rows = u64(P)
        c = u64(counter)
        off, f_off = np.empty((n, d)), np.empty((n, m))
        elite = np.empty(max(r, P + n), dtype=np.uint64)
        ne = u64(0)
        g = _f(ga)
        rc = self.lib.to_generation(C.c_int(PROBLEM_IDS[problem]), u64(n), u64(d), u64(m), u64(seed), C.byref(c),
                                    _p(g), _p(_f(lower)), _p(_f(upper)), u64(t), u64(t_max), C.c_double(alpha),
                                    u64(adapt_every), _p(v0), _p(v), _p(gamma), u64(r), _p(xb), _p(fb),
                                    C.byref(rows), _p(off), _p(f_off), _p(elite, u64p), C.byref(ne))
        if rc:
            raise RuntimeError(f"generation rc={rc}")
        k = rows.value
        return dict(x=xb[:k].copy(), f=fb[:k].copy(), v=v, gamma=gamma, counter=c.value,
                    offspring=off, f_off=f_off, elite=elite[: ne.value].copy())

    def rvea_run(self, problem, n, d, m, generations, seed=42, lattice_h=0, alpha=2.0, fr=0.1, ga=GA_DEFAULT):
        H = lattice_h or self.lattice_density_for(m, n)
        r = self.lattice_count(m, H)
        cap = max(n, r)
        x, f = np.empty((cap, d)), np.empty((cap, m))
        rows = u64(0)
        pops = np.zeros(generations, dtype=np.uint64)
        v, gamma = np.empty((r, m)), np.empty(r)
        c = u64(0)
        g = _f(ga)
        rc = self.lib.to_rvea_run(C.c_int(PROBLEM_IDS[problem]), u64(n), u64(d), u64(m), u64(lattice_h),
                                  u64(generations), C.c_double(alpha), C.c_double(fr), u64(seed), _p(g),
                                  _p(x), _p(f), C.byref(rows), _p(pops, u64p), _p(v), _p(gamma), C.byref(c))
        if rc:
            raise RuntimeError(f"rvea_run rc={rc}")
        k = rows.value
        return dict(x=x[:k].copy(), f=f[:k].copy(), pop_size=pops, v=v, gamma=gamma, counter=c.value)

    def rvea_run_op(self, op, problem, n, d, m, generations, seed=42, lattice_h=0, alpha=2.0, fr=0.1, ga=GA_DEFAULT,
                    opp=OPP_DEFAULT):
        H = lattice_h or self.lattice_density_for(m, n)
        r = self.lattice_count(m, H)
        cap = max(n, r)
        x, f = np.empty((cap, d)), np.empty((cap, m))
        rows, c = u64(0), u64(0)
        pops = np.zeros(generations, dtype=np.uint64)
        rc = self.lib.to_rvea_run_op(C.c_int(PROBLEM_IDS[problem]), C.c_int(OPERATOR_IDS[op]), _p(_f(opp)), u64(n), u64(d), u64(m),
                                     u64(lattice_h), u64(generations), C.c_double(alpha), C.c_double(fr), u64(seed), _p(_f(ga)),
                                     _p(x), _p(f), C.byref(rows), _p(pops, u64p), C.byref(c))
        if rc:
            raise RuntimeError(f"rvea_run_op rc={rc}")
        k = rows.value
        return dict(x=x[:k].copy(), f=f[:k].copy(), pop_size=pops, counter=c.value)


class Ref(_Base):
    """The unmodified reference (oracle/_ref/libtemo_ref.so)."""

    name = "reference"

    @staticmethod
    def available() -> bool:
        try:
            build()
        except Exception:
            pass
        return os.path.exists(REF_SO)

    def __init__(self):
        if not Ref.available():
            raise FileNotFoundError(REF_SO)
        self.lib = C.CDLL(REF_SO)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_value_at.restype = C.c_double
        L.ref_value_at.argtypes = [u64, u64]
        L.ref_polynomial_delta.restype = C.c_double
        L.ref_polynomial_delta.argtypes = [C.c_double] * 5
        L.ref_apd_penalty.restype = C.c_double
        L.ref_apd_penalty.argtypes = [u64, u64, u64, C.c_double]
        for fn in (L.ref_lattice_count, L.ref_lattice_density_for):
            fn.restype = u64
            fn.argtypes = [u64, u64]
        L.ref_num_threads.restype = u64

    def _chk(self, rc):
        if rc:
            msg = self.lib.ref_last_error().decode()
            if rc == -2:
                raise MemoryError(msg)
            raise ValueError(msg)

    def num_threads(self):
        return int(self.lib.ref_num_threads())

    def set_num_threads(self, n):
        self.lib.ref_set_num_threads(u64(n))

    def value_at(self, seed, k):
        return self.lib.ref_value_at(seed, k)

    def uniform(self, seed, counter, count):
        out = np.empty(count)
        self._chk(self.lib.ref_uniform_fill(u64(seed), u64(counter), _p(out), u64(count), u64(1)))
        return out

    def shuffle_indices(self, seed, counter, n):
        out = np.empty(n, dtype=np.uint64)
        c = u64(counter)
        self._chk(self.lib.ref_shuffle_indices(u64(seed), C.byref(c), u64(n), _p(out, u64p)))
        return out, c.value

    def parent_pool_indices(self, current, n, seed, counter):
        out = np.empty(n, dtype=np.uint64)
        c = u64(counter)
        self._chk(self.lib.ref_parent_pool_indices(u64(current), u64(n), u64(seed), C.byref(c), _p(out, u64p)))
        return out, c.value

    def _op(self, which, x, seed, counter, ga, lower, upper):
        x = _f(x)
        n, d = x.shape
        out = np.empty_like(x)
        c = u64(counter)
        g = _f(ga)
        self._chk(self.lib.ref_operator(C.c_int(which), _p(x), u64(n), u64(d), u64(seed), C.byref(c), _p(g),
                                        _p(_f(lower)), _p(_f(upper)), _p(out)))
        return out, c.value

    def sbx(self, x, seed, counter, lower, upper, ga=GA_DEFAULT, scalar=False):
        return self._op(3 if scalar else 0, x, seed, counter, ga, lower, upper)

    def polynomial_mutation(self, x, seed, counter, lower, upper, ga=GA_DEFAULT, scalar=False):
        return self._op(4 if scalar else 1, x, seed, counter, ga, lower, upper)

    def ga_reproduce(self, x, seed, counter, lower, upper, ga=GA_DEFAULT, scalar=False):
        return self._op(5 if scalar else 2, x, seed, counter, ga, lower, upper)

    def de_reproduce(self, x, seed, counter, lower, upper, p=(0.5, 0.9), scalar=False):
        x = _f(x)
        n, d = x.shape
        out, c = np.empty_like(x), u64(counter)
        self._chk(self.lib.ref_de_reproduce(C.c_int(int(scalar)), _p(x), u64(n), u64(d), u64(seed), C.byref(c), _p(_f(p)),
                                            _p(_f(lower)), _p(_f(upper)), _p(out)))
        return out, c.value

    def pso_reproduce(self, x, scores, seed, counter, lower, upper, vel, pb_x, pb_score, p=(0.4, 1.5, 1.5), scalar=False):
        x = _f(x)
        n, d = x.shape
        vel, pb_x, pb_score = _f(vel).copy(), _f(pb_x).copy(), _f(pb_score).reshape(-1).copy()
        out, c = np.empty_like(x), u64(counter)
        self._chk(self.lib.ref_pso_reproduce(C.c_int(int(scalar)), _p(x), _p(_f(scores)), u64(n), u64(d), u64(seed), C.byref(c),
                                             _p(_f(p)), _p(vel), _p(pb_x), _p(pb_score), _p(_f(lower)), _p(_f(upper)), _p(out)))
        return out, c.value, vel, pb_x, pb_score

    def cso_reproduce(self, x, scores, seed, counter, lower, upper, vel, p=(0.1,), scalar=False):
        x = _f(x)
        n, d = x.shape
        vel = _f(vel).copy()
        out, c = np.empty_like(x), u64(counter)
        self._chk(self.lib.ref_cso_reproduce(C.c_int(int(scalar)), _p(x), _p(_f(scores)), u64(n), u64(d), u64(seed), C.byref(c),
                                             _p(_f(p)), _p(vel), _p(_f(lower)), _p(_f(upper)), _p(out)))
        return out, c.value, vel

    def apd_scores(self, f, v, gamma, t, t_max, alpha=2.0):
        f, v = _f(f), _f(v)
        out = np.empty(f.shape[0])
        self._chk(self.lib.ref_apd_scores(_p(f), u64(f.shape[0]), u64(f.shape[1]), _p(v), _p(_f(gamma)), u64(v.shape[0]), u64(t),
                                          u64(t_max), C.c_double(alpha), _p(out)))
        return out

    def random_reproduce(self, n, d, seed, counter, lower, upper):
        out = np.empty((n, d))
        c = u64(counter)
        self._chk(self.lib.ref_random_reproduce(u64(n), u64(d), u64(seed), C.byref(c), _p(_f(lower)), _p(_f(upper)), _p(out)))
        return out, c.value

    def polynomial_delta(self, u, x, lo, hi, xi):
        return self.lib.ref_polynomial_delta(u, x, lo, hi, xi)

    def evaluate(self, problem, x, m, horizon=100):
        pid = PROBLEM_IDS[problem]
        if pid == 101:
            raise NotImplementedError("the reference has no LSMOP1")
        x = _f(x)
        n, d = x.shape
        f = np.empty((n, m))
        if pid > 4:  # toy2 / toy3 through make_problem(...).evaluate (the negated returns)
            self._chk(self.lib.ref_problem_evaluate(problem.encode(), u64(d), u64(m), u64(horizon), _p(x), u64(n), _p(f), None, None,
                                                    None, None))
            return f
        self._chk(self.lib.ref_dtlz_eval(C.c_int(pid), _p(x), u64(n), u64(d), u64(m), _p(f)))
        return f

    def problem_bounds(self, problem, d, m):
        if problem in ("toy2", "toy3"):
            return -np.ones(d), np.ones(d)  # problems.hpp:285-286
        return np.zeros(d), np.ones(d)  # problems.hpp:271-272

    def env_rollout(self, params, horizon=100, num_obj=2, hidden=16):
        """The reference's env_rollout (problems.hpp:211-241): returns in maximisation orientation."""
        params = _f(params)
        f = np.empty((params.shape[0], num_obj))
        self._chk(self.lib.ref_env_rollout(_p(params), u64(params.shape[0]), u64(hidden), u64(horizon), u64(num_obj), _p(f)))
        return f

    def mlp_forward(self, params, obs, hidden=16):
        params, obs = _f(params), _f(obs)
        act = np.empty((params.shape[0], 2))
        for i in range(params.shape[0]):
            self._chk(self.lib.ref_mlp_forward(_p(params[i]), u64(hidden), _p(obs[i]), _p(act[i : i + 1])))
        return act

    def dtlz_pf_reference(self, pid, m, H):
        out = np.empty((self.lattice_count(m, H), m))
        self._chk(self.lib.ref_dtlz_pf_reference(C.c_int(pid), u64(m), u64(H), _p(out)))
        return out

    def lattice_count(self, m, H):
        return self.lib.ref_lattice_count(m, H)

    def lattice_density_for(self, m, target):
        return self.lib.ref_lattice_density_for(m, target)

    def simplex_lattice(self, m, H):
        out = np.empty((self.lattice_count(m, H), m))
        self._chk(self.lib.ref_simplex_lattice(u64(m), u64(H), _p(out)))
        return out

    def normalize_to_unit(self, v):
        v = _f(v)
        out = np.empty_like(v)
        self._chk(self.lib.ref_normalize_to_unit(_p(v), u64(v.shape[0]), u64(v.shape[1]), _p(out)))
        return out

    def min_vector_angles(self, v):
        v = _f(v)
        g = np.empty(v.shape[0])
        self._chk(self.lib.ref_min_vector_angles(_p(v), u64(v.shape[0]), u64(v.shape[1]), _p(g)))
        return g

    def make_ref_set(self, m, H):
        r = self.lattice_count(m, H)
        v0, g = np.empty((r, m)), np.empty(r)
        self._chk(self.lib.ref_make_ref_set(u64(m), u64(H), _p(v0), _p(g)))
        return v0, g

    def adapt(self, v0, v, gamma, zmin, zmax):
        v0 = _f(v0)
        v, gamma = _f(v).copy(), _f(gamma).copy()
        self._chk(self.lib.ref_adapt(_p(v0), _p(v), _p(gamma), u64(v0.shape[0]), u64(v0.shape[1]), _p(_f(zmin)), _p(_f(zmax))))
        return v, gamma

    def apd_penalty(self, m, t, t_max, alpha):
        return self.lib.ref_apd_penalty(m, t, t_max, alpha)

    def rv_select(self, f, v, gamma, t, t_max, alpha=2.0, set_form=False, want_core=True):
        """want_core=False: rv_select alone, as rvea_run calls it (the per-row diagnostics cost a second rv_core pass)."""
        f, v, gamma = _f(f), _f(v), _f(gamma)
        n, m = f.shape
        r = v.shape[0]
        elite = np.empty(max(r, 1), dtype=np.uint64)
        valid = np.empty(r, dtype=np.uint8)
        assoc = np.empty(n, dtype=np.uint64)
        theta, apd = np.empty(n), np.empty(n)
        ne = u64(0)
        if not want_core and not set_form:
            self._chk(self.lib.ref_rv_select(C.c_int(0), _p(f), u64(n), u64(m), _p(v), _p(gamma), u64(r), u64(t), u64(t_max),
                                             C.c_double(alpha), _p(elite, u64p), C.byref(ne), _p(valid, u8p), None, None, None, None))
            return Selection(elite[: ne.value].copy(), valid)
        self._chk(self.lib.ref_rv_select(C.c_int(1 if set_form else 0), _p(f), u64(n), u64(m), _p(v), _p(gamma),
                                         u64(r), u64(t), u64(t_max), C.c_double(alpha), _p(elite, u64p),
                                         C.byref(ne), _p(valid, u8p), _p(assoc, u64p), _p(theta), _p(apd), None))
        if set_form:
            return Selection(elite[: ne.value].copy(), valid)
        return Selection(elite[: ne.value].copy(), valid, assoc, theta, apd)

    def igd(self, f, pf):
        f, pf = _f(f), _f(pf)
        out = C.c_double(0)
        self._chk(self.lib.ref_igd(_p(f), u64(f.shape[0]), u64(f.shape[1]), _p(pf), u64(pf.shape[0]), C.byref(out)))
        return out.value

    def archive_insert(self, x_old, f_old, x_new, f_new, cap=0):
        """The reference's Archive::insert (algorithms.hpp:72-144) -> (x, f) of the updated archive."""
        return self._archive(self.lib.ref_archive_insert, x_old, f_old, x_new, f_new, cap)

    def crowding_distance(self, front):
        front = _f(front)
        out = np.empty(front.shape[0])
        self._chk(self.lib.ref_crowding_distance(_p(front), u64(front.shape[0]), u64(front.shape[1]), _p(out)))
        return out

    def nondominated_sort(self, f):
        f = _f(f)
        rank = np.zeros(f.shape[0], dtype=np.uint64)
        self._chk(self.lib.ref_nondominated_sort(_p(f), u64(f.shape[0]), u64(f.shape[1]), _p(rank, u64p)))
        return rank

    def nsga2_select(self, f, target):
        f = _f(f)
        sel = np.zeros(target, dtype=np.uint64)
        self._chk(self.lib.ref_nsga2_select(_p(f), u64(f.shape[0]), u64(f.shape[1]), u64(target), _p(sel, u64p)))
        return sel

    def nsga2_run(self, problem, n, d, m, generations, seed=42, ga=GA_DEFAULT):
        """The reference's nsga2_run (algorithms.hpp:301-369), track_archive = false."""
        x, f = np.empty((n, d)), np.empty((n, m))
        cfg_u = np.array([n, generations, seed, d, m], dtype=np.uint64)
        self._chk(self.lib.ref_nsga2_run(problem.encode(), _p(cfg_u, u64p), _p(_f(ga)), _p(x), _p(f)))
        return dict(x=x, f=f)

    def hv_mc_box(self, f, lo, ref, samples, seed):
        """(value, std_error) of hv_mc_box; lo=None -> hv_mc (metrics.hpp:76-124)."""
        f = _f(f)
        out = np.zeros(2)
        self._chk(self.lib.ref_hv_mc_box(_p(f), u64(f.shape[0]), u64(f.shape[1]), None if lo is None else _p(_f(lo)), _p(_f(ref)),
                                         u64(samples), u64(seed), _p(out)))
        return out[0], out[1]

    def rvea_run_metrics(self, problem, n, d, m, generations, pf_ref=None, hv_ref=None, seed=42, lattice_h=0, alpha=2.0, fr=0.1,
                         op="ga", hv_scale=1.0, hv_samples=2048, hv_seed=9001, maximization=False):
        """The reference's rvea_run with a MetricContext: per-generation pop_size, igd, hv of the population."""
        cfg_u = np.array([n, lattice_h, generations, seed, d, m], dtype=np.uint64)
        cfg_d = np.array([alpha, fr, 0.0])
        mcp = np.array([hv_scale, float(hv_samples), float(hv_seed), 1.0 if maximization else 0.0])
        pops = np.zeros(generations, dtype=np.uint64)
        g, h = np.full(generations, np.nan), np.full(generations, np.nan)
        pf = None if pf_ref is None else _f(pf_ref)
        self._chk(self.lib.ref_rvea_run_metrics(problem.encode(), op.encode(), _p(cfg_u, u64p), _p(cfg_d), None if pf is None else _p(pf),
                                                u64(0 if pf is None else pf.shape[0]), None if hv_ref is None else _p(_f(hv_ref)),
                                                _p(mcp), _p(pops, u64p), _p(g), _p(h)))
        return dict(pop_size=pops, igd=g, hv=h)

    def rvea_run_archive(self, problem, n, d, m, generations, pf_ref=None, seed=42, lattice_h=0, alpha=2.0, fr=0.1, archive_cap=0,
                         scalar=False, arch_capacity=0):
        """The reference's rvea_run (or oracle_rvea_run) with track_archive = true: per-generation survivor counts, archive
        sizes and archive IGD, and the final archive."""
        cfg_u = np.array([n, lattice_h, generations, seed, d, m], dtype=np.uint64)
        cfg_d = np.array([alpha, fr, 0.0])
        pops, sizes = np.zeros(generations, dtype=np.uint64), np.zeros(generations, dtype=np.uint64)
        g = np.full(generations, np.nan)
        pf = None if pf_ref is None else _f(pf_ref)
        cap = arch_capacity or 64 * max(n, 128)
        ax, af = np.empty((cap, d)), np.empty((cap, m))
        rows = u64(0)
        self._chk(self.lib.ref_rvea_run_archive(C.c_int(1 if scalar else 0), problem.encode(), _p(cfg_u, u64p), _p(cfg_d), u64(archive_cap),
                                                None if pf is None else _p(pf), u64(0 if pf is None else pf.shape[0]),
                                                _p(pops, u64p), _p(sizes, u64p), _p(g), _p(ax), _p(af), u64(cap), C.byref(rows)))
        return dict(pop_size=pops, archive_size=sizes, igd=g, archive_x=ax[: rows.value].copy(), archive_f=af[: rows.value].copy())

    def generation(self, problem, n, m, seed, counter, lower, upper, t, t_max, alpha, adapt_every,
                   v0, v, gamma, x, f, ga=GA_DEFAULT):
        """algorithms.hpp:246-281 composed from the reference's own stage functions."""
        x, f = _f(x), _f(f)
        P = x.shape[0]
        pool_idx, c = self.parent_pool_indices(P, n, seed, counter)
        pool = x[pool_idx.astype(np.int64)]
        off, c = self.ga_reproduce(pool, seed, c, lower, upper, ga)
        f_off = self.evaluate(problem, off, m)
        mx, mf = np.vstack([x, off]), np.vstack([f, f_off])
        sel = self.rv_select(mf, v, gamma, t, t_max, alpha)
        e = sel.elite.astype(np.int64)
        nx, nf = mx[e], mf[e]
        v, gamma = _f(v).copy(), _f(gamma).copy()
        if (t + 1) % adapt_every == 0:
            v, gamma = self.adapt(v0, v, gamma, nf.min(axis=0), nf.max(axis=0))
        return dict(x=nx, f=nf, v=v, gamma=gamma, counter=c, offspring=off, f_off=f_off, elite=sel.elite)

    def rvea_run(self, problem, n, d, m, generations, seed=42, lattice_h=0, alpha=2.0, fr=0.1, ga=GA_DEFAULT,
                 scalar=False, time_budget_s=0.0, igd_H=0, want_x=True):
        H = lattice_h or self.lattice_density_for(m, n)
        r = self.lattice_count(m, H)
        cap = max(n, r)
        x = np.empty((cap, d)) if want_x else None
        f = np.empty((cap, m))
        cfg_u = np.array([n, lattice_h, generations, seed, d, m], dtype=np.uint64)
        cfg_d = np.array([alpha, fr, time_budget_s])
        rows, done = u64(0), u64(0)
        pops = np.zeros(generations, dtype=np.uint64)
        ms = np.zeros(generations)
        igd = np.full(generations, np.nan)
        g = _f(ga)
        self._chk(self.lib.ref_rvea_run(C.c_int(1 if scalar else 0), problem.encode(), _p(cfg_u, u64p), _p(cfg_d),
                                        _p(g), u64(igd_H), _p(x), _p(f), C.byref(rows), C.byref(done),
                                        _p(pops, u64p), _p(ms), _p(igd)))
        k, g_done = rows.value, done.value
        return dict(x=None if x is None else x[:k].copy(), f=f[:k].copy(), pop_size=pops[:g_done],
                    elapsed_ms=ms[:g_done], igd=igd[:g_done])

    def rvea_run_op(self, op, problem, n, d, m, generations, seed=42, lattice_h=0, alpha=2.0, fr=0.1, ga=GA_DEFAULT,
                    opp=OPP_DEFAULT):
        """The reference's own rvea_run with RunConfig::op = op (algorithms.hpp:250-271)."""
        H = lattice_h or self.lattice_density_for(m, n)
        r = self.lattice_count(m, H)
        cap = max(n, r)
        x, f = np.empty((cap, d)), np.empty((cap, m))
        cfg_u = np.array([n, lattice_h, generations, seed, d, m], dtype=np.uint64)
        cfg_d = np.array([alpha, fr, 0.0])
        rows, done = u64(0), u64(0)
        pops = np.zeros(generations, dtype=np.uint64)
        self._chk(self.lib.ref_rvea_run_op(problem.encode(), op.encode(), _p(_f(opp)), _p(cfg_u, u64p), _p(cfg_d), _p(_f(ga)),
                                           _p(x), _p(f), C.byref(rows), C.byref(done), _p(pops, u64p)))
        k = rows.value
        return dict(x=x[:k].copy(), f=f[:k].copy(), pop_size=pops[: done.value])
