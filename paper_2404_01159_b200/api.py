"""Host-side mirror of the reference's operator / problem / selection / algorithm interface
for the TensorRVEA generation loop, bound to the CUDA implementation through the C ABI.

Names, argument meaning, draw-counter behaviour and error behaviour follow the reference's
free functions (reference paths under proj/include/temo/):

    RngStream, uniform_tensor, shuffle_indices           rng.hpp:34-78
    GaParams, sbx, polynomial_mutation, ga_reproduce,
    random_reproduce                                     operators.hpp:22-27,65-161,287-296
    dtlz_eval, ProblemInstance, make_problem             problems.hpp:69-92,246-296
    lattice_count, lattice_density_for, simplex_lattice,
    RefVectorSet, make_ref_set, min_vector_angles, adapt refvec.hpp:15-140
    DeParams, PsoParams, CsoParams, SwarmState, make_swarm_state,
    de_reproduce, pso_reproduce, cso_reproduce           operators.hpp:28-60,166-284
    SelectionOutcome, rv_select, apd_scores              selection.hpp:131-135,200-234
    RunConfig, RunRecord, GenerationRow, rvea_run        algorithms.hpp:21-63,144-150,227-296

A ``Tensor2D`` is a C-contiguous float64 numpy array of shape (rows, cols). Contract
violations raise ValueError where the reference throws std::invalid_argument. Everything
numeric runs in the sm_100a kernels; nothing here computes on the CPU except the pieces the
design keeps on the host (lattice enumeration, Fisher-Yates permutation, scalar APD penalty),
which live in the shared library too.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import GaParamsC, RunConfigC, TemoB200Error, f64p, u64, u64p, u8p

PROBLEM_IDS = {"dtlz1": 1, "dtlz2": 2, "dtlz3": 3, "dtlz4": 4, "lsmop1": 101, "toy2": 201, "toy3": 202}
TOY_HIDDEN = 16  # make_problem's MlpArch{4, 16, 2} (problems.hpp:280)
RNG_SPLITMIX64, RNG_PHILOX = 0, 1


def _call(fn, *args):
    rc = fn(*args)
    if rc != 0:
        msg = _lib.load().temo_b200_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(msg)  # reference: std::invalid_argument
        if rc == 4:
            raise MemoryError(msg)
        raise TemoB200Error(rc, msg)


def _t(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


def _p(a, typ=f64p):
    return None if a is None else a.ctypes.data_as(typ)


def device_count() -> int:
    return int(_lib.load().temo_b200_device_count())


def init(device: int = 0) -> None:
    _call(_lib.load().temo_b200_init, device)


def set_option(name: str, value: int) -> None:
    """Path-selection knobs for tests / A-B runs (results are identical on every path): "k1_generic",
    "k1_bound_arrays", "k1_cand_cap" (see include/temo_b200.h)."""
    _call(_lib.load().temo_b200_set_option, name.encode(), int(value))


def pow_like_host(x, y, on_device: bool = True) -> np.ndarray:
    """Self-test hook: elementwise pow through the libm-exact implementation (device or host twin)."""
    x, y = _t(x).reshape(-1), _t(y).reshape(-1)
    out = np.empty_like(x)
    _call(_lib.load().temo_b200_pow, _p(x), _p(y), u64(x.size), _p(out), 1 if on_device else 0)
    return out


def tanh_like_host(x, on_device: bool = True) -> np.ndarray:
    """tanh with the host libm's bits (csrc/glibc_tanh.cuh): the device kernel, or its host twin (no GPU needed)."""
    x = _t(x).reshape(-1)
    out = np.empty_like(x)
    _call(_lib.load().temo_b200_tanh, _p(x), u64(x.size), _p(out), 1 if on_device else 0)
    return out


# ------------------------------------------------------------------------------- rng.hpp
@dataclass
class RngStream:
    """reference: RngStream (rng.hpp:34-52); `counter` advances exactly as in the reference."""
    seed: int = 0
    counter: int = 0
    mode: int = RNG_SPLITMIX64

    def at(self, c: int) -> "RngStream":
        return RngStream(self.seed, c, self.mode)


def uniform_tensor(stream: RngStream, rows: int, cols: int) -> np.ndarray:
    out = np.empty((rows, cols))
    c = u64(stream.counter)
    _call(_lib.load().temo_b200_uniform_tensor, u64(stream.seed), C.byref(c), u64(rows), u64(cols), stream.mode, _p(out))
    stream.counter = c.value
    return out


def shuffle_indices(stream: RngStream, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    c = u64(stream.counter)
    _call(_lib.load().temo_b200_shuffle_indices, u64(stream.seed), C.byref(c), u64(n), _p(out, u64p))
    stream.counter = c.value
    return out


def parent_pool_indices(current: int, n: int, stream: RngStream) -> np.ndarray:
    """reference: algorithms.hpp:211-221."""
    out = np.empty(n, dtype=np.uint64)
    c = u64(stream.counter)
    _call(_lib.load().temo_b200_parent_pool_indices, u64(current), u64(n), u64(stream.seed), C.byref(c), _p(out, u64p))
    stream.counter = c.value
    return out


# ------------------------------------------------------------------------- operators.hpp
@dataclass
class GaParams:
    pc: float = 1.0
    eta: float = 20.0
    pm: float = 1.0
    xi: float = 20.0

    def c(self) -> GaParamsC:
        return GaParamsC(self.pc, self.eta, self.pm, self.xi)


def _operator(fn, x, stream, p, lower, upper):
    x = _t(x)
    if x.ndim != 2:
        raise ValueError("operator: x must be a 2-D tensor")
    n, d = x.shape
    lower, upper = _t(lower).reshape(-1), _t(upper).reshape(-1)
    if lower.size != d or upper.size != d:
        raise ValueError("operator: bounds shape mismatch")
    out = np.empty_like(x)
    c = u64(stream.counter)
    g = (p or GaParams()).c()
    _call(fn, _p(x), u64(n), u64(d), u64(stream.seed), C.byref(c), C.byref(g), _p(lower), _p(upper), stream.mode, _p(out))
    stream.counter = c.value
    return out


def sbx(x, stream: RngStream, p: GaParams, lower, upper) -> np.ndarray:
    return _operator(_lib.load().temo_b200_sbx, x, stream, p, lower, upper)


def polynomial_mutation(x, stream: RngStream, p: GaParams, lower, upper) -> np.ndarray:
    return _operator(_lib.load().temo_b200_polynomial_mutation, x, stream, p, lower, upper)


def ga_reproduce(x, stream: RngStream, p: GaParams, lower, upper) -> np.ndarray:
    return _operator(_lib.load().temo_b200_ga_reproduce, x, stream, p, lower, upper)


def random_reproduce(n: int, d: int, stream: RngStream, lower, upper) -> np.ndarray:
    lower, upper = _t(lower).reshape(-1), _t(upper).reshape(-1)
    out = np.empty((n, d))
    c = u64(stream.counter)
    _call(_lib.load().temo_b200_random_reproduce, u64(n), u64(d), u64(stream.seed), C.byref(c), _p(lower), _p(upper),
          stream.mode, _p(out))
    stream.counter = c.value
    return out


# ---- the other reproduction operators (operators.hpp:28-60,166-284)
@dataclass
class DeParams:
    """reference: DeParams (operators.hpp:28-31)."""
    f: float = 0.5
    cr: float = 0.9


@dataclass
class PsoParams:
    """reference: PsoParams (operators.hpp:33-37)."""
    inertia: float = 0.4
    c1: float = 1.5
    c2: float = 1.5


@dataclass
class CsoParams:
    """reference: CsoParams (operators.hpp:39-41)."""
    phi: float = 0.1


@dataclass
class SwarmState:
    """reference: SwarmState (operators.hpp:46-56); the operators update it in place."""
    velocities: np.ndarray
    personal_best_x: np.ndarray
    personal_best_score: np.ndarray

    def empty(self) -> bool:
        return self.velocities.shape[0] == 0


def make_swarm_state(x, scores) -> SwarmState:
    """reference: make_swarm_state (operators.hpp:58-60)."""
    x = _t(x)
    return SwarmState(np.zeros_like(x), x.copy(), _t(scores).reshape(-1).copy())


def _bounds(lower, upper, d, who):
    lower, upper = _t(lower).reshape(-1), _t(upper).reshape(-1)
    if lower.size != d or upper.size != d:
        raise ValueError(f"{who}: bounds shape mismatch")
    return lower, upper


def de_reproduce(x, stream: RngStream, p: DeParams, lower, upper, timing: dict | None = None) -> np.ndarray:
    """reference: de_reproduce (operators.hpp:166-200). `timing["kernel_ms"]` receives the device time."""
    x = _t(x)
    n, d = x.shape
    lower, upper = _bounds(lower, upper, d, "de_reproduce")
    p = p or DeParams()
    out, c, ms = np.empty_like(x), u64(stream.counter), C.c_double(0.0)
    _call(_lib.load().temo_b200_de_reproduce, _p(x), u64(n), u64(d), u64(stream.seed), C.byref(c), C.c_double(p.f), C.c_double(p.cr),
          _p(lower), _p(upper), stream.mode, _p(out), C.cast(C.byref(ms), _lib.f64p))
    stream.counter = c.value
    if timing is not None:
        timing["kernel_ms"] = ms.value
    return out


def pso_reproduce(x, state: SwarmState, scores, stream: RngStream, p: PsoParams, lower, upper, timing: dict | None = None) -> np.ndarray:
    """reference: pso_reproduce (operators.hpp:205-240); `state` is updated in place."""
    x, scores = _t(x), _t(scores).reshape(-1)
    n, d = x.shape
    if state.velocities.shape != (n, d) or state.personal_best_x.shape[0] != n or scores.size != n:
        raise ValueError("pso_reproduce: state shape mismatch")  # operators.hpp:209-211
    lower, upper = _bounds(lower, upper, d, "pso_reproduce")
    p = p or PsoParams()
    vel, pbx, pbs = _t(state.velocities).copy(), _t(state.personal_best_x).copy(), _t(state.personal_best_score).reshape(-1).copy()
    out, c, ms = np.empty_like(x), u64(stream.counter), C.c_double(0.0)
    _call(_lib.load().temo_b200_pso_reproduce, _p(x), _p(scores), u64(n), u64(d), u64(stream.seed), C.byref(c), C.c_double(p.inertia),
          C.c_double(p.c1), C.c_double(p.c2), _p(vel), _p(pbx), _p(pbs), _p(lower), _p(upper), stream.mode, _p(out),
          C.cast(C.byref(ms), _lib.f64p))
    stream.counter = c.value
    state.velocities, state.personal_best_x, state.personal_best_score = vel, pbx, pbs
    if timing is not None:
        timing["kernel_ms"] = ms.value
    return out


def cso_reproduce(x, scores, stream: RngStream, p: CsoParams, lower, upper, state: SwarmState, timing: dict | None = None) -> np.ndarray:
    """reference: cso_reproduce (operators.hpp:246-284); `state.velocities` is updated in place."""
    x, scores = _t(x), _t(scores).reshape(-1)
    n, d = x.shape
    if state.velocities.shape != (n, d) or scores.size != n:
        raise ValueError("cso_reproduce: state shape mismatch")  # operators.hpp:251-253
    lower, upper = _bounds(lower, upper, d, "cso_reproduce")
    p = p or CsoParams()
    vel = _t(state.velocities).copy()
    out, c, ms = np.empty_like(x), u64(stream.counter), C.c_double(0.0)
    _call(_lib.load().temo_b200_cso_reproduce, _p(x), _p(scores), u64(n), u64(d), u64(stream.seed), C.byref(c), C.c_double(p.phi),
          _p(vel), _p(lower), _p(upper), stream.mode, _p(out), C.cast(C.byref(ms), _lib.f64p))
    stream.counter = c.value
    state.velocities = vel
    if timing is not None:
        timing["kernel_ms"] = ms.value
    return out


# -------------------------------------------------------------------------- problems.hpp
def evaluate(problem: str | int, x, m: int, horizon: int = 100) -> np.ndarray:
    """ProblemInstance::evaluate of make_problem(problem, d, m, horizon) (problems.hpp:261-296), minimisation orientation."""
    pid = PROBLEM_IDS[problem] if isinstance(problem, str) else int(problem)
    x = _t(x)
    if x.ndim != 2:
        raise ValueError("evaluate: x must be a 2-D tensor")
    n, d = x.shape
    f = np.empty((n, m))
    _call(_lib.load().temo_b200_evaluate_h, pid, _p(x), u64(n), u64(d), u64(m), u64(horizon), _p(f))
    return f


def mlp_param_count(hidden: int = TOY_HIDDEN) -> int:
    """reference: MlpArch::param_count (problems.hpp:113-115) for obs_dim 4, act_dim 2."""
    return 4 * hidden + hidden + hidden * 2 + 2


def env_rollout(params, horizon: int = 100, num_obj: int = 2, hidden: int = TOY_HIDDEN) -> np.ndarray:
    """reference: env_rollout (problems.hpp:211-241): n x d flat MLP parameters -> n x num_obj returns (maximisation)."""
    params = _t(params)
    if params.ndim != 2 or params.shape[1] != mlp_param_count(hidden):
        raise ValueError("env_rollout: parameter length mismatch")
    n, d = params.shape
    f = np.empty((n, num_obj))
    _call(_lib.load().temo_b200_env_rollout, _p(params), u64(n), u64(d), u64(hidden), u64(horizon), u64(num_obj), _p(f))
    return f


def mlp_forward(params, obs, hidden: int = TOY_HIDDEN) -> np.ndarray:
    """reference: mlp_forward (problems.hpp:149-163), batched: individual i on observation i; n x 4 -> n x 2."""
    params, obs = _t(params), _t(obs)
    if params.ndim != 2 or params.shape[1] != mlp_param_count(hidden):
        raise ValueError("mlp_decode: length mismatch")
    if obs.shape != (params.shape[0], 4):
        raise ValueError("mlp_forward: observations must be n x 4")
    act = np.empty((params.shape[0], 2))
    _call(_lib.load().temo_b200_mlp_forward, _p(params), u64(params.shape[0]), u64(params.shape[1]), u64(hidden), _p(obs), _p(act))
    return act


def dtlz_eval(id: int, x, m: int) -> np.ndarray:
    """reference: dtlz_eval (problems.hpp:69-92)."""
    if not 1 <= id <= 4:
        raise ValueError("dtlz_eval: id must be in 1..4")
    return evaluate(id, x, m)


@dataclass
class ProblemInstance:
    """reference: ProblemInstance (problems.hpp:246-257)."""
    name: str
    dim: int
    num_obj: int
    lower: np.ndarray
    upper: np.ndarray
    dtlz_id: int = 0
    pf_extent: float = 1.0
    maximization: bool = False
    problem_id: int = 0
    horizon: int = 100  # toy environments: make_problem's toy_horizon

    def evaluate(self, x) -> np.ndarray:
        return evaluate(self.problem_id, x, self.num_obj, self.horizon)


def make_problem(name: str, dim: int = 0, m: int = 3, toy_horizon: int = 100) -> ProblemInstance:
    """reference: make_problem (problems.hpp:261-296): dtlz1..dtlz4, toy2, toy3, plus 'lsmop1' (an extension)."""
    if name not in PROBLEM_IDS:
        raise ValueError(f"make_problem: unknown problem '{name}'")
    pid = PROBLEM_IDS[name]
    L = _lib.load()
    toy = name in ("toy2", "toy3")
    if toy:
        m = 2 if name == "toy2" else 3
        if dim not in (0, mlp_param_count()):
            raise ValueError("make_problem: toy env dimension is fixed")
    d = dim or int(L.temo_b200_problem_default_dim(pid, u64(m)))
    if d < m:
        raise ValueError("make_problem: DTLZ needs d >= m")
    lo, hi = np.empty(d), np.empty(d)
    _call(L.temo_b200_problem_bounds, pid, u64(d), u64(m), _p(lo), _p(hi))
    return ProblemInstance(name, d, m, lo, hi, dtlz_id=pid if pid <= 4 else 0,
                           pf_extent=0.5 if pid == 1 else 1.0, problem_id=pid, maximization=toy, horizon=toy_horizon)


# ---------------------------------------------------------------------------- refvec.hpp
def lattice_count(m: int, H: int) -> int:
    return int(_lib.load().temo_b200_lattice_count(u64(m), u64(H)))


def lattice_density_for(m: int, target: int) -> int:
    return int(_lib.load().temo_b200_lattice_density_for(u64(m), u64(target)))


def simplex_lattice(m: int, H: int) -> np.ndarray:
    if m < 2:
        raise ValueError("simplex_lattice: m must be at least 2")
    if H < 1:
        raise ValueError("simplex_lattice: H must be at least 1")
    out = np.empty((lattice_count(m, H), m))
    _call(_lib.load().temo_b200_simplex_lattice, u64(m), u64(H), _p(out))
    return out


@dataclass
class RefVectorSet:
    """reference: RefVectorSet (refvec.hpp:102-106)."""
    v0: np.ndarray
    v: np.ndarray
    gamma: np.ndarray


def min_vector_angles(v) -> np.ndarray:
    v = _t(v)
    gamma = np.empty(v.shape[0])
    _call(_lib.load().temo_b200_min_vector_angles, _p(v), u64(v.shape[0]), u64(v.shape[1]), _p(gamma))
    return gamma


def make_ref_set(m: int, H: int) -> RefVectorSet:
    if m < 2:
        raise ValueError("simplex_lattice: m must be at least 2")
    if H < 1:
        raise ValueError("simplex_lattice: H must be at least 1")
    r = lattice_count(m, H)
    v0, gamma = np.empty((r, m)), np.empty(r)
    _call(_lib.load().temo_b200_make_ref_set, u64(m), u64(H), _p(v0), _p(gamma))
    return RefVectorSet(v0, v0.copy(), gamma)


def adapt(refs: RefVectorSet, z_min, z_max) -> None:
    """reference: adapt (refvec.hpp:135-140): in place; untouched unless every range is > 0."""
    z_min, z_max = _t(z_min).reshape(-1), _t(z_max).reshape(-1)
    v0 = _t(refs.v0)
    r, m = v0.shape
    if z_min.size != m or z_max.size != m:
        raise ValueError("adapt_vectors: range shape mismatch")
    v, gamma = _t(refs.v).copy(), _t(refs.gamma).reshape(-1).copy()
    _call(_lib.load().temo_b200_adapt, _p(v0), _p(v), _p(gamma), u64(r), u64(m), _p(z_min), _p(z_max))
    refs.v, refs.gamma = v, gamma


# ------------------------------------------------------------------------- selection.hpp
@dataclass
class SelectionOutcome:
    """reference: SelectionOutcome (selection.hpp:131-135) + RvCore (selection.hpp:139-143)."""
    elite_indices: np.ndarray
    validity: np.ndarray
    assoc: np.ndarray
    theta: np.ndarray
    apd: np.ndarray


def apd_penalty(m: int, t: int, t_max: int, alpha: float) -> float:
    return float(_lib.load().temo_b200_apd_penalty(u64(m), u64(t), u64(t_max), alpha))


def rv_select(f, refs: RefVectorSet, t: int, t_max: int, alpha: float = 2.0) -> SelectionOutcome:
    f, v, gamma = _t(f), _t(refs.v), _t(refs.gamma).reshape(-1)
    if f.ndim != 2 or f.shape[1] != v.shape[1]:
        raise ValueError("rv_select: objective count mismatch")  # selection.hpp:150
    n, m = f.shape
    r = v.shape[0]
    elite = np.empty(max(r, 1), dtype=np.uint64)
    valid = np.empty(r, dtype=np.uint8)
    assoc = np.empty(n, dtype=np.uint64)
    theta, apd = np.empty(n), np.empty(n)
    ne = u64(0)
    _call(_lib.load().temo_b200_rv_select, _p(f), u64(n), u64(m), _p(v), _p(gamma), u64(r), u64(t), u64(t_max),
          C.c_double(alpha), _p(elite, u64p), C.byref(ne), _p(valid, u8p), _p(assoc, u64p), _p(theta), _p(apd))
    return SelectionOutcome(elite[: ne.value].copy(), valid, assoc, theta, apd)


def apd_scores(f, refs: RefVectorSet, t: int, t_max: int, alpha: float = 2.0) -> np.ndarray:
    """reference: apd_scores (selection.hpp:228-234): every row's APD against its associated vector, n x 1."""
    return rv_select(f, refs, t, t_max, alpha).apd.reshape(-1, 1).copy()


# ------------------------------------------------------------------------ algorithms.hpp
OPERATOR_IDS = {"ga": 0, "de": 1, "pso": 2, "cso": 3, "random": 4}  # TEMO_B200_OP_*


@dataclass
class RunConfig:
    """reference: RunConfig (algorithms.hpp:21-41); op = ga / de / pso / cso / random. track_archive defaults to false
    here (the reference's default is true; its own timing harness switches it off, temo.cpp:260)."""
    problem: str = "dtlz2"
    op: str = "ga"
    pop: int = 105
    lattice_h: int = 0
    generations: int = 100
    alpha: float = 2.0
    fr: float = 0.1
    seed: int = 42
    time_budget_s: float = 0.0
    dim: int = 0
    obj: int = 3
    ga: GaParams = field(default_factory=GaParams)
    de: tuple = (0.5, 0.9)         # DeParams {f, cr}, operators.hpp:28-31
    pso: tuple = (0.4, 1.5, 1.5)   # PsoParams {inertia, c1, c2}, operators.hpp:33-37
    cso: tuple = (0.1,)            # CsoParams {phi}, operators.hpp:39-41
    rng_mode: int = RNG_SPLITMIX64
    fuse_eval: object = None       # None: by shape (rows wider than 1024 genes), True: whenever possible, False: never
    horizon: int = 100             # algorithms.hpp:35 (toy environments)
    track_archive: bool = False    # algorithms.hpp:31
    archive_cap: int = 0           # algorithms.hpp:32 (0: unbounded)
    archive_history: bool = False  # algorithms.hpp:33

    def c(self) -> RunConfigC:
        if self.op not in OPERATOR_IDS:
            raise ValueError(f"rvea_run: unknown operator '{self.op}'")  # algorithms.hpp:270
        if self.problem not in PROBLEM_IDS:
            raise ValueError(f"make_problem: unknown problem '{self.problem}'")
        cfg = RunConfigC()
        _lib.load().temo_b200_default_run_config(C.byref(cfg))
        cfg.problem = PROBLEM_IDS[self.problem]
        cfg.rng_mode = self.rng_mode
        cfg.pop, cfg.lattice_h, cfg.generations, cfg.seed = self.pop, self.lattice_h, self.generations, self.seed
        cfg.dim, cfg.obj = self.dim, self.obj
        cfg.alpha, cfg.fr, cfg.time_budget_s = self.alpha, self.fr, self.time_budget_s
        cfg.ga = self.ga.c()
        cfg.fuse_eval = 2 if self.fuse_eval is None else (1 if self.fuse_eval else 0)
        cfg.op = OPERATOR_IDS[self.op]
        cfg.opp.de_f, cfg.opp.de_cr = self.de
        cfg.opp.pso_inertia, cfg.opp.pso_c1, cfg.opp.pso_c2 = self.pso
        (cfg.opp.cso_phi,) = self.cso
        cfg.horizon = self.horizon
        return cfg


@dataclass
class GenerationRow:
    t: int
    elapsed_ms: float
    pop_size: int
    igd_value: float = float("nan")
    hv_value: float = float("nan")


# ---- metrics.hpp --------------------------------------------------------------------------
@dataclass
class HvEstimate:
    """reference: HvEstimate (metrics.hpp:68-71)."""
    value: float = 0.0
    std_error: float = 0.0


@dataclass
class MetricContext:
    """reference: MetricContext (algorithms.hpp:46-54); the expected-utility weights are not on this path."""
    pf_ref: np.ndarray | None = None   # IGD reference front (None -> no IGD)
    hv_ref: np.ndarray | None = None   # reference point, m values (None -> no HV)
    hv_scale: float = 1.0
    hv_samples: int = 2048
    hv_seed: int = 9001
    maximization: bool = False


def crowding_distance(front) -> np.ndarray:
    """reference: crowding_distance (selection.hpp:289-312); host code."""
    front = _t(front)
    if front.shape[0] < 1:
        raise ValueError("crowding_distance: empty front")
    out = np.empty(front.shape[0])
    _call(_lib.load().temo_b200_crowding_distance, _p(front), u64(front.shape[0]), u64(front.shape[1]), _p(out))
    return out


class Archive:
    """reference: Archive (algorithms.hpp:68-144): running set of mutually nondominated solutions."""

    def __init__(self):
        self.x = np.empty((0, 0))
        self.f = np.empty((0, 0))

    def insert(self, xn, fn, cap: int = 0) -> None:
        xn, fn = _t(xn), _t(fn)
        n_old, n_new = self.f.shape[0], fn.shape[0]
        d, m = xn.shape[1], fn.shape[1]
        x_out, f_out = np.empty((n_old + n_new, d)), np.empty((n_old + n_new, m))
        rows = u64(0)
        xo = _t(self.x) if n_old else None
        fo = _t(self.f) if n_old else None
        _call(_lib.load().temo_b200_archive_insert, _p(xo), _p(fo), u64(n_old), _p(xn), _p(fn), u64(n_new), u64(d), u64(m), u64(cap),
              _p(x_out), _p(f_out), C.byref(rows))
        self.x, self.f = x_out[: rows.value].copy(), f_out[: rows.value].copy()


def igd(f, f_ref) -> float:
    """reference: igd (metrics.hpp:21-44)."""
    f, f_ref = _t(f), _t(f_ref)
    if f.shape[0] < 1 or f_ref.shape[0] < 1:
        raise ValueError("igd: empty set")
    if f.shape[1] != f_ref.shape[1]:
        raise ValueError("igd: objective count mismatch")
    out = C.c_double(0)
    _call(_lib.load().temo_b200_igd, _p(f), u64(f.shape[0]), u64(f.shape[1]), _p(f_ref), u64(f_ref.shape[0]), C.byref(out))
    return out.value


def hv_mc_box(f, lo, ref, samples: int, seed: int) -> HvEstimate:
    """reference: hv_mc_box (metrics.hpp:76-117)."""
    f, lo, ref = _t(f), _t(lo).reshape(-1), _t(ref).reshape(-1)
    if samples < 1:
        raise ValueError("hv_mc: needs at least one sample")
    if f.shape[0] < 1 or ref.shape[0] != f.shape[1]:
        raise ValueError("hv_mc: bad shapes")
    if lo.shape[0] != f.shape[1]:
        raise ValueError("hv_mc: bad box")
    v, e = C.c_double(0), C.c_double(0)
    _call(_lib.load().temo_b200_hv_mc_box, _p(f), u64(f.shape[0]), u64(f.shape[1]), _p(lo), _p(ref), u64(samples), u64(seed),
          C.byref(v), C.byref(e))
    return HvEstimate(v.value, e.value)


def hv_mc(f, ref, samples: int, seed: int) -> HvEstimate:
    """reference: hv_mc (metrics.hpp:121-124): the box is [col_min(f), ref]."""
    f, ref = _t(f), _t(ref).reshape(-1)
    if samples < 1:
        raise ValueError("hv_mc: needs at least one sample")
    if f.shape[0] < 1 or ref.shape[0] != f.shape[1]:
        raise ValueError("hv_mc: bad shapes")
    v, e = C.c_double(0), C.c_double(0)
    _call(_lib.load().temo_b200_hv_mc, _p(f), u64(f.shape[0]), u64(f.shape[1]), _p(ref), u64(samples), u64(seed), C.byref(v), C.byref(e))
    return HvEstimate(v.value, e.value)


@dataclass
class RunRecord:
    """reference: RunRecord (algorithms.hpp:144-150); archive = (x, f) in insertion order or None."""
    rows: list
    final_x: np.ndarray
    final_f: np.ndarray
    archive: tuple | None = None
    archive_f_history: list = field(default_factory=list)


class _PinnedBlock:
    """Owner of one temo_b200_host_alloc block; freed when the last numpy view on it is gone."""

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            _lib.load().temo_b200_host_free(C.c_void_p(self.ptr))
        except Exception:
            pass


def _pinned_array(rows: int, cols: int) -> np.ndarray:
    """rows x cols float64 in page-locked host memory (pageable numpy memory if the allocation fails)."""
    ptr = _lib.load().temo_b200_host_alloc(rows * cols * 8)
    if not ptr:
        return np.empty((rows, cols))
    buf = (C.c_double * (rows * cols)).from_address(ptr)
    buf._owner = _PinnedBlock(ptr)  # the array's base keeps the block alive
    return np.ctypeslib.as_array(buf).reshape(rows, cols)


class RveaRun:
    """Device-resident generation loop (session form of rvea_run): create -> step()* -> download()."""

    def __init__(self, cfg: RunConfig):
        self._L = _lib.load()
        self._h = C.c_void_p()
        ccfg = cfg.c()
        _call(self._L.temo_b200_run_create, C.byref(ccfg), C.byref(self._h))
        self.cfg = cfg
        st = self.state()
        self.r, self.d, self.m, self.n = st["r"], st["d"], st["m"], cfg.pop
        # survivors' objectives land in page-locked memory (full-rate D2H); the views handed out are valid until close()
        rows = max(self.r, self.n)
        self._fbuf = _pinned_array(rows, self.m)

    def close(self):
        if self._h:
            _call(self._L.temo_b200_run_destroy, self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def step(self, want_f: bool = False):
        """One generation; returns the survivor count (and the survivors' objectives if asked)."""
        p = u64(0)
        _call(self._L.temo_b200_run_step, self._h, C.byref(p), _p(self._fbuf) if want_f else None)
        if want_f:
            return p.value, self._fbuf[: p.value]
        return p.value

    def step_injected(self, f_off) -> int:
        """Lock-step testing: selection runs on the given offspring objectives (n x m)."""
        f_off = _t(f_off)
        if f_off.shape != (self.n, self.m):
            raise ValueError("step_injected: f_off must be n x m")
        p = u64(0)
        _call(self._L.temo_b200_run_step_injected, self._h, _p(f_off), C.byref(p))
        return p.value

    def state(self) -> dict:
        vals = [u64(0) for _ in range(6)]
        _call(self._L.temo_b200_run_state, self._h, *[C.byref(v) for v in vals])
        return dict(zip(("rows", "counter", "t", "r", "d", "m"), (v.value for v in vals)))

    def inject(self, x=None, f=None, v=None, gamma=None, counter=0, t=0, rows=None):
        x = None if x is None else _t(x)
        f = None if f is None else _t(f)
        v = None if v is None else _t(v)
        gamma = None if gamma is None else _t(gamma).reshape(-1)
        if rows is None:
            rows = x.shape[0] if x is not None else (f.shape[0] if f is not None else self.state()["rows"])
        _call(self._L.temo_b200_run_inject, self._h, u64(rows), _p(x), _p(f), _p(v), _p(gamma), u64(counter), u64(t))

    def download(self, want_x=True):
        rows = self.state()["rows"]
        x = np.empty((rows, self.d)) if want_x else None
        f = np.empty((rows, self.m))
        v, gamma = np.empty((self.r, self.m)), np.empty(self.r)
        _call(self._L.temo_b200_run_download, self._h, _p(x), _p(f), _p(v), _p(gamma))
        return dict(x=x, f=f, v=v, gamma=gamma)

    def last_generation(self):
        rows = self.state()["rows"]
        off, f_off = np.empty((self.n, self.d)), np.empty((self.n, self.m))
        elite = np.empty(rows, dtype=np.uint64)
        _call(self._L.temo_b200_run_last_generation, self._h, _p(off), _p(f_off), _p(elite, u64p))
        return dict(offspring=off, f_off=f_off, elite=elite)

    def timings(self) -> dict:
        ms = np.zeros(8)
        _call(self._L.temo_b200_run_timings, self._h, _p(ms))
        return dict(generation=ms[0], reproduce=ms[1], evaluate=ms[2], select=ms[3], adapt=ms[4], host_perm=ms[5],
                    launches=int(ms[6]), prep=ms[7])

    def timing_history(self, max_steps: int = 1024, reset: bool = True) -> list:
        """Stage timings (the dict of timings()) of each of the last steps since the last reset, oldest first; the library
        reads a step's events while the next step runs, so a timed loop asks once after the loop."""
        ms = np.zeros((max_steps, 8))
        count = C.c_uint64(0)
        _call(self._L.temo_b200_run_timing_history, self._h, _p(ms), u64(max_steps), C.c_int(1 if reset else 0), C.byref(count))
        keys = ("generation", "reproduce", "evaluate", "select", "adapt", "host_perm", "launches", "prep")
        return [{k: (int(row[i]) if k == "launches" else float(row[i])) for i, k in enumerate(keys)} for row in ms[:count.value]]

    def set_metrics(self, mc: MetricContext) -> None:
        """MetricContext of this run (algorithms.hpp:46-54): the references move to the device once."""
        pf = None if mc.pf_ref is None else _t(mc.pf_ref)
        hv = None if mc.hv_ref is None else _t(mc.hv_ref).reshape(-1)
        if pf is not None and pf.shape[1] != self.m:
            raise ValueError("igd: objective count mismatch")
        if hv is not None and hv.shape[0] != self.m:
            raise ValueError("hv_mc: bad shapes")
        _call(self._L.temo_b200_run_set_metrics, self._h, _p(pf), u64(0 if pf is None else pf.shape[0]), _p(hv),
              C.c_double(mc.hv_scale), u64(mc.hv_samples), u64(mc.hv_seed), int(mc.maximization))

    def track_archive(self, cap: int = 0) -> None:
        """Archive of the run kept in HBM (algorithms.hpp:68-142): call right after construction (inserts the initial
        population, algorithms.hpp:243); every step then inserts its survivors and metrics() reports the archive."""
        _call(self._L.temo_b200_run_track_archive, self._h, u64(cap))

    def archive(self) -> tuple:
        """(x, f) of the archive in insertion order."""
        rows = u64(0)
        _call(self._L.temo_b200_run_archive_rows, self._h, C.byref(rows))
        x, f = np.empty((rows.value, self.d)), np.empty((rows.value, self.m))
        _call(self._L.temo_b200_run_archive, self._h, _p(x), _p(f))
        return x, f

    def metrics(self) -> tuple:
        """fill_metrics (algorithms.hpp:161-180) on the survivors' objectives (the archive's when one is tracked),
        evaluated on the device: (igd, hv)."""
        a, b = C.c_double(0), C.c_double(0)
        _call(self._L.temo_b200_run_metrics, self._h, C.byref(a), C.byref(b))
        return a.value, b.value

    def time_stage(self, stage: int, reps: int = 5) -> float:
        out = C.c_double(0)
        _call(self._L.temo_b200_run_time_stage, self._h, stage, reps, C.byref(out))
        return out.value


# ---- NSGA-II baseline ---------------------------------------------
def nondominated_sort(f) -> np.ndarray:
    """reference: nondominated_sort (selection.hpp:251-283): front rank of every row."""
    f = _t(f)
    rank = np.zeros(f.shape[0], dtype=np.uint64)
    _call(_lib.load().temo_b200_nondominated_sort, _p(f), u64(f.shape[0]), u64(f.shape[1]), _p(rank, u64p))
    return rank


def nsga2_select(f, target: int) -> np.ndarray:
    """reference: nsga2_select (selection.hpp:316-346)."""
    f = _t(f)
    if target > f.shape[0]:
        raise ValueError("nsga2_select: target exceeds population")
    sel = np.zeros(target, dtype=np.uint64)
    _call(_lib.load().temo_b200_nsga2_select, _p(f), u64(f.shape[0]), u64(f.shape[1]), u64(target), _p(sel, u64p))
    return sel


class Nsga2Run:
    """Device-resident NSGA-II loop (session form of nsga2_run, algorithms.hpp:301-369)."""

    def __init__(self, cfg: RunConfig):
        self._L = _lib.load()
        self._h = C.c_void_p()
        ccfg = cfg.c()
        _call(self._L.temo_b200_nsga2_create, C.byref(ccfg), C.byref(self._h))
        self.n, self.m = cfg.pop, cfg.obj
        self.d = self.state()["d"]

    def close(self):
        if self._h:
            self._L.temo_b200_nsga2_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def state(self) -> dict:
        vals = [u64(0) for _ in range(3)]
        _call(self._L.temo_b200_nsga2_state, self._h, *[C.byref(v) for v in vals])
        return dict(zip(("counter", "t", "d"), (v.value for v in vals)))

    def step(self, f_off=None) -> None:
        f_off = None if f_off is None else _t(f_off)
        if f_off is not None and f_off.shape != (self.n, self.m):
            raise ValueError("nsga2 step: f_off must be n x m")
        _call(self._L.temo_b200_nsga2_step, self._h, _p(f_off))

    def inject(self, x=None, f=None, counter=0, t=0) -> None:
        x = None if x is None else _t(x)
        f = None if f is None else _t(f)
        _call(self._L.temo_b200_nsga2_inject, self._h, _p(x), _p(f), u64(counter), u64(t))

    def download(self) -> dict:
        x, f = np.empty((self.n, self.d)), np.empty((self.n, self.m))
        _call(self._L.temo_b200_nsga2_download, self._h, _p(x), _p(f))
        return dict(x=x, f=f)

    def last_generation(self) -> dict:
        off, f_off = np.empty((self.n, self.d)), np.empty((self.n, self.m))
        sel, pool = np.zeros(self.n, dtype=np.uint64), np.zeros(self.n, dtype=np.uint64)
        _call(self._L.temo_b200_nsga2_last_generation, self._h, _p(off), _p(f_off), _p(sel, u64p), _p(pool, u64p))
        return dict(offspring=off, f_off=f_off, sel=sel, pool_idx=pool)


def nsga2_run(prob: ProblemInstance, cfg: RunConfig) -> RunRecord:
    """reference: nsga2_run (algorithms.hpp:301-369), track_archive = false."""
    cfg = RunConfig(**{**cfg.__dict__, "problem": prob.name, "dim": prob.dim, "obj": prob.num_obj, "horizon": prob.horizon})
    ccfg = cfg.c()
    x, f = np.empty((cfg.pop, prob.dim)), np.empty((cfg.pop, prob.num_obj))
    done = u64(0)
    ms = np.zeros(cfg.generations)
    _call(_lib.load().temo_b200_nsga2_run, C.byref(ccfg), _p(x), _p(f), C.byref(done), _p(ms))
    return RunRecord([GenerationRow(t, float(ms[t]), cfg.pop) for t in range(done.value)], x, f)


def rvea_run(prob: ProblemInstance, cfg: RunConfig, mc: MetricContext | None = None) -> RunRecord:
    """reference: rvea_run (algorithms.hpp:227-296). `prob` supplies name/dim/num_obj like the
    reference's ProblemInstance; the evaluator itself runs on the device. With a MetricContext every
    GenerationRow carries igd_value / hv_value of the population, or of the archive with cfg.track_archive
    (fill_metrics, algorithms.hpp:288); RunRecord.archive / archive_f_history as in the reference."""
    cfg = RunConfig(**{**cfg.__dict__, "problem": prob.name, "dim": prob.dim, "obj": prob.num_obj, "horizon": prob.horizon})
    with_metrics = mc is not None and (mc.pf_ref is not None or mc.hv_ref is not None)
    if with_metrics or cfg.track_archive:
        t0 = time.perf_counter()
        rows, history = [], []
        with RveaRun(cfg) as run:
            if cfg.track_archive:
                run.track_archive(cfg.archive_cap)
            if with_metrics:
                run.set_metrics(mc)
            for t in range(cfg.generations):
                pop = run.step()
                g, h = run.metrics() if with_metrics else (float("nan"), float("nan"))
                if cfg.track_archive and cfg.archive_history:
                    history.append(run.archive()[1])
                ms = (time.perf_counter() - t0) * 1e3
                rows.append(GenerationRow(t, ms, pop, g, h))
                if cfg.time_budget_s > 0.0 and ms >= cfg.time_budget_s * 1e3:
                    break
            out = run.download()
            arch = run.archive() if cfg.track_archive else None
        return RunRecord(rows, out["x"], out["f"], arch, history)
    ccfg = cfg.c()
    L = _lib.load()
    H = cfg.lattice_h or lattice_density_for(prob.num_obj, cfg.pop)
    cap = max(cfg.pop, lattice_count(prob.num_obj, H))
    x, f = np.empty((cap, prob.dim)), np.empty((cap, prob.num_obj))
    rows, done = u64(0), u64(0)
    pops = np.zeros(cfg.generations, dtype=np.uint64)
    ms = np.zeros(cfg.generations)
    _call(L.temo_b200_rvea_run, C.byref(ccfg), _p(x), _p(f), C.byref(rows), C.byref(done), _p(pops, u64p), _p(ms))
    rec_rows = [GenerationRow(t, float(ms[t]), int(pops[t])) for t in range(done.value)]
    return RunRecord(rec_rows, x[: rows.value].copy(), f[: rows.value].copy())
