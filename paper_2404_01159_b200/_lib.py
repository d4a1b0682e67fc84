"""ctypes loader for libtemo_b200.so (the C ABI declared in include/temo_b200.h).

The shared library is the product; this module only binds it. There is no Python or CPU
fallback: if the library is missing, or no CUDA device is visible when a compute entry point
is called, the call fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# TEMO_B200_LIB: developer override used to A/B differently compiled builds of the same library
LIB_PATH = os.environ.get("TEMO_B200_LIB") or os.path.join(HERE, "libtemo_b200.so")

u64 = C.c_uint64
f64p = C.POINTER(C.c_double)
u64p = C.POINTER(C.c_uint64)
u8p = C.POINTER(C.c_ubyte)


class GaParamsC(C.Structure):
    _fields_ = [("pc", C.c_double), ("eta", C.c_double), ("pm", C.c_double), ("xi", C.c_double)]


class OpParamsC(C.Structure):
    _fields_ = [("de_f", C.c_double), ("de_cr", C.c_double), ("pso_inertia", C.c_double), ("pso_c1", C.c_double),
                ("pso_c2", C.c_double), ("cso_phi", C.c_double)]


class RunConfigC(C.Structure):
    _fields_ = [
        ("problem", C.c_int32), ("rng_mode", C.c_int32),
        ("pop", u64), ("lattice_h", u64), ("generations", u64), ("seed", u64), ("dim", u64), ("obj", u64),
        ("alpha", C.c_double), ("fr", C.c_double), ("time_budget_s", C.c_double),
        ("ga", GaParamsC), ("fuse_eval", C.c_int32), ("op", C.c_int32), ("opp", OpParamsC),
        ("horizon", u64),
    ]


class TemoB200Error(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"temo_b200 error {code}: {msg}")
        self.code = code


# Every symbol include/temo_b200.h declares: (restype, argtypes). tests/test_cabi.py checks that
# this table and the header agree and that the .so exports each of them.
_GA = C.POINTER(GaParamsC)
_CFG = C.POINTER(RunConfigC)
_RUN = C.c_void_p
SIGNATURES = {
    "temo_b200_last_error": (C.c_char_p, []),
    "temo_b200_version": (C.c_char_p, []),
    "temo_b200_device_count": (C.c_int, []),
    "temo_b200_init": (C.c_int, [C.c_int]),
    "temo_b200_default_run_config": (None, [_CFG]),
    "temo_b200_default_ga_params": (None, [_GA]),
    "temo_b200_uniform_tensor": (C.c_int, [u64, u64p, u64, u64, C.c_int, f64p]),
    "temo_b200_shuffle_indices": (C.c_int, [u64, u64p, u64, u64p]),
    "temo_b200_parent_pool_indices": (C.c_int, [u64, u64, u64, u64p, u64p]),
    "temo_b200_sbx": (C.c_int, [f64p, u64, u64, u64, u64p, _GA, f64p, f64p, C.c_int, f64p]),
    "temo_b200_polynomial_mutation": (C.c_int, [f64p, u64, u64, u64, u64p, _GA, f64p, f64p, C.c_int, f64p]),
    "temo_b200_ga_reproduce": (C.c_int, [f64p, u64, u64, u64, u64p, _GA, f64p, f64p, C.c_int, f64p]),
    "temo_b200_random_reproduce": (C.c_int, [u64, u64, u64, u64p, f64p, f64p, C.c_int, f64p]),
    "temo_b200_de_reproduce": (C.c_int, [f64p, u64, u64, u64, u64p, C.c_double, C.c_double, f64p, f64p, C.c_int, f64p, f64p]),
    "temo_b200_pso_reproduce": (C.c_int, [f64p, f64p, u64, u64, u64, u64p, C.c_double, C.c_double, C.c_double, f64p, f64p, f64p,
                                          f64p, f64p, C.c_int, f64p, f64p]),
    "temo_b200_cso_reproduce": (C.c_int, [f64p, f64p, u64, u64, u64, u64p, C.c_double, f64p, f64p, f64p, C.c_int, f64p, f64p]),
    "temo_b200_evaluate": (C.c_int, [C.c_int, f64p, u64, u64, u64, f64p]),
    "temo_b200_evaluate_h": (C.c_int, [C.c_int, f64p, u64, u64, u64, u64, f64p]),
    "temo_b200_env_rollout": (C.c_int, [f64p, u64, u64, u64, u64, u64, f64p]),
    "temo_b200_mlp_forward": (C.c_int, [f64p, u64, u64, u64, f64p, f64p]),
    "temo_b200_problem_bounds": (C.c_int, [C.c_int, u64, u64, f64p, f64p]),
    "temo_b200_problem_default_dim": (u64, [C.c_int, u64]),
    "temo_b200_lattice_count": (u64, [u64, u64]),
    "temo_b200_lattice_density_for": (u64, [u64, u64]),
    "temo_b200_simplex_lattice": (C.c_int, [u64, u64, f64p]),
    "temo_b200_make_ref_set": (C.c_int, [u64, u64, f64p, f64p]),
    "temo_b200_min_vector_angles": (C.c_int, [f64p, u64, u64, f64p]),
    "temo_b200_adapt": (C.c_int, [f64p, f64p, f64p, u64, u64, f64p, f64p]),
    "temo_b200_rv_select": (C.c_int, [f64p, u64, u64, f64p, f64p, u64, u64, u64, C.c_double, u64p, u64p, u8p,
                                      u64p, f64p, f64p]),
    "temo_b200_apd_penalty": (C.c_double, [u64, u64, u64, C.c_double]),
    "temo_b200_nondominated_sort": (C.c_int, [f64p, u64, u64, u64p]),
    "temo_b200_nsga2_select": (C.c_int, [f64p, u64, u64, u64, u64p]),
    "temo_b200_nsga2_create": (C.c_int, [_CFG, C.POINTER(_RUN)]),
    "temo_b200_nsga2_step": (C.c_int, [_RUN, f64p]),
    "temo_b200_nsga2_inject": (C.c_int, [_RUN, f64p, f64p, u64, u64]),
    "temo_b200_nsga2_state": (C.c_int, [_RUN, u64p, u64p, u64p]),
    "temo_b200_nsga2_download": (C.c_int, [_RUN, f64p, f64p]),
    "temo_b200_nsga2_last_generation": (C.c_int, [_RUN, f64p, f64p, u64p, u64p]),
    "temo_b200_nsga2_destroy": (C.c_int, [_RUN]),
    "temo_b200_nsga2_run": (C.c_int, [_CFG, f64p, f64p, u64p, f64p]),
    "temo_b200_igd": (C.c_int, [f64p, u64, u64, f64p, u64, f64p]),
    "temo_b200_hv_mc_box": (C.c_int, [f64p, u64, u64, f64p, f64p, u64, u64, f64p, f64p]),
    "temo_b200_hv_mc": (C.c_int, [f64p, u64, u64, f64p, u64, u64, f64p, f64p]),
    "temo_b200_archive_insert": (C.c_int, [f64p, f64p, u64, f64p, f64p, u64, u64, u64, u64, f64p, f64p, u64p]),
    "temo_b200_crowding_distance": (C.c_int, [f64p, u64, u64, f64p]),
    "temo_b200_run_set_metrics": (C.c_int, [_RUN, f64p, u64, f64p, C.c_double, u64, u64, C.c_int]),
    "temo_b200_run_metrics": (C.c_int, [_RUN, f64p, f64p]),
    "temo_b200_run_track_archive": (C.c_int, [_RUN, u64]),
    "temo_b200_run_archive_rows": (C.c_int, [_RUN, u64p]),
    "temo_b200_run_archive": (C.c_int, [_RUN, f64p, f64p]),
    "temo_b200_run_create": (C.c_int, [_CFG, C.POINTER(_RUN)]),
    "temo_b200_run_step": (C.c_int, [_RUN, u64p, f64p]),
    "temo_b200_run_step_injected": (C.c_int, [_RUN, f64p, u64p]),
    "temo_b200_run_inject": (C.c_int, [_RUN, u64, f64p, f64p, f64p, f64p, u64, u64]),
    "temo_b200_run_state": (C.c_int, [_RUN, u64p, u64p, u64p, u64p, u64p, u64p]),
    "temo_b200_run_download": (C.c_int, [_RUN, f64p, f64p, f64p, f64p]),
    "temo_b200_run_last_generation": (C.c_int, [_RUN, f64p, f64p, u64p]),
    "temo_b200_run_timings": (C.c_int, [_RUN, f64p]),
    "temo_b200_run_timing_history": (C.c_int, [_RUN, f64p, C.c_uint64, C.c_int, C.POINTER(C.c_uint64)]),
    "temo_b200_run_destroy": (C.c_int, [_RUN]),
    "temo_b200_rvea_run": (C.c_int, [_CFG, f64p, f64p, u64p, u64p, u64p, f64p]),
    "temo_b200_dev_alloc": (C.c_void_p, [C.c_size_t]),
    "temo_b200_dev_free": (C.c_int, [C.c_void_p]),
    "temo_b200_host_alloc": (C.c_void_p, [C.c_size_t]),
    "temo_b200_host_free": (C.c_int, [C.c_void_p]),
    "temo_b200_dev_upload": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
    "temo_b200_dev_download": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
    "temo_b200_dev_sync": (C.c_int, []),
    "temo_b200_run_time_stage": (C.c_int, [_RUN, C.c_int, C.c_int, f64p]),
    "temo_b200_shard_last_error": (C.c_char_p, []),
    "temo_b200_shard_create": (C.c_int, [_CFG, C.c_int, C.c_int, C.POINTER(_RUN)]),
    "temo_b200_shard_destroy": (C.c_int, [_RUN]),
    "temo_b200_shard_info": (C.c_int, [_RUN, u64p]),
    "temo_b200_shard_state": (C.c_int, [_RUN, u64p]),
    "temo_b200_shard_buffer": (C.c_void_p, [_RUN, C.c_int]),
    "temo_b200_shard_stream": (C.c_void_p, [_RUN]),
    "temo_b200_shard_ipc_handle": (C.c_int, [_RUN, C.POINTER(C.c_ubyte)]),
    "temo_b200_shard_open_peers": (C.c_int, [_RUN, C.POINTER(C.c_ubyte)]),
    "temo_b200_shard_set_peer_pointers": (C.c_int, [_RUN, C.POINTER(C.c_void_p)]),
    "temo_b200_shard_begin": (C.c_int, [_RUN]),
    "temo_b200_shard_reproduce": (C.c_int, [_RUN]),
    "temo_b200_shard_place_initial_f": (C.c_int, [_RUN]),
    "temo_b200_shard_select_local": (C.c_int, [_RUN]),
    "temo_b200_shard_select_rows": (C.c_int, [_RUN]),
    "temo_b200_shard_finish": (C.c_int, [_RUN, u64p]),
    "temo_b200_shard_download": (C.c_int, [_RUN, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), u64p, u64p, f64p, f64p, f64p, f64p]),
    "temo_b200_pow": (C.c_int, [f64p, f64p, u64, f64p, C.c_int]),
    "temo_b200_tanh": (C.c_int, [f64p, u64, f64p, C.c_int]),
    "temo_b200_flush_l2": (C.c_int, []),
    "temo_b200_set_option": (C.c_int, [C.c_char_p, C.c_long]),
}

_lib = None


def load():
    """Loads libtemo_b200.so; raises if it has not been built (python -c 'import __graft_entry__ as g; g.build()')."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2404_01159_b200/csrc` "
            "(there is no CPU fallback for the temo_b200 path)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc):
    if rc != 0:
        raise TemoB200Error(rc, load().temo_b200_last_error().decode(errors="replace"))
