"""B200-native TensorRVEA generation loop (sm_100a CUDA behind a C ABI).

The product is paper_2404_01159_b200/libtemo_b200.so (sources in csrc/, ABI in
include/temo_b200.h). `api` mirrors the reference's operator/problem/selection/algorithm
interface on numpy tensors; `dist` holds the multi-GPU host orchestration.
"""
from . import _lib  # noqa: F401
from .api import *  # noqa: F401,F403
