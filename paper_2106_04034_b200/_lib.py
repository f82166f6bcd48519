"""ctypes binding of libgsgp_b200.so (include/gsgp_b200.h).

There is no CPU fallback: `load()` raises if the library is missing, and every
compute entry point fails with GsgpError when no CUDA device is present.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .core import ConfigError, GsgpError

# GSGP_LIB overrides the in-tree build (A/B kernel experiments); either way a
# missing library is an error, never a fallback
LIB_PATH = Path(os.environ.get("GSGP_LIB") or Path(__file__).resolve().parent / "libgsgp_b200.so")

_lock = threading.Lock()
_lib = None

GSGP_OK, GSGP_ERR_CONFIG, GSGP_ERR_CUDA, GSGP_ERR_NCCL, GSGP_ERR_OOM = range(5)

EXPORTS = (
    "gsgp_version", "gsgp_last_error", "gsgp_device_info", "gsgp_set_device", "gsgp_trim_device_memory", "gsgp_rng_draw",
    "gsgp_derive_seed", "gsgp_create_population", "gsgp_compute_semantics", "gsgp_compute_fitness",
    "gsgp_build_mutation_plan", "gsgp_gsm", "gsgp_gsm_step_f32", "gsgp_survive", "gsgp_run",
    "gsgp_comm_unique_id", "gsgp_comm_init", "gsgp_comm_init_host", "gsgp_comm_destroy",
    "gsgp_shard_range",
    "gsgp_sigmoid", "gsgp_argminmax", "gsgp_canonical_sum",
    "gsgp_init", "gsgp_finalize", "gsgp_device_count_in_use", "gsgp_replay",
)


class GsgpConfig(C.Structure):
    _fields_ = [
        ("population_size", C.c_int64), ("random_trees", C.c_int64),
        ("program_size", C.c_int64), ("generations", C.c_int64),
        ("seed", C.c_uint64),
        ("p_function", C.c_double), ("p_feature", C.c_double), ("p_constant", C.c_double),
        ("erc_low", C.c_double), ("erc_high", C.c_double),
        ("mutation_step_uniform", C.c_int32), ("gsm_sign", C.c_int32),
        ("mutation_step", C.c_double), ("division_eps", C.c_double),
        ("storage_f64", C.c_int32), ("use_graph", C.c_int32),
        ("time_kernels", C.c_int32), ("virtual_shards", C.c_int32),
        ("window_start", C.c_int64),
    ]


class GsgpOutputs(C.Structure):
    _fields_ = [
        ("train_trace", C.c_void_p), ("test_trace", C.c_void_p),
        ("elite_src", C.c_void_p), ("elite_idx", C.c_void_p), ("elite_slot", C.c_void_p),
        ("elite_fit", C.c_void_p),
        ("plan_u", C.c_void_p), ("plan_v", C.c_void_p), ("plan_ms", C.c_void_p),
        ("elite_train_semantics", C.c_void_p),
        ("gsm_ms", C.c_void_p),
        ("overflow", C.c_int64),
        ("shard_train_lo", C.c_int64), ("shard_train_hi", C.c_int64),
        ("stage_ms", C.c_double * 20),
        ("storage_f64_used", C.c_int64),
        ("interp_info", C.c_int64 * 4),
        ("interp_div", C.c_int64 * 2),
        ("interp_ops", C.c_int64 * 6),
    ]


P = C.c_void_p
I64 = C.c_int64
U64 = C.c_uint64
I32 = C.c_int32
D = C.c_double

_SIGS = {
    "gsgp_version": (C.c_char_p, []),
    "gsgp_last_error": (C.c_char_p, []),
    "gsgp_device_info": (C.c_int, [P, P, C.c_char_p, C.c_int]),
    "gsgp_set_device": (C.c_int, [C.c_int]),
    "gsgp_trim_device_memory": (C.c_int, []),
    "gsgp_rng_draw": (C.c_int, [U64, U64, P, I64, P, P]),
    "gsgp_derive_seed": (U64, [U64, U64]),
    "gsgp_create_population": (C.c_int, [C.POINTER(GsgpConfig), I64, U64, I32, P, P, P]),
    "gsgp_compute_semantics": (C.c_int, [P, P, P, I64, I64, P, I64, I32, D, I32, P, P]),
    "gsgp_compute_fitness": (C.c_int, [P, P, I64, I64, P]),
    "gsgp_build_mutation_plan": (C.c_int, [I64, I64, U64, I64, I32, D, P, P, P]),
    "gsgp_gsm": (C.c_int, [P, I64, I64, P, I64, P, P, P, I32, I32, P, P]),
    "gsgp_gsm_step_f32": (C.c_int, [P, P, P, P, I64, I64, I64, I64, P, P, P, P, P, I32, P, P, P, P]),
    "gsgp_survive": (C.c_int, [P, P, I64, P]),
    "gsgp_run": (C.c_int, [C.POINTER(GsgpConfig), P, P, I64, P, P, I64, I32, C.POINTER(GsgpOutputs)]),
    "gsgp_comm_unique_id": (C.c_int, [P]),
    "gsgp_comm_init": (C.c_int, [C.c_int, C.c_int, P]),
    "gsgp_comm_init_host": (C.c_int, [C.c_int, C.c_int, P]),
    "gsgp_comm_destroy": (C.c_int, []),
    "gsgp_shard_range": (None, [I64, I64, I64, P, P]),
    "gsgp_sigmoid": (C.c_int, [P, I64, P]),
    "gsgp_argminmax": (C.c_int, [P, I64, P]),
    "gsgp_canonical_sum": (C.c_int, [P, I64, I64, I32, P]),
    "gsgp_init": (C.c_int, [C.c_int, P]),
    "gsgp_replay": (C.c_int, [P, I64, I64, P, I64, I64, P, P, P, P, P, P, I64, I32, P]),
    "gsgp_finalize": (C.c_int, []),
    "gsgp_device_count_in_use": (C.c_int, []),
}


def load():
    """Load (once) and return the CUDA library; raise loudly if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise GsgpError(
                    f"CUDA engine library missing: {LIB_PATH} "
                    "(build it with `python -m paper_2106_04034_b200.build`); "
                    "there is no CPU fallback")
            lib = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == GSGP_OK:
        return
    msg = load().gsgp_last_error().decode(errors="replace")
    if rc == GSGP_ERR_CONFIG:
        raise ConfigError(msg)
    raise GsgpError(f"[gsgp_b200 error {rc}] {msg}")


def ptr(a: np.ndarray | None):
    """Raw data pointer of a C-contiguous array (None -> NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays passed to the C ABI must be C-contiguous"
    return a.ctypes.data


def u64(x: int) -> int:
    """Python int seed/stream -> its 64-bit two's-complement word (rng.py:33)."""
    return int(x) & ((1 << 64) - 1)
