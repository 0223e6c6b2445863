"""ctypes binding of the sm_100a C-ABI library (include/dice_b200.h).

The product path has no fallback: if ``_dice_b200.so`` is missing or cannot be
loaded, every op raises ``NativeLibraryError`` instead of computing anything
elsewhere.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import (ConfigurationError, ContractError, NativeLibraryError, NumericsError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_dice_b200.so")
# experiment builds (tools/*_probe.py): another build of the same library
LIB_PATH = os.environ.get("DICE_LIB_PATH", LIB_PATH)

c_void_p, c_int, c_int64, c_uint64, c_double, c_float = (
    ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double,
    ctypes.c_float)
P = c_void_p

# name -> (restype, argtypes); mirrors include/dice_b200.h
SIGNATURES = {
    "dice_version": (c_int, []),
    "dice_event_create": (c_int, [ctypes.POINTER(c_void_p)]),
    "dice_event_destroy": (c_int, [P]),
    "dice_event_record": (c_int, [P, P]),
    "dice_event_elapsed_ms": (c_int, [P, P, ctypes.POINTER(c_float)]),
    "dice_status_reset": (c_int, [P, P]),
    "dice_splitmix_fill": (c_int, [c_uint64, c_uint64, c_int64, c_int64, c_double, c_int, c_int,
                                   P, c_int64, P]),
    "dice_splitmix_bits": (c_int, [c_uint64, c_uint64, c_int64, P, P]),
    "dice_gate_topk": (c_int, [P, P, c_int64, c_int, c_int, c_int, P, P, P, P, c_int, c_int, P]),
    "dice_gate_topk_decide": (c_int, [P, P, c_int64, c_int, c_int, c_int, P, P, P, P, c_int, c_int,
                                      c_int, c_int, c_int, c_int, c_uint64, P, P, P, P, P, P, P]),
    "dice_expert_gemm1_with_dense": (c_int, [P, c_int64, c_int64, P, c_int, c_int, c_int, P, P, P,
                                             c_int64, P, c_int, P, P]),
    "dice_gate_route_state_words": (c_int64, [c_int64]),
    "dice_gate_route": (c_int, [P, P, c_int64, c_int, c_int, c_int, P, P, P, P, c_int, c_int,
                                c_int, c_int, c_int, c_int, c_int, c_uint64, P, P, P, P, P, P,
                                P, c_int64, P, P, P, P, c_int, c_int64, P, P]),
    "dice_expert_gemm2": (c_int, [P, c_int64, P, c_int, c_int, c_int, P, P, P]),
    "dice_cond_decide": (c_int, [P, c_int64, c_int, c_int, c_int, c_int, c_int, c_int, c_uint64,
                                 P, P, P, P, P, P, P]),
    "dice_route_permute": (c_int, [P, P, c_int64, c_int, c_int, P, c_int, P, c_int64, P, P, P,
                                   c_int, c_int64, c_int64, P, P, P]),
    "dice_permute_max_rows": (c_int64, [c_int64, c_int, c_int]),
    "dice_permute_scratch_ints": (c_int64, [c_int64, c_int, c_int]),
    "dice_grouped_ffn": (c_int, [P, c_int64, P, P, c_int, c_int, c_int, P, P, P, P]),
    "dice_cache_assemble": (c_int, [P, P, P, P, P, P, c_int64, c_int, c_int, P, P, P, P, P, P, P]),
    "dice_gemm": (c_int, [c_int, P, c_int64, P, c_int, c_int, P, c_int64, P, c_int64, P, c_int64,
                          P]),
    "dice_expert_gemm2_pairs": (c_int, [P, c_int64, P, c_int, c_int, c_int, P, P, c_int64, P, P,
                                        c_int, c_int64, P, P, P, P]),
    "dice_gemm_consume": (c_int, [P, c_int64, P, c_int, c_int, P, c_int64, P, P, c_int, P,
                                  c_int64, P, c_int64, P]),
    "dice_consume_rows": (c_int, [P, P, P, c_int64, c_int, c_int, P, P, P]),
    "dice_combine": (c_int, [P, P, P, P, c_int64, c_int, c_int, P, P, P]),
    "dice_denoise": (c_int, [P, P, P, c_float, c_int64, c_int, P, c_int, P]),
    "dice_similarity_partial_words": (c_int64, []),
    "dice_step_similarity": (c_int, [P, P, c_int64, c_int, c_int64, c_int64, P, c_int64, P, c_int,
                                     c_int, P, P, P]),
    "dice_pack_rows": (c_int, [P, c_int64, c_int, c_int64, c_int, P, P, P]),
    "dice_device_alloc": (c_int, [c_int64, ctypes.POINTER(c_void_p)]),
    "dice_device_free": (c_int, [P]),
    "dice_ipc_get_handle": (c_int, [P, ctypes.c_char_p]),
    "dice_ipc_open": (c_int, [ctypes.c_char_p, ctypes.POINTER(c_void_p)]),
    "dice_ipc_close": (c_int, [P]),
    "dice_stream_wait_eq": (c_int, [ctypes.POINTER(c_uint64), c_int, ctypes.c_uint32, P]),
    "dice_stream_write": (c_int, [ctypes.POINTER(c_uint64), c_int, ctypes.c_uint32, P]),
    "dice_ep_dispatch": (c_int, [P, P, P, c_int64, c_int, c_int, c_int, c_int, P, c_int, P, P, P,
                                 c_int64, c_int64, P, ctypes.POINTER(c_uint64),
                                 ctypes.POINTER(c_uint64), ctypes.POINTER(c_uint64), P]),
    "dice_ep_expert": (c_int, [P, P, P, c_int, c_int64, c_int, c_int, c_int, c_int, P, P, P, P, P,
                               P, P, c_int64, P, P, ctypes.POINTER(c_uint64),
                               ctypes.POINTER(c_uint64), ctypes.POINTER(c_uint64),
                               ctypes.POINTER(c_int64), P, c_int64, P, c_int, P, P]),
    "dice_ep_regroup": (c_int, [P, P, P, c_int, c_int64, c_int, c_int, P, P, P, P, P, P, P]),
    "dice_ep_expert_ffn": (c_int, [P, c_int64, P, c_int64, c_int, c_int, c_int, c_int, c_int, P,
                                   P, P, P, P, ctypes.POINTER(c_uint64),
                                   ctypes.POINTER(c_uint64), ctypes.POINTER(c_uint64),
                                   ctypes.POINTER(c_int64), P, c_int64, P, c_int, P, P]),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load the CUDA library once; raise NativeLibraryError when unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not built; run `python build.py` (nvcc, sm_100a). There is no "
                "CPU fallback.")
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:  # pragma: no cover - depends on the box
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


_ERRORS = {1: ContractError, 2: ConfigurationError, 3: NumericsError}


def check(rc: int, what: str) -> None:
    """Map a DICE_ERR_* code onto the reference exception types (errors.py:4-29)."""
    if rc == 0:
        return
    exc = _ERRORS.get(rc)
    if exc is None:
        raise NativeLibraryError(f"{what}: CUDA failure (code {rc})")
    raise exc(f"{what}: rejected by the CUDA library (code {rc})")


# kernels each entry point launches (for the bench's gpu_launches count)
KERNELS_PER_CALL = {"dice_route_permute": 3, "dice_gate_route_state_words": 0,
                    "dice_grouped_ffn": 2, "dice_event_create": 0, "dice_event_destroy": 0,
                    "dice_event_record": 0, "dice_event_elapsed_ms": 0,
                    "dice_permute_max_rows": 0, "dice_permute_scratch_ints": 0,
                    "dice_device_alloc": 0, "dice_device_free": 0, "dice_ipc_get_handle": 0,
                    "dice_ipc_open": 0, "dice_ipc_close": 0, "dice_stream_wait_eq": 0,
                    "dice_stream_write": 0, "dice_version": 0,
                    "dice_similarity_partial_words": 0, "dice_step_similarity": 2,
                    # count + scatter + send
                    "dice_ep_dispatch": 3,
                    # receive ids + count + scatter + gather + GEMM1 + GEMM2 (the
                    # combine's peer stores ride in the GEMM2 epilogue)
                    "dice_ep_expert": 6,
                    "dice_ep_regroup": 4, "dice_ep_expert_ffn": 2}
launch_count = [0]


def call(name: str, *args):
    rc = getattr(load(), name)(*args)
    check(rc, name)
    launch_count[0] += KERNELS_PER_CALL.get(name, 1)
    return rc
