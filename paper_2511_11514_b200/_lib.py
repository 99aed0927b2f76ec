"""ctypes binding of libflowcover_b200.so (the C ABI in include/flowcover_b200.h).

The shared library is the only compute path: there is no CPU fallback.  If it
is missing or cannot be loaded, every entry point raises
NativeLibraryError instead of silently running something else.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# FCB_LIB_PATH selects an alternative build of the same library (tuning runs)
LIB_PATH = os.environ.get("FCB_LIB_PATH") or os.path.join(_HERE, "libflowcover_b200.so")

# status codes (include/flowcover_b200.h)
FCB_OK = 0
FCB_EINPUT = 1
FCB_EFLOW = 2
FCB_EROLLOUT = 3
FCB_ERICCATI = 4
FCB_ECUDA = 5
FCB_ENOTSUP = 6
FCB_EWORKSPACE = 7

FCB_FP32 = 0
FCB_FP64 = 1

FCB_MODEL_SINGLE_INTEGRATOR_2D = 0
FCB_MODEL_DIFF_DRIVE = 1
FCB_MODEL_AIRCRAFT_3D = 2
FCB_MODEL_DOUBLE_INTEGRATOR_2D = 3
FCB_MODEL_LTI = 4

FCB_OT_ASYM = 0
FCB_OT_SYM = 1
FCB_OT_SWEEP = 2

STATE_STOP, STATE_STAGE, STATE_ITER, STATE_INDEX, STATE_FLOWS, STATE_UPDATES = range(6)


class NativeLibraryError(RuntimeError):
    """libflowcover_b200.so is missing, failed to load, or a CUDA call failed."""


_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_Z = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/flowcover_b200.h exactly
SIGNATURES: dict[str, tuple] = {
    "fcb_version": (ctypes.c_char_p, []),
    "fcb_last_error": (ctypes.c_char_p, []),
    "fcb_launch_count": (ctypes.c_longlong, []),
    "fcb_last_kernel": (ctypes.c_char_p, []),
    "fcb_device_info": (_I, [_P, _P, _P]),
    "fcb_omega_workspace_bytes": (_Z, [_I, _I]),
    "fcb_resolve_omega": (_I, [_I, _P, _I, _P, _I, _I, _D, _P, _P, _Z, _P]),
    "fcb_ot_workspace_bytes": (_Z, [_I, _I, _I, _I, _I]),
    "fcb_ot_solve": (
        _I,
        [_I, _I, _P, _I, _P, _I, _I, _P, _I, _D, _P, _P, _P, _P, _P, _P, _P, _P, _Z, _P],
    ),
    "fcb_ot_cost": (_I, [_I, _P, _P, _I, _P, _I, _P, _P]),
    "fcb_ot_plan": (_I, [_P, _I, _P, _I, _I, _P, _P, _P, _P, _P]),
    "fcb_sinkhorn_flow_workspace_bytes": (_Z, [_I, _I, _I, _I]),
    "fcb_sinkhorn_flow": (
        _I,
        [_I, _P, _I, _P, _I, _I, _D, _I, _D, _P, _P, _P, _P, _P, _P, _I, _P, _D, _P, _Z, _P],
    ),
    "fcb_sinkhorn_divergence_workspace_bytes": (_Z, [_I, _I, _I, _I]),
    "fcb_sinkhorn_divergence": (_I, [_I, _P, _I, _P, _I, _I, _D, _I, _D, _P, _P, _P, _Z, _P]),
    "fcb_sinkhorn_divergence_cached": (_I, [_I, _P, _I, _P, _I, _I, _D, _I, _D, _P, _P, _P, _P, _Z,
                                            _P]),
    "fcb_gmm_eval": (_I, [_P, _I, _I, _I, _P, _P, _P, _P, _P]),
    "fcb_gather_rows": (_I, [_P, _I, _I, _P, _I, _P, _P, _P]),
    "fcb_median_workspace_bytes": (_Z, [_I]),
    "fcb_median_bandwidth": (_I, [_P, _I, _I, _D, _P, _P, _P, _Z, _P]),
    "fcb_stein_workspace_bytes": (_Z, [_I, _I, _I]),
    "fcb_stein_flow": (_I, [_I, _P, _I, _I, _P, _P, _P, _P, _P, _Z, _P]),
    "fcb_stein_flow_full_workspace_bytes": (_Z, [_I, _I, _I]),
    "fcb_stein_flow_full": (
        _I,
        [_I, _P, _I, _I, _I, _P, _D, _D, _P, _P, _P, _I, _P, _D, _P, _Z, _P],
    ),
    "fcb_rollout_workspace_bytes": (_Z, [_I, _I]),
    "fcb_rollout": (_I, [_I, _I, _I, _P, _P, _P, _I, _D, _P, _I, _P, _P, _P, _P, _I, _I, _P, _P]),
    "fcb_linearize": (_I, [_I, _I, _I, _P, _P, _P, _I, _P, _P, _P]),
    "fcb_lqr_workspace_bytes": (_Z, [_I, _I, _I]),
    "fcb_lqr_solve": (
        _I,
        [_I, _I, _I, _D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    ),
    "fcb_plan_update_workspace_bytes": (_Z, [_I, _I, _I]),
    "fcb_plan_update": (
        _I,
        [_I, _I, _I, _P, _P, _P, _I, _D, _I, _P, _P, _P, _P, _D, _P, _P, _P, _P, _I, _I, _P, _Z,
         _P],
    ),
    "fcb_plan_fused_workspace_bytes": (_Z, [_I, _I, _I, _I, _I]),
    "fcb_plan_fused": (
        _I,
        [_I, _I, _I, _P, _P, _P, _P, _P, _P, _I, _D, _I, _P, _P, _P, _P, _P, _D, _P, _P, _I, _D,
         _I, _D, _D, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _Z, _P],
    ),
    "fcb_plan_fused_stein_workspace_bytes": (_Z, [_I, _I, _I]),
    "fcb_plan_fused_stein": (
        _I,
        [_I, _I, _I, _P, _P, _P, _P, _P, _P, _I, _D, _I, _P, _P, _P, _P, _P, _D, _P, _I, _P, _D,
         _D, _D, _P, _P, _P, _P, _P, _I, _I, _P, _P, _Z, _P],
    ),
    "fcb_point_sums": (_I, [_P, _I, _I, _P, _P]),
    "fcb_lse_sweep_workspace_bytes": (_Z, [_I, _I, _I, _I]),
    "fcb_lse_sweep": (_I, [_I, _P, _I, _P, _I, _I, _P, _P, _P, _D, _D, _D, _P, _P, _P, _P, _Z,
                           _P]),
    "fcb_shard_init": (_I, [_I, _P, _I, _I, _P, _D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "fcb_shard_cross_merge": (
        _I, [_I, _I, _I, _P, _P, _D, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "fcb_shard_self_rows": (_I, [_I, _I, _I, _I, _P, _P, _P, _P, _P, _P]),
    "fcb_shard_self_commit": (
        _I, [_I, _I, _I, _I, _P, _D, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "fcb_shard_finish_workspace_bytes": (_Z, [_I]),
    "fcb_shard_flow_finish": (
        _I,
        [_P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I,
         _P, _D, _P, _P, _Z, _P],
    ),
    "fcb_stein_partial_workspace_bytes": (_Z, [_I, _I, _I, _I]),
    "fcb_stein_partial": (_I, [_I, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _Z, _P]),
    "fcb_median_tiles": (ctypes.c_longlong, [_I]),
    "fcb_median_hist_offset": (_Z, []),
    "fcb_median_shard_init": (_I, [_I, _P, _Z, _P, _P]),
    "fcb_median_shard_pass": (_I, [_P, _I, _I, _I, ctypes.c_longlong,
                                   ctypes.c_longlong, _P, _P, _P]),
    "fcb_median_shard_select": (_I, [_I, _I, _P, _P, _P]),
    "fcb_median_shard_finish": (_I, [_I, _D, _P, _P, _P, _P]),
    "fcb_stein_combine_workspace_bytes": (_Z, [_I]),
    "fcb_stein_combine": (_I, [_P, _I, _I, _I, _P, _P, _P, _P, _P, _I, _P, _D, _P, _Z, _P]),
    "fcb_tsp_tours": (_I, [_P, _I, _I, _I, _P, _I, _P, _P, _P]),
    "fcb_peak_probe": (_I, [_I, _I, _P, _P]),
    "fcb_debug_timeline": (_I, [_P, _I]),
    "fcb_debug_careful_items": (ctypes.c_longlong, []),
    "fcb_debug_careful_rows_resident": (ctypes.c_longlong, []),
}

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load the native library once; raise NativeLibraryError if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not found; build it with `python __graft_entry__.py build` "
                "(make -C paper_2511_11514_b200/csrc)"
            )
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:  # pragma: no cover - depends on the host
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().fcb_last_error()
    return msg.decode() if msg else ""


def launch_count() -> int:
    return int(load().fcb_launch_count())


def last_kernel() -> str:
    """Name of the last kernel this library launched (path checks in tests)."""
    return load().fcb_last_kernel().decode()


def check(rc: int, what: str, input_error: type = ValueError) -> None:
    """Map a C status code to the reference's exception types."""
    if rc == FCB_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == FCB_EINPUT:
        raise input_error(msg)
    if rc == FCB_ENOTSUP:
        raise NotImplementedError(msg)
    raise NativeLibraryError(msg)


def call(name: str, *args, what: str | None = None, input_error: type = ValueError) -> None:
    rc = getattr(load(), name)(*args)
    check(rc, what or name, input_error)
