"""ctypes binding of the C-ABI in include/lmg.h (liblmg.so, built in-tree for sm_100a).

There is no CPU fallback: if the library or a CUDA device is missing every compute call raises.
torch is used only for device memory and the current stream (plumbing); the .so itself has no
torch types in its signatures.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ConfigurationError, DimensionError, LmgCudaError, ProtocolError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblmg.so")

LMG_OK, LMG_ERR_DIMENSION, LMG_ERR_CONFIGURATION, LMG_ERR_PROTOCOL, LMG_ERR_CUDA = range(5)
ACT = {"relu": 0, "tanh": 1, "identity": 2}
SRC_DENSE, SRC_HEAD = 0, 1
DENSE, DENSE_ADJOINT, CONV, CONV_ADJOINT = range(4)

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int32_p = ctypes.POINTER(ctypes.c_int32)


class LmgSystem(ctypes.Structure):
    """struct lmg_system (include/lmg.h)."""

    _fields_ = [
        ("num_layers", ctypes.c_int32),
        ("width", ctypes.c_int32),
        ("kind", ctypes.c_int32),
        ("act", ctypes.c_int32),
        ("step", ctypes.c_double),
        ("W", ctypes.c_void_p),
        ("w_stride", ctypes.c_int64),
        ("b", ctypes.c_void_p),
        ("b_stride", ctypes.c_int64),
        ("D", ctypes.c_void_p),
        ("d_stride", ctypes.c_int64),
        ("channels", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("px_width", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


# name -> (restype, argtypes)
_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_SYS = ctypes.POINTER(LmgSystem)
SIGNATURES = {
    "lmg_abi_version": (_I, []),
    "lmg_last_error": (ctypes.c_char_p, []),
    "lmg_launch_count": (ctypes.c_ulonglong, []),
    "lmg_timing_enable": (_I, [_I]),
    "lmg_route_counts": (_I, [ctypes.POINTER(ctypes.c_ulonglong), _I]),
    "lmg_set_canonical_order": (_I, [_I]),
    "lmg_debug_sweep_trace": (_I, [_P]),
    "lmg_debug_sweep_clusters": (_I, [_I, _I, _I]),
    "lmg_timing_read": (_I, [_I, c_double_p, c_double_p, c_double_p,
                             ctypes.POINTER(ctypes.c_ulonglong)]),
    "lmg_propagate": (_I, [_SYS, _I, _P, _P, _I, _I, _I, _P, _P]),
    "lmg_sequential_forward": (_I, [_SYS, _I, _P, _I, _P, _P]),
    "lmg_propagation_operator": (_I, [_SYS, _I, _P, _P, _P]),
    "lmg_residual_workspace": (ctypes.c_size_t, [_SYS, _I]),
    "lmg_compute_residual": (_I, [_SYS, _I, _P, _P, _I, _P, _P, _P, _P]),
    "lmg_restrict": (_I, [_P, _I, _I, _I, _I, _P, _P]),
    "lmg_assemble_coarse_source": (_I, [_SYS, _I, _P, _P, _P, _P]),
    "lmg_f_relax": (_I, [_SYS, _I, _I, _P, _P, _I, _P]),
    "lmg_c_relax": (_I, [_SYS, _I, _I, _P, _P, _I, _P]),
    "lmg_fcf_relax": (_I, [_SYS, _I, _I, _P, _P, _I, _P]),
    "lmg_num_levels": (_I, [_I, _I, _I, ctypes.POINTER(ctypes.c_int)]),
    "lmg_solver_workspace": (ctypes.c_size_t, [_SYS, _I, _I, _I]),
    "lmg_mg_cycle": (_I, [_SYS, _I, _I, _I, _P, _P, _I, _P, _P, ctypes.c_size_t, _P]),
    "lmg_solve": (_I, [_SYS, _I, _I, _I, _P, _P, _I, _I, _D, _I, c_double_p, c_int32_p,
                       c_int32_p, _P, ctypes.c_size_t, _P]),
    "lmg_act_deriv": (_I, [_SYS, _I, _P, _P, _P]),
    "lmg_param_grads": (_I, [_SYS, _I, _P, _P, _P, _D, _D, _P, _P, _P]),
    "lmg_param_grads_ex": (_I, [_SYS, _I, _P, _P, _P, _D, _D, _P, _P, _I, _P]),
    "lmg_local_fcf_a": (_I, [_SYS, _I, _I, _P, _P, _I, _I, _I, _P, _P]),
    "lmg_local_fcf_b": (_I, [_SYS, _I, _I, _P, _P, _I, _P, _I, _P, _P, _P]),
    "lmg_local_fcf_fused_ok": (_I, [_SYS, _I, _I, _I, _I]),
    "lmg_local_fcf_fused": (_I, [_SYS, _I, _I, _P, _P, _I, _I, _I, _P, _P, _P, _P, _I, _P, _P]),
    "lmg_halo_finish": (_I, [_P, _P, _P, ctypes.c_int64, _P]),
    "lmg_local_coarse_source": (_I, [_SYS, _I, _I, _P, _P, _I, _P, _P, _I, _P, _P, _P, _P]),
    "lmg_local_correct": (_I, [_I, _I, _I, _I, _P, _P, _P]),
    "lmg_local_workspace": (ctypes.c_size_t, [_I, _I, _I]),
    "lmg_local_residual_post": (_I, [_SYS, _I, _I, _P, _P, _I, _P, _I, _P, _P, _P, _P]),
    "lmg_local_residual_full_a": (_I, [_SYS, _I, _P, _P, _I, _I, _P, _P, _P]),
    "lmg_local_residual_full_b": (_I, [_SYS, _I, _I, _P, _P, _I, _P, _I, _P, _P, _P]),
    "lmg_norms_from_blocks": (_I, [_P, _I, _I, _P, _P]),
    "lmg_apply_block": (_I, [_SYS, _I, _I, _P, _P, _P]),
    "lmg_vjp_block": (_I, [_SYS, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "lmg_dense_apply": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P]),
    "lmg_dense_vjp": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "lmg_l2_norms": (_I, [_P, _I, _I, _I, _P, _P, _P]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load liblmg.so and declare every exported symbol (raises if anything is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -m paper_2007_07336_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == LMG_OK:
        return
    msg = load().lmg_last_error().decode()
    if rc == LMG_ERR_DIMENSION:
        raise DimensionError(msg)
    if rc == LMG_ERR_CONFIGURATION:
        raise ConfigurationError(msg)
    if rc == LMG_ERR_PROTOCOL:
        raise ProtocolError(msg)
    raise LmgCudaError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else t.data_ptr()


def stream_handle(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


def launch_count() -> int:
    return int(load().lmg_launch_count())


ROUTES = ("step_small", "step_small_full", "step_wide", "step_wide_full", "step_tiny",
          "step_tiny_full", "tgemm_big", "tgemm_small", "serial_splitk", "sweep_fcf", "sweep_seq",
          "conv_fwd", "conv_adj", "conv_pgrad", "chain", "wsweep")


def set_canonical_order(on: bool) -> bool:
    """Canonical summation order on/off (include/lmg.h); returns the previous setting."""
    return bool(load().lmg_set_canonical_order(1 if on else 0))


def route_counts() -> dict:
    """Launches per kernel variant since the library was loaded (include/lmg.h LMG_ROUTE_*)."""
    buf = (ctypes.c_ulonglong * len(ROUTES))()
    n = load().lmg_route_counts(buf, len(ROUTES))
    if n != len(ROUTES):
        raise RuntimeError(f"liblmg reports {n} route counters, expected {len(ROUTES)}")
    return dict(zip(ROUTES, (int(v) for v in buf)))


def timing_enable(on: bool) -> None:
    check(load().lmg_timing_enable(1 if on else 0))


def timing_read(cls: int = -1):
    """(ms, flops, bytes, launches) summed over the recorded launches of class `cls`."""
    ms, fl, by = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    n = ctypes.c_ulonglong()
    check(load().lmg_timing_read(cls, ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(by),
                                 ctypes.byref(n)))
    return ms.value, fl.value, by.value, int(n.value)
