"""ctypes binding of libhsweep.so (the C ABI in include/hsweep.h).

The CUDA library is REQUIRED: importing the device layer without it, or
without a CUDA device, raises -- there is no CPU fallback on the hot path.
Status codes become the reference's exception classes.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("HSWEEP_LIB", Path(__file__).resolve().parent / "libhsweep.so"))

HS_OK, HS_E_SHAPE, HS_E_ZERO_PIVOT, HS_E_ZERO_DIAG, HS_E_NONFINITE, HS_E_CUDA, HS_E_ARG, \
    HS_E_BUFFER = range(8)
HS_VARIANT_UD, HS_VARIANT_X = 0, 1

_vp = C.c_void_p
_i64p = C.POINTER(C.c_int64)

# name -> (restype, argtypes)
SIGNATURES = {
    "hs_version": (C.c_int, []),
    "hs_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "hs_ctx_destroy": (C.c_int, [_vp]),
    "hs_ctx_set_stream": (C.c_int, [_vp, _vp]),
    "hs_ctx_set_sweep_segments": (C.c_int, [_vp, C.c_int]),
    "hs_ctx_set_sweep_cluster": (C.c_int, [_vp, C.c_int]),
    "hs_last_error": (C.c_char_p, [_vp]),
    "hs_last_error_index": (C.c_longlong, [_vp]),
    "hs_launch_count": (C.c_longlong, [_vp]),
    "hs_synchronize": (C.c_int, [_vp]),
    "hs_profile_enable": (C.c_int, [_vp, C.c_int]),
    "hs_profile_reset": (C.c_int, [_vp]),
    "hs_profile_read": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                  C.POINTER(C.c_longlong)]),
    "hs_stencil_create": (C.c_int, [_vp, C.c_int, _i64p, C.c_int, C.POINTER(C.c_int8),
                                    C.POINTER(C.c_double), C.POINTER(_vp)]),
    "hs_stencil_destroy": (C.c_int, [_vp, _vp]),
    "hs_stencil_download": (C.c_int, [_vp, _vp, C.POINTER(C.c_double)]),
    "hs_assemble_fd": (C.c_int, [_vp, C.c_int, _i64p, C.c_double, C.POINTER(C.c_double),
                                 C.POINTER(C.c_double), C.POINTER(C.c_double), _vp,
                                 C.POINTER(_vp)]),
    "hs_assemble_fe": (C.c_int, [_vp, C.c_int, _i64p, C.POINTER(C.c_double),
                                 C.POINTER(C.c_double), C.POINTER(C.c_double),
                                 C.POINTER(C.c_double), _vp, C.c_int64, _vp, C.c_int64,
                                 C.POINTER(C.c_int32), C.c_double, C.c_int, C.c_int,
                                 C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(_vp)]),
    "hs_stencil_apply": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int]),
    "hs_stencil_residual": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int]),
    "hs_jacobi": (C.c_int, [_vp, _vp, _vp, _vp, C.c_double, C.c_int, C.c_int, C.c_int]),
    "hs_transfer_create": (C.c_int, [_vp, C.c_int, _i64p, _i64p, C.POINTER(C.c_uint8),
                                     C.POINTER(_vp)]),
    "hs_transfer_create_window": (C.c_int, [_vp, C.c_int, _i64p, _i64p, C.POINTER(C.c_uint8),
                                            _i64p, C.POINTER(_vp)]),
    "hs_transfer_destroy": (C.c_int, [_vp, _vp]),
    "hs_restrict": (C.c_int, [_vp, _vp, _vp, _vp, C.c_double, C.c_int]),
    "hs_restrict_residual": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, C.c_double, C.c_int]),
    "hs_prolong_add": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int, C.c_int]),
    "hs_sweep_create": (C.c_int, [_vp, _vp, C.c_int, _i64p, _i64p, _i64p, _i64p,
                                  C.POINTER(_vp), C.POINTER(_vp)]),
    "hs_sweep_destroy": (C.c_int, [_vp, _vp]),
    "hs_sweep_apply": (C.c_int, [_vp, _vp, C.c_int, _vp, _vp]),
    "hs_sweep_apply_many": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp, _vp, C.c_longlong]),
    "hs_sweep_rhs_width": (C.c_int, [_vp]),
    "hs_sweep_max_fronts": (C.c_int, [_vp]),
    "hs_sweep_factor_bytes": (C.c_longlong, [_vp]),
    "hs_sweep_plan_launches": (C.c_int, [_vp, C.c_int]),
    "hs_sweep_segments": (C.c_int, [_vp]),
    "hs_sweep_chunks": (C.c_int, [_vp]),
    "hs_sweep_solve_one": (C.c_int, [_vp, _vp, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                     C.c_int64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hs_exact_create": (C.c_int, [_vp, _vp, C.POINTER(_vp)]),
    "hs_csr_create": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p,
                                C.POINTER(C.c_double), C.POINTER(_vp)]),
    "hs_csr_destroy": (C.c_int, [_vp, _vp]),
    "hs_csr_apply": (C.c_int, [_vp, _vp, _vp, _vp, C.c_double, C.c_double, C.c_int]),
    "hs_exact_create_csr": (C.c_int, [_vp, C.c_int64, C.c_int64, _i64p, _i64p,
                                      C.POINTER(C.c_double), C.c_int, C.POINTER(_vp)]),
    "hs_sweep_plan_nx": (C.c_int, [_vp, _vp, C.c_int, _i64p, _i64p, C.POINTER(C.c_int)]),
    "hs_sweep_plan_relay": (C.c_int, [_vp, _vp, C.c_int, C.POINTER(C.c_int)]),
    "hs_cycle_create": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_double, C.c_int, C.c_double,
                                  C.c_int, C.POINTER(_vp)]),
    "hs_cycle_create_lane": (C.c_int, [_vp, _vp, C.POINTER(_vp)]),
    "hs_cycle_destroy": (C.c_int, [_vp, _vp]),
    "hs_vcycle": (C.c_int, [_vp, _vp, _vp, _vp]),
    "hs_vcycle_many": (C.c_int, [_vp, _vp, C.c_int, _vp, _vp, C.c_longlong]),
    "hs_vcycle_apply_a": (C.c_int, [_vp, _vp, _vp, _vp]),
    "hs_vcycle_apply_a_begin": (C.c_int, [_vp, _vp, _vp]),
    "hs_vcycle_apply_a_end": (C.c_int, [_vp, _vp, _vp, _vp]),
    "hs_vcycle_apply_a_part": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int]),
    "hs_vcycle_apply_az_part": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int]),
    "hs_block_dot": (C.c_int, [_vp, _vp, C.c_int64, C.c_int, _vp, C.c_int64, _vp]),
    "hs_block_dot_gated": (C.c_int, [_vp, _vp, C.c_int64, C.c_int, _vp, C.c_int64, _vp, _vp,
                                     _vp, C.c_double]),
    "hs_block_update_gated": (C.c_int, [_vp, _vp, C.c_int64, C.c_int, _vp, _vp, C.c_int64,
                                        _vp, _vp, _vp, C.c_double]),
    "hs_scale_inv_sqrt": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
    "hs_block_update_dot": (C.c_int, [_vp, _vp, C.c_int64, C.c_int, _vp, _vp, C.c_int64, _vp, _vp]),
    "hs_block_update": (C.c_int, [_vp, _vp, C.c_int64, C.c_int, _vp, _vp, C.c_int64, _vp]),
    "hs_lincomb": (C.c_int, [_vp, _vp, C.c_int64, C.c_int, _vp, _vp, C.c_int64]),
    "hs_scale": (C.c_int, [_vp, _vp, C.c_int64, C.c_double, C.c_double]),
    "hs_axpby": (C.c_int, [_vp, C.c_double, C.c_double, _vp, C.c_double, C.c_double, _vp,
                           C.c_int64]),
    "hs_norm2": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
}

_lib = None
_lock = threading.Lock()


def load_library(path: Path | str | None = None):
    """Load and type libhsweep.so (raises OSError when it is missing)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else Path(os.environ.get("HS_LIB", LIB_PATH))
        if not p.exists():
            raise OSError(f"libhsweep.so not built at {p}: run "
                          "`python -m paper_1412_0464_b200.build` (nvcc, sm_100a)")
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            if not hasattr(lib, name) and "HS_LIB" in os.environ:
                continue   # an A/B variant library built from older sources
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


class HsError(RuntimeError):
    pass


def raise_for(code: int, ctx) -> None:
    if code == HS_OK:
        return
    lib = load_library()
    msg = lib.hs_last_error(ctx).decode() if ctx else f"status {code}"
    if code in (HS_E_SHAPE, HS_E_ARG):
        raise ValueError(msg)
    if code in (HS_E_ZERO_PIVOT, HS_E_ZERO_DIAG):
        raise ZeroDivisionError(msg)
    if code == HS_E_NONFINITE:
        raise FloatingPointError(msg)
    if code == HS_E_BUFFER:
        raise RuntimeError(msg)
    raise HsError(f"CUDA failure in libhsweep: {msg}")


# ---------------------------------------------------------------------------
# per-device context bound to torch's current stream

class Context:
    def __init__(self, device: int):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1412_0464_b200 needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.device = device
        h = C.c_void_p()
        with torch.cuda.device(device):
            code = self.lib.hs_ctx_create(device, C.byref(h))
        if code != HS_OK:
            raise HsError(f"hs_ctx_create failed with status {code}")
        self.h = h
        self._stream = None
        self.bind_stream()

    def bind_stream(self):
        import torch
        s = torch.cuda.current_stream(self.device).cuda_stream
        if s != self._stream:
            self.lib.hs_ctx_set_stream(self.h, C.c_void_p(s))
            self._stream = s
        return self

    def call(self, name, *args):
        self.bind_stream()
        code = getattr(self.lib, name)(self.h, *args)
        raise_for(code, self.h)

    @property
    def launches(self) -> int:
        return int(self.lib.hs_launch_count(self.h))

    def synchronize(self):
        raise_for(self.lib.hs_synchronize(self.h), self.h)

    # built-in per-kernel-class event profiler
    KERNEL_CLASSES = ("stencil", "residual", "jacobi", "jacobi2z", "restrict", "prolong",
                      "sweep_gather", "sweep_front", "krylov_dot", "krylov_update",
                      "krylov_other", "setup", "pre_fused", "post_fused")

    def profile(self, on: bool):
        raise_for(self.lib.hs_profile_enable(self.h, int(on)), self.h)

    def profile_reset(self):
        raise_for(self.lib.hs_profile_reset(self.h), self.h)

    def profile_read(self) -> dict:
        k = len(self.KERNEL_CLASSES)
        ms = (C.c_double * k)()
        by = (C.c_double * k)()
        cnt = (C.c_longlong * k)()
        raise_for(self.lib.hs_profile_read(self.h, k, ms, by, cnt), self.h)
        return {name: {"ms": ms[i], "bytes": by[i], "launches": int(cnt[i])}
                for i, name in enumerate(self.KERNEL_CLASSES) if cnt[i]}


_contexts: dict = {}


def context(device: int | None = None) -> Context:
    import torch
    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    with _lock:
        ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lock:
            _contexts[device] = ctx
    return ctx


def i64(arr):
    a = np.ascontiguousarray(arr, dtype=np.int64)
    return a, a.ctypes.data_as(_i64p)
