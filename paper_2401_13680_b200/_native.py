"""ctypes binding of libpastila.so (include/pastila.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is usable, every device call raises ``RuntimeError`` naming the
cause.  One context per (process, device); one process per GPU.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

# PASTILA_LIB: alternative in-tree build (kernel tuning experiments)
LIB_PATH = Path(os.environ.get("PASTILA_LIB") or (Path(__file__).resolve().parent / "libpastila.so"))

PST_OK, PST_EINVAL, PST_ECUDA, PST_ENOMEM, PST_ESTATE = 0, -1, -2, -3, -4

_i64 = C.c_int64
_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int32)
_vp = C.c_void_p


class Snippets(C.Structure):
    _fields_ = [
        ("indices", _lp), ("fracs", _dp), ("curve", _dp), ("profiles", _dp),
        ("counts", _lp), ("nearest", _ip), ("labels", _lp),
        ("profile_area", C.c_double), ("profile_max", C.c_double),
        ("criterion", C.c_double), ("unassigned", C.c_int64),
    ]


# symbol -> (restype, argtypes); the ABI test checks every one is exported
SIGNATURES = {
    "pst_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "pst_destroy": (C.c_int, [_vp]),
    "pst_last_error": (C.c_char_p, []),
    "pst_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "pst_comm_unique_id": (C.c_int, [C.c_char_p]),
    "pst_set_series": (C.c_int, [_vp, _dp, _i64]),
    "pst_set_series_dev": (C.c_int, [_vp, _vp, _i64]),
    "pst_sliding_stats": (C.c_int, [_vp, _i64, _dp, _dp, _dp]),
    "pst_distance_rows": (C.c_int, [_vp, _i64, _i64, _i64, C.c_int, _dp]),
    "pst_mpdist_profiles": (C.c_int, [_vp, _i64, _i64, _i64, _i64, _i64, _dp]),
    "pst_select_snippets": (C.c_int, [_vp, _i64, _i64, _i64, _i64, C.POINTER(Snippets)]),
    "pst_select_from_profiles": (C.c_int, [_vp, _dp, _i64, _i64, _i64, _i64, C.POINTER(Snippets)]),
    "pst_profiles_dev": (C.c_int, [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _i64]),
    "pst_areas_dev": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp]),
    "pst_colmin_dev": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp]),
    "pst_max_dev": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp]),
    "pst_profile_reduce_dev": (C.c_int, [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "pst_sweep": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "pst_criterion": (C.c_int, [_vp, _dp, _i64, _i64, C.c_double, _dp]),
    "pst_labels": (C.c_int, [_vp, _dp, _i64, _i64, _i64, _lp]),
    "pst_profile_keys": (C.c_int, [_vp, _i64, _i64, _i64, _i64, _i64, _ip]),
    "pst_window_exact": (C.c_int, [_vp, _i64, _i64, _i64, _lp, _lp, _i64, _dp]),
    "pst_cert_stats": (C.c_int, [_vp, _lp, C.c_int]),
    "pst_prune_stats": (C.c_int, [_vp, _lp, C.c_int]),
    "pst_kernel_times": (C.c_int, [_vp, _dp]),
    "pst_comm_init": (C.c_int, [_vp, C.c_char_p, C.c_int, C.c_int]),
    "pst_comm_destroy": (C.c_int, [_vp]),
    "pst_comm_allreduce": (C.c_int, [_vp, _vp, _i64, C.c_int, C.c_int]),
    "pst_comm_broadcast": (C.c_int, [_vp, _vp, _i64, C.c_int]),
    "pst_comm_allgather": (C.c_int, [_vp, _vp, _vp, _i64]),
    "pst_local_best_dev": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _vp]),
    "pst_pick_global_dev": (C.c_int, [_vp, _vp, C.c_int, _i64, _i64, _vp, _vp]),
    "pst_tie_index_dev": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, _vp]),
    "pst_curve_min_dev": (C.c_int, [_vp, _vp, _vp, _i64, C.c_int]),
    "pst_debug_hist": (C.c_int, [_vp, _lp]),
    "pst_stream": (C.c_int, [_vp, C.POINTER(_vp)]),
    "pst_timing": (C.c_int, [_vp, C.c_int]),
    "pst_timing_read": (C.c_int, [_vp, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "pst_sync": (C.c_int, [_vp]),
    "pst_launch_count": (C.c_int64, [_vp]),
}

_lib = None
_lib_err: str | None = None
_lock = threading.Lock()


def load_library():
    """Load libpastila.so once; raise RuntimeError (loudly) if it is absent."""
    global _lib, _lib_err
    if _lib is not None:
        return _lib
    if _lib_err is not None:
        raise RuntimeError(_lib_err)
    if not LIB_PATH.exists():
        _lib_err = (f"CUDA extension {LIB_PATH} is not built; run `python -c \"import __graft_entry__ as g; "
                    f"g.build()\"` (no CPU fallback exists)")
        raise RuntimeError(_lib_err)
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(rc: int, what: str) -> None:
    if rc == PST_OK:
        return
    msg = load_library().pst_last_error().decode(errors="replace")
    if rc == PST_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"{what}: {msg}")


def ptr(a: np.ndarray | None, ctype=C.c_double):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


class Context:
    """One device context: owns the uploaded series and device buffers.

    A context is shared by all threads of a process that use its GPU (ctypes
    releases the GIL), so every upload-then-compute sequence runs under the
    context's lock: ``with ctx.using(values): ctx.call(...)``."""

    def __init__(self, device: int):
        lib = load_library()
        h = _vp()
        _check(lib.pst_create(int(device), C.byref(h)), f"pst_create(device={device})")
        self.h = h
        self.device = int(device)
        self._series_key = None
        self._series_ref = None
        self.lock = threading.RLock()

    @contextlib.contextmanager
    def using(self, values: np.ndarray):
        """Hold the context with ``values`` as its current series."""
        with self.lock:
            self.set_series(values)
            yield self

    def close(self):
        if self.h:
            load_library().pst_destroy(self.h)
            self.h = None

    def set_series(self, values: np.ndarray) -> None:
        with self.lock:
            self._set_series(values)

    def _set_series(self, values: np.ndarray) -> None:
        key = (id(values), values.ctypes.data, values.size)
        if key == self._series_key and self._series_ref is values:
            return
        v = np.ascontiguousarray(values, dtype=np.float64)
        _check(load_library().pst_set_series(self.h, ptr(v), v.size), "pst_set_series")
        self._series_key = key
        self._series_ref = values

    def call(self, name: str, *args):
        with self.lock:
            _check(getattr(load_library(), name)(self.h, *args), name)

    def launches(self) -> int:
        return int(load_library().pst_launch_count(self.h))


_ctxs: dict[int, Context] = {}


def current_device() -> int:
    env = os.environ.get("PASTILA_DEVICE")
    if env is not None:
        return int(env)
    return int(os.environ.get("LOCAL_RANK", "0"))


def context(device: int | None = None) -> Context:
    dev = current_device() if device is None else int(device)
    with _lock:
        ctx = _ctxs.get(dev)
        if ctx is None:
            ctx = Context(dev)
            _ctxs[dev] = ctx
        return ctx


def device_count() -> int:
    lib = load_library()
    n = C.c_int(0)
    rc = lib.pst_device_count(C.byref(n))
    return int(n.value) if rc == PST_OK else 0
