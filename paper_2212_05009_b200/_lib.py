"""ctypes binding of the in-tree sm_100a library `lib/libgcnb.so` (include/gcnb.h).

This is the reference-side binding a maintainer of `gcnpart` would add (see
INTEGRATION.md): plain device pointers, sizes and stream handles cross the
boundary, never torch or numpy objects.  There is no fallback: importing the
product path without the built library raises immediately.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

# GCNB_LIB: an alternative build of the same library (A/B measurements of kernel variants)
LIB_PATH = Path(os.environ.get("GCNB_LIB") or Path(__file__).resolve().parent / "lib" / "libgcnb.so")

GCNB_OK, GCNB_EINVAL, GCNB_ECUDA, GCNB_ECOMM, GCNB_EKEY = range(5)
ACT = {"relu": 0, "identity": 1}
MAX_PEERS = 64

_c_int = ctypes.c_int32
_c_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_f32 = ctypes.c_float
_f64 = ctypes.c_double

# name -> (restype, argtypes)
_SIGNATURES = {
    "gcnb_last_error": (ctypes.c_char_p, []),
    "gcnb_version": (_c_int, []),
    "gcnb_set_watchdog_ms": (_c_int, [_c_i64]),
    "gcnb_launch_count": (ctypes.c_uint64, []),
    "gcnb_device_count": (_c_int, [ctypes.POINTER(_c_int)]),
    "gcnb_malloc": (_c_int, [ctypes.POINTER(_vp), ctypes.c_size_t]),
    "gcnb_free": (_c_int, [_vp]),
    "gcnb_memset_async": (_c_int, [_vp, _c_int, ctypes.c_size_t, _vp]),
    "gcnb_ipc_get_handle": (_c_int, [_vp, ctypes.c_char_p]),
    "gcnb_ipc_open_handle": (_c_int, [ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "gcnb_ipc_close_handle": (_c_int, [_vp]),
    "gcnb_enable_peer_access": (_c_int, [_c_int]),
    "gcnb_event_create": (_c_int, [ctypes.POINTER(_vp)]),
    "gcnb_event_destroy": (_c_int, [_vp]),
    "gcnb_event_record": (_c_int, [_vp, _vp, _c_int]),
    "gcnb_event_elapsed_ms": (_c_int, [_vp, _vp, ctypes.POINTER(_f32)]),
    "gcnb_stream_is_capturing": (_c_int, [_vp, ctypes.POINTER(_c_int)]),
    "gcnb_spmm_f32": (_c_int, [_vp, _vp, _vp, _vp, _c_int, _vp, _c_int, _c_int, _vp, _c_int, _vp]),
    "gcnb_window_csr": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _c_int, _vp, _vp, _vp]),
    "gcnb_aggwin_applies": (_c_int, [_c_int, _c_int, ctypes.POINTER(_c_int)]),
    "gcnb_set_aggwin_passes": (_c_int, [_c_int]),
    "gcnb_aggwin_f32": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _vp, _c_int, _c_int, _vp, _c_int, _c_int, _vp]),
    "gcnb_pack_rows_f32": (_c_int, [_vp, _c_int, _c_int, _vp, _vp, _c_int, _vp, _c_int, _vp, _vp, _vp]),
    "gcnb_wait_flags": (_c_int, [_vp, _vp, _c_int, _vp, _vp, _c_int, _vp]),
    "gcnb_fwd_layer_f32": (
        _c_int, [_vp, _vp, _vp, _vp, _c_int, _vp, _c_int, _c_int, _vp, _c_int, _vp, _c_int, _c_int, _vp]),
    "gcnb_dense_f32": (_c_int, [_vp, _c_int, _vp, _c_int, _c_int, _vp, _c_int, _vp, _c_int, _c_int, _vp]),
    "gcnb_set_dense_mode": (_c_int, [_c_int]),
    "gcnb_set_dw_mode": (_c_int, [_c_int]),
    "gcnb_bwd_grid": (_c_int, [_c_int, _c_int, _c_int, _c_int, ctypes.POINTER(_c_int)]),
    "gcnb_set_agg_shape": (_c_int, [_c_int, _c_int]),
    "gcnb_set_agg_gather": (_c_int, [_c_int]),
    "gcnb_bwd_epilogue_f32": (_c_int, [_vp, _c_int, _c_int, _vp, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _vp,
                                       _c_int, _vp, _c_int, _vp, _vp]),
    "gcnb_dense_tc_applies": (_c_int, [_c_int, _c_int, ctypes.POINTER(_c_int)]),
    "gcnb_dense_bits_f32": (_c_int, [_vp, _c_int, _c_int, _c_int, _vp, _c_int, _vp, _c_int, _vp, _c_int, _vp]),
    "gcnb_dw_f32": (_c_int, [_vp, _c_int, _c_int, _vp, _c_int, _c_int, _vp, _c_int, _vp, _vp]),
    "gcnb_bwd_layer_f32": (
        _c_int,
        [_vp, _vp, _vp, _vp, _c_int, _vp, _c_int, _c_int, _vp, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _vp,
         _vp, _vp]),
    "gcnb_bwd_workspace_ld": (_c_int, [_c_int, _c_int, ctypes.POINTER(_c_int)]),
    "gcnb_set_split_all": (_c_int, [_c_int]),
    "gcnb_set_fwd_tf": (_c_int, [_c_int]),
    "gcnb_reduce_partials_f32": (_c_int, [_vp, _c_int, _c_i64, _vp, _c_int, _vp]),
    "gcnb_reduce_sgd_f32": (_c_int, [_vp, _c_int, _c_i64, _vp, _c_int, _vp, _f32, _vp]),
    "gcnb_loss_scratch_doubles": (_c_int, []),
    "gcnb_loss_grad_f32": (
        _c_int, [_vp, _c_int, _c_int, _c_int, _vp, _f64, _vp, _c_int, _c_int, _vp, _vp, _vp]),
    "gcnb_loss_grad_pack_f32": (
        _c_int, [_vp, _c_int, _c_int, _c_int, _vp, _f64, _vp, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _c_int,
                 _c_int, _vp, _vp]),
    "gcnb_dense_pack_f32": (_c_int, [_vp, _c_int, _c_int, _c_int, _vp, _c_int, _vp, _c_int, _c_int, _vp, _c_int,
                                     _vp, _vp]),
    "gcnb_fwd_layer_pack_f32": (_c_int, [_vp, _vp, _vp, _c_int, _vp, _c_int, _c_int, _vp, _c_int, _vp, _c_int,
                                         _c_int, _vp, _vp]),
    "gcnb_bwd_layer_pack_f32": (_c_int, [_vp, _vp, _vp, _c_int, _vp, _c_int, _c_int, _vp, _c_int, _c_int, _vp, _vp,
                                         _c_int, _c_int, _vp, _vp, _vp, _vp]),
    "gcnb_bwd_epilogue_pack_f32": (_c_int, [_vp, _c_int, _c_int, _vp, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _vp,
                                            _c_int, _c_int, _vp, _vp, _vp]),
    "gcnb_sum_buffers_f32": (_c_int, [_vp, _c_int, _c_i64, _vp, _vp]),
    "gcnb_sum_buffers_f64": (_c_int, [_vp, _c_int, _c_i64, _vp, _vp]),
    "gcnb_sgd_f32": (_c_int, [_vp, _vp, _c_i64, _f32, _vp]),
    "gcnb_push_f32": (_c_int, [_vp, _c_i64, _vp, _vp, _c_int, _vp, _vp]),
    "gcnb_sum_slots_f32": (_c_int, [_vp, _c_int, _c_i64, _c_i64, _vp, _vp, _vp]),
    "gcnb_signal_peers": (_c_int, [_vp, _c_int, _vp]),
    "gcnb_cast_pad_f64_f32": (_c_int, [_vp, _c_int, _c_i64, _c_int, _vp, _c_int, _vp]),
    "gcnb_plan_build": (_c_int, [_vp, _vp, _c_i64, _vp, _c_int, ctypes.POINTER(_vp), ctypes.POINTER(_c_i64), _vp, _vp,
                                 _vp, _vp, _vp]),
    "gcnb_plan_free": (_c_int, [_vp]),
    "gcnb_layout_fill": (_c_int, [_vp, _vp, _vp, _c_i64, _vp, _c_int, _vp, _c_i64, _c_i64, _c_int, _vp, _vp, _vp,
                                  _vp, _vp, _vp]),
    "gcnb_copy_d2h": (_c_int, [_vp, _vp, ctypes.c_size_t]),
    "gcnb_normalize_f64": (_c_int, [_vp, _vp, _vp, _c_i64, _vp, _vp, _vp, ctypes.POINTER(_c_i64), _vp]),
    "gcnb_transpose_f64": (_c_int, [_vp, _vp, _vp, _c_i64, _c_i64, _vp, _vp, _vp, _vp]),
    "gcnb_induced_pattern": (_c_int, [_vp, _vp, _c_i64, _vp, _c_i64, _vp, _vp, _vp, _vp, ctypes.POINTER(_c_i64),
                                      _vp]),
}


class CommError(RuntimeError):
    """A rank did not receive a message its plan promised (runtime.py:47-48)."""


_lib = None


def load() -> ctypes.CDLL:
    """Load libgcnb.so (fail loudly when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the GPU path has no CPU fallback)"
        )
    lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | ctypes.RTLD_GLOBAL)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    if os.environ.get("GCNB_WATCHDOG_MS"):
        check(lib.gcnb_set_watchdog_ms(int(os.environ["GCNB_WATCHDOG_MS"])))
    if os.environ.get("GCNB_DW_MODE"):
        check(lib.gcnb_set_dw_mode(int(os.environ["GCNB_DW_MODE"])))
    if os.environ.get("GCNB_FWD_TF"):  # A/B knob (gcnb_set_fwd_tf)
        check(lib.gcnb_set_fwd_tf(int(os.environ["GCNB_FWD_TF"])))
    if os.environ.get("GCNB_SPLIT_ALL"):  # measurement knob: aggregation + dense kernels for every layer
        check(lib.gcnb_set_split_all(int(os.environ["GCNB_SPLIT_ALL"])))
    if os.environ.get("GCNB_AGG_GATHER"):  # tuning knob (gcnb_set_agg_gather), e.g. for A/B bench runs
        check(lib.gcnb_set_agg_gather(int(os.environ["GCNB_AGG_GATHER"])))
    return lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def check(rc: int) -> None:
    """Map a gcnb status code to the reference's exception classes."""
    if rc == GCNB_OK:
        return
    msg = load().gcnb_last_error().decode(errors="replace")
    if rc == GCNB_EINVAL:
        raise ValueError(msg)
    if rc == GCNB_EKEY:
        raise KeyError(msg)
    if rc == GCNB_ECOMM:
        raise CommError(msg)
    raise RuntimeError(f"gcnb: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def ptr_array(ptrs) -> ctypes.Array:
    arr = (ctypes.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


class HaloPack(ctypes.Structure):
    """gcnb_halo_pack (include/gcnb.h): a halo pack fused into a producer's epilogue."""

    _fields_ = [("map_ptr", ctypes.c_void_p), ("map", ctypes.c_void_p), ("dst", ctypes.c_void_p),
                ("flags", ctypes.c_void_p), ("n_seg", ctypes.c_int32), ("ldd", ctypes.c_int32),
                ("counter", ctypes.c_void_p)]


def halo_pack(map_ptr: int, map_: int, dsts, flags, ldd: int, counter: int):
    """A HaloPack (by reference) plus the host arrays it points at (keep both alive for the call)."""
    d = ptr_array(dsts)
    f = ptr_array(flags) if flags is not None else None
    hp = HaloPack(map_ptr, map_, ctypes.cast(d, ctypes.c_void_p),
                  ctypes.cast(f, ctypes.c_void_p) if f is not None else None, len(dsts), ldd, counter)
    return ctypes.byref(hp), (hp, d, f)


def int_array(vals) -> ctypes.Array:
    arr = (ctypes.c_int32 * max(1, len(vals)))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr


def launch_count() -> int:
    return int(load().gcnb_launch_count())


def dense_tc_applies(d_in: int, d_out: int) -> bool:
    out = _c_int(0)
    call("gcnb_dense_tc_applies", d_in, d_out, ctypes.byref(out))
    return bool(out.value)


def bwd_grid(n_rows: int, d_prev: int, d_k: int, with_gprev: bool) -> int:
    out = ctypes.c_int32(0)
    call("gcnb_bwd_grid", n_rows, d_prev, d_k, int(with_gprev), ctypes.byref(out))
    return int(out.value)


def bwd_workspace_ld(d_prev: int, d_k: int) -> int:
    out = ctypes.c_int32(0)
    call("gcnb_bwd_workspace_ld", d_prev, d_k, ctypes.byref(out))
    return int(out.value)


def aggwin_applies(d: int, bt: int) -> bool:
    out = _c_int(0)
    call("gcnb_aggwin_applies", d, bt, ctypes.byref(out))
    return bool(out.value)


def loss_scratch_doubles() -> int:
    return int(load().gcnb_loss_scratch_doubles())
