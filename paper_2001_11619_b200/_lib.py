"""ctypes binding of libskelb200.so (the C ABI declared in include/skelb200.h).

There is deliberately no CPU fallback: if the shared library is missing or no
CUDA device is visible, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SKB_LIB") or os.path.join(_HERE, "libskelb200.so")   # SKB_LIB: A/B builds

GEMM_DT = np.dtype([("A", "u8"), ("B", "u8"), ("C", "u8"), ("D", "u8"),
                    ("m", "i8"), ("n", "i8"), ("k", "i8"),
                    ("lda", "i8"), ("ldb", "i8"), ("ldc", "i8"), ("ldd", "i8"),
                    ("alpha", "f8"), ("beta", "f8"), ("transA", "i4"), ("transB", "i4"),
                    ("tile_begin", "i8")])
assert GEMM_DT.itemsize == 120
MAT_DT = np.dtype([("ptr", "u8"), ("rows", "i8"), ("cols", "i8"), ("ld", "i8")])

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_f64 = ctypes.c_double

SIGNATURES = {
    "skb_version": [],
    "skb_prof_enable": [_i32],
    "skb_capture_begin": [_i64],
    "skb_capture_end": [],
    "skb_capture_release": [_i32],
    "skb_h2d": [_vp, _i64, _vp, _vp],
    "skb_prof_add": [_i32, _f64, _f64],
    "skb_prof_read": [_vp, _vp, _vp, _vp, _i32],
    "skb_gemm_grouped": [_vp, _i64, _vp],
    "skb_assemble_stack": [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp,
                           _vp, _i64, _i64, _vp],
    "skb_assemble_self": [_vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                          _i64, _vp],
    "skb_assemble_stack_lap": [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp,
                               _vp, _i64, _i64, _vp],
    "skb_assemble_self_lap": [_vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                              _i64, _vp],
    "skb_system_matvec_lap": [_vp, _vp, _vp, _vp, _i64, _vp, _i64, _vp, _vp],
    "skb_eval_interior_lap": [_vp, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp],
    "skb_assemble_aug": [_vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp],
    "skb_geqrf_batched": [_i64, _vp, _vp, _vp, _vp, _vp],
    "skb_qrcp_id_batched": [_i64, _vp, _vp, _vp, _vp, _vp, _f64, _vp, _vp, _vp, _vp, _vp, _vp,
                            _vp],
    "skb_copy2d_batched": [_i64, _vp, _vp, _i32, _vp],
    "skb_id_T_batched": [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "skb_getrf_batched": [_i64, _vp, _vp, _vp, _vp, _vp],
    "skb_getrs_batched": [_i64, _vp, _vp, _vp, _vp],
    "skb_gather_rows": [_i64, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _i64, _i64,
                        _vp],
    "skb_scatter_rows": [_i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _i32, _f64,
                         _i64, _i64, _vp],
    "skb_schur_accumulate": [_i64, _vp, _vp, _vp, _vp, _vp],
    "skb_diag_fill": [_i64, _vp, _i64, _f64, _vp, _i64, _f64, _vp],
    "skb_fill_rows": [_i64, _vp, _vp, _i64, _vp, _i64, _f64, _vp],
    "skb_psi_dot": [_i64, _vp, _vp, _vp, _i64, _vp, _i64, _i64, _vp, _i64, _f64, _vp, _i64, _vp],
    "skb_sum_partials": [_i64, _i32, _vp, _i64, _vp, _f64, _vp, _vp],
    "skb_system_matvec": [_vp, _vp, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _vp],
    "skb_eval_interior": [_vp, _vp, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp],
    "skb_point_in_domain": [_vp, _vp, _i64, _vp, _i64, _vp, _vp],
    "skb_level_schur": [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                        _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp],
    "skb_level_aug": [_i64, _vp, _vp, _i64] + [_vp] * 17 + [_vp, _vp, _vp, _vp, _i32, _vp],
    "skb_level_schur_acc": [_i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp],
    "skb_level_aug_narrow": [_i64, _vp, _vp, _i64, _i64] + [_vp] * 16 + [_vp, _vp, _vp],
    "skb_restore_rows": [_i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp],
    "skb_level_aug_update": [_i64, _vp, _vp, _i64] + [_vp] * 16 + [_i64] + [_vp] * 11,
    "skb_copy_rows_cols": [_i64, _vp, _i64, _vp, _i64, _i64, _vp, _vp, _vp],
    "skb_engine_start": [_vp, _i64, _vp, _f64, _vp, _i64, _vp, _i64, _f64, _vp, _i64, _i64, _i32, _vp],
    "skb_engine_wait": [_i64, _i64, _vp, _vp],
    "skb_engine_stream_wait": [_i64, _i64, _vp],
    "skb_engine_release": [_i64, _i64, _vp],
    "skb_engine_stop": [_i64],
    "skb_engine_ack": [_i64, _i64],
    "skb_engine_set_update": [_i64, _vp, _vp, _vp],
    "skb_engine_set_update_table": [_i64, _vp, _vp],
    "skb_pool_prewarm": [_i64, _i64],
    "skb_drv_run": [_i64, _vp, _f64, _vp],
    "skb_drv_resolve": [_i64],
    "skb_drv_level": [_i64, _i64, _vp, _vp],
    "skb_drv_free": [_i64],
    "skb_engine_go": [_i64],
    "skb_engine_set_lead": [_i64, _i64],
    "skb_engine_free": [_i64, _vp],
    "skb_debug_snap": [_i32, _vp, _i64],
    "skb_d2h": [_vp, _vp, _i64],
    "skb_dev_alloc": [_i64, _vp, _vp],
    "skb_dev_free": [ctypes.c_uint64, _vp],
    # native host runtime (host arrays only, no device)
    "skb_host_far_lists": [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _f64,
                           _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _i32],
    "skb_host_proxies": [_i64, _vp, _vp, _vp, _f64, _i64, _vp, _vp, _vp, _vp],
    "skb_host_leaf_actives": [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _vp, _vp],
    "skb_host_init": [],
    "skb_tree_build": [_vp, _i64, _i64, _i64, _vp, _vp],
    "skb_tree_sizes": [_i64, _vp],
    "skb_tree_export": [_i64] + [_vp] * 15,
    "skb_tree_free": [_i64],
    "skb_dirty_set": [_vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _i64, _vp, _i64, _f64, _vp],
}

_LIB = None


class SkbError(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load the shared library and declare argument types (no device needed)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise SkbError(f"{path} not built -- run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int64 if name in ("skb_debug_snap", "skb_host_leaf_actives") else ctypes.c_int
    lib.skb_host_init()
    _LIB = lib
    return lib


CALL_TIMES: dict | None = None     # set to {} to accumulate host time per entry point


def call(name: str, *args):
    """Invoke an entry point; numpy arrays are passed by address and kept alive
    for the duration of the call, torch tensors by data_ptr()."""
    if CALL_TIMES is not None:
        import time as _t
        t0 = _t.perf_counter()
        try:
            return _call(name, *args)
        finally:
            c = CALL_TIMES.setdefault(name, [0, 0.0])
            c[0] += 1
            c[1] += _t.perf_counter() - t0
    return _call(name, *args)


def _call(name: str, *args):
    lib = load()
    conv = []
    for a in args:
        if isinstance(a, np.ndarray):
            conv.append(a.ctypes.data)
        elif hasattr(a, "data_ptr"):
            conv.append(a.data_ptr())
        else:
            conv.append(a)
    rc = getattr(lib, name)(*conv)
    del conv
    if name == "skb_capture_end":
        return rc
    if rc != 0:
        raise SkbError(f"{name} returned {rc}")
    return rc


def ptr(x) -> int | None:
    """Device/host address of a torch tensor or numpy array (None passes NULL)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


FAMILIES = ("assemble", "geqrf", "qrcp", "id_T", "gemm", "getrf", "trsm", "move")


PROF_ON = False


def prof_enable(on: bool = True):
    global PROF_ON
    PROF_ON = bool(on)
    call("skb_prof_enable", 1 if on else 0)


def prof_add(family: str, flops: float = 0.0, nbytes: float = 0.0):
    """Register algorithmic work for a family (only while profiling)."""
    if PROF_ON:
        call("skb_prof_add", FAMILIES.index(family), float(flops), float(nbytes))


def prof_read(reset: bool = True) -> dict:
    """Per-family {ms, launches, flops, bytes} from the live event timers."""
    n = len(FAMILIES)
    ms = np.zeros(n)
    cnt = np.zeros(n, np.int64)
    fl = np.zeros(n)
    by = np.zeros(n)
    call("skb_prof_read", ms, cnt, fl, by, 1 if reset else 0)
    return {f: {"ms": float(ms[i]), "launches": int(cnt[i]), "flops": float(fl[i]),
                "bytes": float(by[i])} for i, f in enumerate(FAMILIES)}
