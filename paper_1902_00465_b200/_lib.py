"""ctypes binding of ``librp.so`` (C ABI declared in ``include/rp.h``).

The library is built in-tree (``paper_1902_00465_b200/librp.so``) by
``__graft_entry__.build()`` / ``make -C paper_1902_00465_b200/csrc``. Loading fails
loudly when it is missing: there is no CPU or PyTorch fallback on the product path.
"""

from __future__ import annotations

import ctypes
import os

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RP_LIBRARY", os.path.join(HERE, "librp.so"))

# dtype codes (include/rp.h; 0/1 are the reference's DTYPE_CODES, tensor.py:16-21)
F32, F64, BF16, F16 = 0, 1, 2, 3
# ops
SUM, MEAN, MAX, PREMEAN = 0, 1, 2, 3
OPS = {"sum": SUM, "mean": MEAN, "max": MAX, "premean": PREMEAN}
# algorithms
AUTO, ONESHOT, TWOSHOT = 0, 1, 2
DIRECT, SCATTER = 1, 2
NVLS = 3
RELAY = 4
FLAT = 5
# fused optimizer apply (rp_all_reduce_apply)
OPT_SGD, OPT_ADAM, OPT_ADAMW = 0, 1, 2
ALGOS = {"auto": AUTO, "oneshot": ONESHOT, "twoshot": TWOSHOT, "direct": DIRECT, "scatter": SCATTER, "nvls": NVLS,
         "relay": RELAY, "flat": FLAT}
# link kinds (rp_comm_import topology discovery, rp_topology_check)
LINK_SELF, LINK_NVLINK, LINK_PCIE, LINK_NONE, LINK_UNKNOWN, LINK_SAME_DEVICE, LINK_LOOPBACK = range(7)
# layouts
NHWC, NCHW = 0, 1
# status codes -> exception classes (errors.py)
_ERRORS = {
    1: errors.ShapeError,
    2: errors.ConfigurationError,
    3: errors.CollectiveError,
    4: errors.CollectiveAbortedError,
    5: errors.ProtocolError,
}

_c_void_p = ctypes.c_void_p
_size_t = ctypes.c_size_t
_i = ctypes.c_int
_i64 = ctypes.c_int64
_f = ctypes.c_float
_d = ctypes.c_double
_pp = ctypes.POINTER(ctypes.c_void_p)
_pi64 = ctypes.POINTER(ctypes.c_int64)

# name -> (restype, argtypes); mirrors include/rp.h one-to-one
SIGNATURES = {
    "rp_last_error": (ctypes.c_char_p, []),
    "rp_version": (ctypes.c_char_p, []),
    "rp_comm_create": (_i, [_i, _i, _i, _size_t, _pp]),
    "rp_comm_create_virtual": (_i, [_i, _i, _size_t, _pp]),
    "rp_comm_export_size": (_size_t, []),
    "rp_comm_export": (_i, [_c_void_p, _c_void_p, ctypes.POINTER(_size_t)]),
    "rp_comm_import": (_i, [_c_void_p, _c_void_p, _size_t]),
    "rp_comm_set_loopback": (_i, [_c_void_p, _i]),
    "rp_loopback_prepare": (_i, [_i]),
    "rp_topology_check": (_i, [_i, _i, ctypes.POINTER(_i), _i, _i]),
    "rp_topology_uniform": (_i, [_i, ctypes.POINTER(_i)]),
    "rp_comm_topology": (_i, [_c_void_p, ctypes.POINTER(_i), ctypes.POINTER(_i)]),
    "rp_comm_destroy": (_i, [_c_void_p]),
    "rp_comm_pool": (_i, [_c_void_p, _i, _pp, ctypes.POINTER(_size_t)]),
    "rp_comm_info": (_i, [_c_void_p, ctypes.POINTER(_i), ctypes.POINTER(_i), ctypes.POINTER(_i),
                          ctypes.POINTER(_i), ctypes.POINTER(_size_t)]),
    "rp_comm_reserve": (_i, [_c_void_p, _size_t]),
    "rp_comm_check": (_i, [_c_void_p]),
    "rp_comm_set_timeout": (_i, [_c_void_p, ctypes.c_uint64]),
    "rp_comm_set_block_cap": (_i, [_c_void_p, ctypes.c_int]),
    "rp_all_reduce": (_i, [_c_void_p, _c_void_p, _c_void_p, _size_t, _i, _i, _i, _i, _i, _c_void_p]),
    "rp_register_export_size": (_size_t, []),
    "rp_register_export": (_i, [_c_void_p, _c_void_p, _size_t, _c_void_p, ctypes.POINTER(_size_t)]),
    "rp_register_import": (_i, [_c_void_p, _c_void_p, _size_t, ctypes.POINTER(_i)]),
    "rp_unregister": (_i, [_c_void_p, _i]),
    "rp_all_gather": (_i, [_c_void_p, _c_void_p, _c_void_p, _size_t, _c_void_p]),
    "rp_broadcast": (_i, [_c_void_p, _c_void_p, _c_void_p, _size_t, _i, _i, _c_void_p]),
    "rp_apply_shard": (_i, [_c_void_p, _size_t, _i, ctypes.POINTER(_size_t), ctypes.POINTER(_size_t)]),
    "rp_all_reduce_apply": (_i, [_c_void_p, _c_void_p, _c_void_p, _size_t, _i, _i, ctypes.POINTER(_d), _c_void_p,
                                 _c_void_p, _c_void_p, _c_void_p]),
    "rp_all_reduce_apply_v": (_i, [_c_void_p, _pp, _pp, _size_t, _i, _i, ctypes.POINTER(_d), _pp, _pp, _pp,
                                   _c_void_p]),
    "rp_all_reduce_algo": (_i, [_c_void_p, _c_void_p, _c_void_p, _size_t, _i, _i, _i, _i, _i,
                                ctypes.POINTER(ctypes.c_int)]),
    "rp_all_reduce_plan": (_i, [_c_void_p, _c_void_p, _c_void_p, _size_t, _i, _i, _i, _i, _i, _pi64]),
    "rp_all_reduce_v": (_i, [_c_void_p, _pp, _pp, _size_t, _i, _i, _i, _i, _i, _c_void_p]),
    "rp_all_gather_v": (_i, [_c_void_p, _pp, _pp, _size_t, _c_void_p]),
    "rp_broadcast_v": (_i, [_c_void_p, _pp, _pp, _size_t, _i, _i, _c_void_p]),
    "rp_bn_stats": (_i, [_c_void_p, _c_void_p, _i, _i64, _i64, _i64, _i, _f, _c_void_p, _c_void_p,
                         _c_void_p, _c_void_p, _c_void_p]),
    "rp_bn_bwd_stats": (_i, [_c_void_p, _c_void_p, _c_void_p, _i, _i64, _i64, _i64, _i, _c_void_p,
                             _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p]),
    "rp_bn_apply": (_i, [_c_void_p, _c_void_p, _i, _i64, _i64, _i64, _i, _c_void_p, _c_void_p,
                         _c_void_p, _c_void_p, _c_void_p]),
    "rp_bn_bwd_apply": (_i, [_c_void_p, _c_void_p, _c_void_p, _i, _i64, _i64, _i64, _i, _c_void_p,
                             _c_void_p, _c_void_p, _c_void_p, _c_void_p, _d, _c_void_p, _c_void_p]),
    "rp_nvls_create": (_i, [_c_void_p, _size_t, ctypes.c_char_p, _size_t]),
    "rp_nvls_serve": (_i, [_c_void_p]),
    "rp_nvls_join": (_i, [_c_void_p, ctypes.c_char_p]),
    "rp_nvls_add": (_i, [_c_void_p]),
    "rp_nvls_bind": (_i, [_c_void_p]),
    "rp_nvls_pool": (_i, [_c_void_p, _pp, ctypes.POINTER(_size_t)]),
    "rp_pack": (_i, [_c_void_p, _i, _pp, _pi64, _pi64, _i, _i, _c_void_p]),
    "rp_unpack": (_i, [_c_void_p, _i, _pp, _pi64, _pi64, _i, _i, _c_void_p]),
}

_LIB = None


def load():
    """Load librp.so once; raise NativeLibraryError if it is absent or incomplete."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise errors.NativeLibraryError(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_1902_00465_b200/csrc` (no CPU fallback exists)")
    try:
        lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    except OSError as e:
        raise errors.NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from e
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:
            raise errors.NativeLibraryError(f"{LIB_PATH} does not export {name}")
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def last_error() -> str:
    return load().rp_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Raise the reference exception class matching a nonzero status (include/rp.h)."""
    if rc == 0:
        return
    cls = _ERRORS.get(rc, errors.CollectiveError)
    msg = last_error()
    raise cls(f"{what}: {msg}" if what else msg)


def ptr_array(ptrs):
    arr = (ctypes.c_void_p * len(ptrs))(*[ctypes.c_void_p(int(p)) for p in ptrs])
    return ctypes.cast(arr, _pp), arr


def i64_array(vals):
    arr = (ctypes.c_int64 * len(vals))(*[int(v) for v in vals])
    return ctypes.cast(arr, _pi64), arr
