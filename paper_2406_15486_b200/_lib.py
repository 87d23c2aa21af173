"""ctypes binding of libsampleattn.so (the C ABI in include/sampleattn.h).

There is no fallback: if the library is missing or was built for another
architecture, every entry point raises.  torch is only used by the callers
for device memory and streams; nothing here imports it.
"""

from __future__ import annotations

import ctypes
import os

from .errors import InputError, InternalInvariantError

LIB_PATH = os.environ.get("SA_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                         "libsampleattn.so")

SA_OK, SA_ERR_INVALID, SA_ERR_UNSUPPORTED, SA_ERR_INTERNAL, SA_ERR_CUDA = 0, -1, -2, -3, -4
SA_BF16, SA_FP32 = 0, 1
SA_STATUS_EMPTY_BLOCK, SA_STATUS_MASK, SA_STATUS_NORMALISER = 1, 2, 4
SA_STAGE1_TENSOR, SA_STAGE1_EXACT = 0, 1
SA_WS_ROW_STATS = 0

_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_L = ctypes.c_longlong
_Z = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/sampleattn.h
SIGNATURES = {
    "sa_version": (_I, []),
    "sa_last_error": (ctypes.c_char_p, []),
    "sa_launch_count": (_L, []),
    "sa_status": (_I, [ctypes.POINTER(ctypes.c_uint), _I]),
    "sa_workspace_bytes": (_Z, [_I, _I, _I, _I, _I, _I, _I]),
    "sa_check_finite": (_I, [_P, _I, ctypes.c_int64, _P, _P]),
    "sa_copy2d_async": (_I, [_P, ctypes.c_size_t, _P, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t, _P]),
    "sa_stage1": (_I, [_P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P, _P, _Z, _P]),
    "sa_select": (_I, [_P, _P, _I, _I, _I, _D, _D, _D, _P, _D, _P, _P, _P, _P, _P, _P, _D, _P]),
    "sa_band_table_len": (_I, [_I, _I]),
    "sa_refine_bands": (_I, [_P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _Z, _P]),
    "sa_certify_band_ties": (_I, [_I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _D, _D, _P, _Z, _P]),
    "sa_workspace_offset": (ctypes.c_longlong, [_I, _I, _I, _I, _I, _I, _I, _I]),
    "sa_merge": (_I, [_P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P]),
    "sa_sampled_retained": (_I, [_I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _Z, _P, _P]),
    "sa_full_mask": (_I, [_I, _I, _P, _P, _P]),
    "sa_schedule_len": (_I, [_I, _I, _I, _I]),
    "sa_schedule": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P]),
    "sa_sparse_forward": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "sa_sparse_forward_peers": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P,
                                     ctypes.POINTER(_P), _I, _P]),
    "sa_ipc_export": (_I, [_P, _P, ctypes.POINTER(ctypes.c_ulonglong)]),
    "sa_ipc_open": (_I, [_P, ctypes.POINTER(_P)]),
    "sa_ipc_close": (_I, [_P]),
}
SA_MAX_PEERS = 7
SA_IPC_HANDLE_BYTES = 64

_lib = None
_load_error = None


def load():
    """Load (once) and return the library; raise if it is unavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is not None:
        raise RuntimeError(_load_error)
    if not os.path.exists(LIB_PATH):
        _load_error = (f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                       f"g.build()'` (there is no CPU fallback)")
        raise RuntimeError(_load_error)
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols() -> list:
    return list(SIGNATURES)


def call(name: str, *args) -> int:
    """Call an entry point, translating status codes into the reference's
    exception types (InputError / InternalInvariantError) or RuntimeError."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc == SA_OK:
        return rc
    msg = lib.sa_last_error().decode(errors="replace")
    if rc in (SA_ERR_INVALID, SA_ERR_UNSUPPORTED):
        raise InputError(f"{name}: {msg}")
    if rc == SA_ERR_INTERNAL:
        raise InternalInvariantError(f"{name}: {msg}")
    raise RuntimeError(f"{name} failed ({rc}): {msg}")


def launch_count() -> int:
    return int(load().sa_launch_count())
