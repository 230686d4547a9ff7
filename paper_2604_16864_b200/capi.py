"""ctypes binding of the C ABI in include/hierasparse_b200.h.

Loads the in-tree ``lib/libhierasparse_b200.so``.  There is no fallback: if the
library is missing or cannot be loaded the import of any compute entry point
raises, so a GPU run can never silently route around the CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError, CudaError, DataError, IoError

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HS_LIB") or os.path.join(PKG, "lib", "libhierasparse_b200.so")  # HS_LIB: A/B tooling

HS_OK, HS_ERR_CONFIG, HS_ERR_IO, HS_ERR_DATA, HS_ERR_CUDA = 0, 2, 3, 4, 5
DTYPE_BF16, DTYPE_F16 = 0, 1
AXIS_CHANNEL, AXIS_SEQUENCE = 0, 1


class SparsityConfigC(C.Structure):
    _fields_ = [("s_key", C.c_double), ("s_value", C.c_double), ("block_size", C.c_uint32),
                ("reserved", C.c_uint32), ("sink_tokens", C.c_uint64), ("local_window", C.c_uint64)]


class DeviceCacheC(C.Structure):
    _fields_ = [("dtype", C.c_int), ("axis", C.c_int), ("head_dim", C.c_uint32),
                ("block_size", C.c_uint32), ("n_units", C.c_uint32), ("logical_blocks", C.c_uint32),
                ("dense_count", C.c_uint32), ("sparse_count", C.c_uint32),
                ("index_map", C.c_void_p), ("dense_pool", C.c_void_p), ("nnz_pool", C.c_void_p),
                ("meta_pool", C.c_void_p), ("slot_block", C.c_void_p)]


# Exported symbols (every one declared in include/hierasparse_b200.h).
EXPORTS = ("hs_last_error", "hs_version", "hs_status_word_decode", "hs_pool_counts", "hs_cache_bytes",
           "hs_prune_compress", "hs_block_losses", "hs_select_blocks", "hs_compress_with_flags", "hs_compress_with_mask", "hs_decompress", "hs_recompress",
           "hs_absorb_tail", "hs_decode", "hs_decode_workspace_bytes", "hs_decode_ws", "hs_decode_partial",
           "hs_decode_combine", "hs_prefill", "hs_kernel_launches")

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load (once) and type the shared library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    u32, u64, vp, i32 = C.c_uint32, C.c_uint64, C.c_void_p, C.c_int
    P = C.POINTER
    lib.hs_last_error.restype = C.c_char_p
    lib.hs_version.restype = i32
    lib.hs_kernel_launches.restype = u64
    sig = {
        "hs_pool_counts": [u64, P(SparsityConfigC), C.c_double, P(u32), P(u32), P(u32), P(u32), P(u32)],
        "hs_cache_bytes": [P(DeviceCacheC), P(u64), P(u64), P(u64), P(u64), P(u64)],
        "hs_prune_compress": [vp, u64, u64, P(SparsityConfigC), C.c_double, P(DeviceCacheC), vp, vp, vp],
        "hs_status_word_decode": [u64],
        "hs_block_losses": [vp, u64, u64, P(DeviceCacheC), vp, vp],
        "hs_select_blocks": [vp, u32, u32, P(SparsityConfigC), C.c_double, vp, vp],
        "hs_compress_with_flags": [vp, u64, u64, vp, P(DeviceCacheC), vp, vp],
        "hs_compress_with_mask": [vp, u64, u64, vp, u64, vp, P(DeviceCacheC), vp, vp],
        "hs_decompress": [P(DeviceCacheC), vp, vp, vp],
        "hs_recompress": [P(DeviceCacheC), P(SparsityConfigC), C.c_double, P(DeviceCacheC), vp, vp, vp, vp],
        "hs_absorb_tail": [P(DeviceCacheC), vp, u64, u64, P(SparsityConfigC), C.c_double, P(DeviceCacheC), vp, vp,
                           vp, vp],
        "hs_decode": [vp, P(DeviceCacheC), P(DeviceCacheC), vp, vp, u32, u32, C.c_float, u32, vp, vp],
        "hs_decode_workspace_bytes": [P(DeviceCacheC), u32, u32, P(u64)],
        "hs_decode_ws": [vp, P(DeviceCacheC), P(DeviceCacheC), vp, vp, u32, u32, C.c_float, u32, vp, vp, u64, vp],
        "hs_decode_partial": [vp, P(DeviceCacheC), P(DeviceCacheC), vp, vp, u32, u32, C.c_float, u32, u32,
                              i32, vp, vp],
        "hs_decode_combine": [vp, u32, u32, u32, u32, vp, vp],
        "hs_prefill": [vp, u32, u32, P(DeviceCacheC), P(DeviceCacheC), vp, vp, u32, i32, C.c_float, vp, vp],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = i32
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a status code to the reference's exception taxonomy (errors.hpp:10-25)."""
    if rc == HS_OK:
        return
    msg = _lib.hs_last_error().decode() if _lib is not None else "unknown"
    if rc == HS_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == HS_ERR_DATA:
        raise DataError(msg)
    if rc == HS_ERR_IO:
        raise IoError(msg)
    raise CudaError(msg)


def check_status_word(word: int) -> None:
    """Raise the reference exception recorded in a device status word (0 = OK)."""
    if word:
        check(load().hs_status_word_decode(word & 0xFFFFFFFFFFFFFFFF))


def kernel_launches() -> int:
    return int(load().hs_kernel_launches())
