"""ctypes binding of libebz200.so (include/ebz200.h).

There is no CPU fallback: if the library is missing or no sm_100 device is
usable, every product entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
# EBZ_LIB: load another build of the same library (A/B timing tools only)
LIB_PATH = os.environ.get("EBZ_LIB") or os.path.join(PKG, "libebz200.so")


class NativeUnavailable(RuntimeError):
    """The CUDA library or a B200 device is not available."""


class EbzInfo(ctypes.Structure):
    _fields_ = [
        ("eb", ctypes.c_double),
        ("vmin", ctypes.c_double),
        ("vmax", ctypes.c_double),
        ("range", ctypes.c_double),
        ("n_unpred", ctypes.c_ulonglong),
        ("bit_length", ctypes.c_ulonglong),
        ("zeros_decoded", ctypes.c_ulonglong),
        ("used", ctypes.c_ulonglong),
        ("decoded", ctypes.c_longlong),
        ("status", ctypes.c_int),
        ("max_len", ctypes.c_int),
        ("blocks_done", ctypes.c_uint),
        ("pad0", ctypes.c_uint),
        ("total_bytes", ctypes.c_ulonglong),
    ]


# status bits (ebz200.h)
ST_EB_NONPOSITIVE = 0x001
ST_NONFINITE_IN = 0x002
ST_DEPTH_GT_64 = 0x004
ST_EMPTY_HIST = 0x008
ST_DEC_EXHAUSTED = 0x010
ST_DEC_INVALID = 0x020
ST_DEC_ANOMALY = 0x040
ST_UNPRED_MISMATCH = 0x080
ST_UNDERRUN = 0x100
ST_NONFINITE_OUT = 0x200
ST_CAPACITY = 0x400

_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_U64 = ctypes.c_uint64
_I64 = ctypes.c_int64
_SZ = ctypes.c_size_t
_INFO_P = ctypes.POINTER(EbzInfo)

EXPORTS = {
    "ebz_abi_version": (_I, []),
    "ebz_ctx_create": (_P, [_I]),
    "ebz_ctx_destroy": (None, [_P]),
    "ebz_ctx_trim": (_I, [_P]),
    "ebz_compress_trials": (_I, [_P, _I, _P, _I, _I, _I, _P, _I, _I, _P, _I, _D, _I, _D, _P]),
    "ebz_compress_trial_finish": (_I, [_P, _I, _P, _P]),
    "ebz_last_error": (ctypes.c_char_p, []),
    "ebz_device_info": (_I, [_P, ctypes.POINTER(_I), ctypes.c_char_p, _I]),
    "ebz_grid_range": (_I, [_P, _P, _I, _U64, _I, _D, _I, _D, _P, _P]),
    "ebz_compress_scan": (_I, [_P, _P, _I, _I, _P, _I, _I, _P, _P, _P, _P, _P]),
    "ebz_decompress_scan": (_I, [_P, _P, _I, _I, _P, _I, _I, _P, _U64, _P, _P, _P]),
    "ebz_build_code": (_I, [_P, _P, _I, _P, _P, _P, _P]),
    "ebz_pack_bits": (_I, [_P, _P, _I, _U64, _P, _I, _P, _P, _P, _SZ, _P, _P, _P]),
    "ebz_unpack_bits": (_I, [_P, _P, _U64, _P, _I, _U64, _P, _P, _P]),
    "ebz_compress": (_I, [_P, _I, _P, _I, _I, _I, _P, _I, _I, _I, _D, _I, _D, _P, _INFO_P]),
    "ebz_compress_flags": (_I, [_P, _I, _P, _I, _I, _I, _P, _I, _I, _I, _I, _D, _I, _D, _P,
                                _INFO_P]),
    "ebz_tr_pack": (_I, [_P, _P, _U64, _I, _D, _P, _U64, _P]),
    "ebz_tr_unpack": (_I, [_P, _P, _U64, _U64, _I, _D, _P]),
    "ebz_compress_async": (_I, [_P, _I, _P, _I, _I, _P, _I, _I, _I, _D, _I, _D, _P]),
    "ebz_compress_fetch": (_I, [_P, _I, _P, _P, _P, _P]),
    "ebz_compress_outputs": (_I, [_P, _I, _P, _P, _P, _P]),
    "ebz_decompress": (_I, [_P, _I, _I, _I, _I, _P, _I, _I, _D, _P, _P, _U64, _P, _U64, _P,
                            _P, _INFO_P]),
    "ebz_decompress_async": (_I, [_P, _I, _I, _P, _P]),
    "ebz_compress_batch": (_I, [_P, _I, _I, _P, _I, _I, _P, _I, _I, _I, _D, _I, _D, _P]),
    "ebz_decompress_batch": (_I, [_P, _I, _I, _I, _P, _P]),
    "ebz_decompress_batch_ptrs": (_I, [_P, _I, _I, _I, _I, _P, _I, _I, _P, _P, _P, _P, _P, _P,
                                       _P, _P]),
    "ebz_copy_async": (_I, [_P, _P, _P, _SZ, _P]),
    "ebz_slot_info_async": (_I, [_P, _I, _I, _P, _P]),
    "ebz_compress_fetch_async": (_I, [_P, _I, _P, _P, _P, _P, _P]),
    "ebz_original_hits": (_I, [_P, _P, _I, _I, _P, _I, _D, _P, _P]),
    "ebz_metrics": (_I, [_P, _P, _P, _I, _U64, _I, _P, _P]),
    "ebz_slot_info": (_I, [_P, _I, _INFO_P, _P]),
    "ebz_slot_decode_info": (_I, [_P, _I, _INFO_P, _P]),
    "ebz_launch_count": (ctypes.c_ulonglong, [_P]),
    "ebz_debug_set_epoch": (ctypes.c_uint, [_P, ctypes.c_uint]),
    "ebz_epoch_max": (ctypes.c_uint, []),
    "ebz_sweep_kernel_choice": (_I, [_I, _I, _P, _I, _I, _I]),
    "ebz_profile": (_I, [_P, _I]),
    "ebz_stage_times": (_I, [_P, _P, _P, _I]),
    # reference kernel seam on host buffers (kernels.py)
    "ebz_ref_compress_scan": (_I, [_P, _P, _I, _P, _P, _P, _P, _I64, _P, _P, _I64, _P, _I,
                                   _I64, _I64, _D, _P]),
    "ebz_ref_decompress_scan": (_I, [_P, _P, _P, _I, _P, _U64, _P, _P, _I64, _P, _P, _I64,
                                     _P, _I, _I64, _I64, _D, _P]),
    "ebz_ref_pack_bits": (_I, [_P, _P, _U64, _P, _P, _U64, _P, _U64, _P]),
    "ebz_ref_unpack_bits": (_I, [_P, _P, _U64, _U64, _P, _P, _P, _P, _U64, _I, _P, _U64, _P]),
    "ebz_ref_original_hits": (_I, [_P, _P, _I, _P, _P, _I64, _P, _P, _I64, _P, _I, _I64, _D,
                                   _P]),
}

_lib = None
_lib_lock = threading.Lock()
_ctx = {}


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Open the library and bind every exported symbol (no device needed)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: run `python -m paper_1706_03791_b200._build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load_library().ebz_last_error()
    return msg.decode() if msg else ""


class Context:
    """One device context (workspace slots live on the C side)."""

    def __init__(self, device: int = 0):
        lib = load_library()
        handle = lib.ebz_ctx_create(device)
        if not handle:
            raise NativeUnavailable(f"no usable B200 device {device}: {last_error()}")
        self.lib = lib
        self.handle = handle
        self.device = device
        self.lock = threading.RLock()
        sms = _I(0)
        name = ctypes.create_string_buffer(128)
        lib.ebz_device_info(handle, ctypes.byref(sms), name, 128)
        self.sms = sms.value
        self.name = name.value.decode()

    def check(self, rc: int, what: str):
        if rc != 0:
            raise RuntimeError(f"{what} failed ({rc}): {last_error()}")

    def launches(self) -> int:
        return int(self.lib.ebz_launch_count(self.handle))

    def trim(self):
        """Give every workspace back to the driver (ebz_ctx_trim)."""
        with self.lock:
            self.check(self.lib.ebz_ctx_trim(self.handle), "ebz_ctx_trim")

    def close(self):
        if self.handle:
            self.lib.ebz_ctx_destroy(self.handle)
            self.handle = None


def context(device: int | None = None) -> Context:
    """Process-wide context for a device (created on first use)."""
    if device is None:
        device = int(os.environ.get("EBZ_DEVICE", "0"))
    with _lib_lock:
        ctx = _ctx.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lib_lock:
            _ctx.setdefault(device, ctx)
            ctx = _ctx[device]
    return ctx


def tr_pack(values, width: int, eb: float, device: int | None = None) -> bytes:
    """Version-2 unpredictable block of `values` (ebz_tr_pack, opt-in)."""
    import numpy as np
    ctx = context(device)
    v = np.ascontiguousarray(values, np.float64 if width == 64 else np.float32)
    nbits = ctypes.c_uint64(0)
    with ctx.lock:
        ctx.check(ctx.lib.ebz_tr_pack(ctx.handle, ptr(v) if v.size else None, v.size, width,
                                      float(eb), None, 0, ctypes.byref(nbits)), "ebz_tr_pack")
        out = np.zeros(max(1, (nbits.value + 7) // 8), np.uint8)
        ctx.check(ctx.lib.ebz_tr_pack(ctx.handle, ptr(v) if v.size else None, v.size, width,
                                      float(eb), ptr(out), out.size, ctypes.byref(nbits)),
                  "ebz_tr_pack")
    return out[: (nbits.value + 7) // 8].tobytes()


def tr_unpack(block: bytes, k: int, width: int, eb: float, device: int | None = None):
    """Values of a version-2 unpredictable block (ebz_tr_unpack, opt-in)."""
    import numpy as np
    ctx = context(device)
    src = np.frombuffer(bytes(block), np.uint8) if len(block) else np.zeros(1, np.uint8)
    out = np.empty(k, np.float64 if width == 64 else np.float32)
    with ctx.lock:
        rc = ctx.lib.ebz_tr_unpack(ctx.handle, ptr(src), len(block), k, width, float(eb),
                                   ptr(out) if k else None)
    if rc != 0:
        from .core import PayloadMismatchError
        raise PayloadMismatchError(last_error())
    return out


def ptr(array) -> ctypes.c_void_p:
    """Raw address of a numpy array / bytes-backed array."""
    return ctypes.c_void_p(array.ctypes.data)


def dims_array(dims) -> ctypes.Array:
    arr = (ctypes.c_uint64 * 4)(*([int(v) for v in dims] + [1] * (4 - len(dims))))
    return arr


def to_device(array, ctx: "Context"):
    """Device copy of a host numpy array as a torch tensor (plain buffer;
    works for read-only arrays, synchronous)."""
    import numpy as np
    import torch
    a = np.ascontiguousarray(array)
    dt = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}.get(
        a.dtype, torch.uint8)
    shape = (a.size,) if dt != torch.uint8 else (a.nbytes,)
    t = torch.empty(shape, dtype=dt, device=torch.device("cuda", ctx.device))
    if a.nbytes:
        ctx.check(ctx.lib.ebz_copy_async(ctx.handle, ctypes.c_void_p(t.data_ptr()),
                                         ctypes.c_void_p(a.ctypes.data), a.nbytes, None),
                  "ebz_copy_async")
        torch.cuda.synchronize(t.device)
    return t

