"""ctypes binding of the C ABI in ``include/splitzip_b200.h``.

The product path has exactly one implementation: the sm_100a kernels in
``libsz_b200.so``.  If the library is missing, or no CUDA device is present,
every codec call raises :class:`NativeError` — there is no CPU fallback.
PyTorch provides device memory (caching allocator) and the current stream;
nothing torch-typed crosses the ABI (plain pointers, sizes, a stream handle).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import torch

from .errors import ConfigError, NativeError

LIB_PATH = Path(__file__).resolve().parent / "libsz_b200.so"
# A/B experiments only (scripts/ab_variants.sh): load a variant build of the
# same library from another in-tree path
if os.environ.get("SZ_LIB_VARIANT"):
    LIB_PATH = Path(__file__).resolve().parent / f"libsz_b200.{os.environ['SZ_LIB_VARIANT']}.so"
ABI_VERSION = 1

SZ_OK, SZ_ECONFIG, SZ_EWORKSPACE, SZ_EALIGN, SZ_ECUDA, SZ_EOUTPUT = range(6)
NUM_CHECKS = 13
(DEC_CODE_PAD, DEC_SM_PAD, DEC_VALUE_DOMAIN, DEC_VALUE_IN_BOOK, DEC_SENTINEL_COUNT,
 DEC_ABS_PAST_END, DEC_ABS_NOT_INC, DEC_COUNTS_TOTAL, DEC_POS_OVER_CHUNK,
 DEC_POS_PAST_END, DEC_POS_NOT_INC, DEC_CODE_RANGE, DEC_NONDUMMY) = range(NUM_CHECKS)
DEC_CAPACITY = 13   # flag only: device-resident M above the escape capacity


class SzParams(C.Structure):
    _fields_ = [("fmt", C.c_uint32), ("code_bits", C.c_uint32), ("sentinel", C.c_uint32),
                ("abs32", C.c_uint32), ("chunk_size", C.c_uint32), ("n_entries", C.c_uint32),
                ("enc_lut", C.c_uint8 * 256), ("dec_lut", C.c_uint8 * 16)]


class SzEncoded(C.Structure):
    _fields_ = [("d_codes", C.c_void_p), ("d_sm", C.c_void_p), ("d_counts", C.c_void_p),
                ("d_positions", C.c_void_p), ("d_values", C.c_void_p),
                ("d_values_packed", C.c_void_p), ("d_n_escapes", C.c_void_p),
                ("escape_capacity", C.c_uint64), ("d_escape_base", C.c_void_p)]


class SzEncodedIn(C.Structure):
    _fields_ = [("d_codes", C.c_void_p), ("d_sm", C.c_void_p), ("d_counts", C.c_void_p),
                ("d_positions", C.c_void_p), ("d_values", C.c_void_p),
                ("n_elements", C.c_uint64), ("n_escapes", C.c_uint64), ("n_counts", C.c_uint64),
                ("d_n_escapes", C.c_void_p)]


class SzDecodeStatus(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("_pad", C.c_uint32),
                ("first_inv", C.c_uint64 * NUM_CHECKS), ("counts_total", C.c_uint64),
                ("marks_total", C.c_uint64)]


STATUS_BYTES = C.sizeof(SzDecodeStatus)

_P = C.c_void_p
_U64 = C.c_uint64
_U32 = C.c_uint32
_SIGNATURES = {
    "sz_abi_version": (C.c_int, []),
    "sz_last_cuda_error": (C.c_char_p, []),
    "sz_split_fields": (C.c_int, [_P, _U64, _U32, _P, _P, _P]),
    "sz_reconstruct": (C.c_int, [_P, _P, _U64, _U32, _P, _P]),
    "sz_pack_bits": (C.c_int, [_P, _U64, _U32, _P, _P]),
    "sz_unpack_bits": (C.c_int, [_P, _U64, _U32, _P, _P, _P]),
    "sz_max_u8": (C.c_int, [_P, _U64, _P, _P]),
    "sz_histogram_workspace_bytes": (C.c_size_t, [_U64, _U32]),
    "sz_histogram": (C.c_int, [_P, _U64, _U32, _P, _P, C.c_size_t, _P]),
    "sz_encode_workspace_bytes": (C.c_size_t, [_U64, C.POINTER(SzParams)]),
    "sz_encode": (C.c_int, [_P, _U64, C.POINTER(SzParams), C.POINTER(SzEncoded), _P,
                            C.c_size_t, _P]),
    "sz_decode_workspace_bytes": (C.c_size_t, [_U64, _U64, C.POINTER(SzParams)]),
    "sz_decode": (C.c_int, [C.POINTER(SzEncodedIn), C.POINTER(SzParams), _P, _P, _P,
                            C.c_size_t, _P]),
    "sz_check_values": (C.c_int, [_P, _U64, C.POINTER(SzParams), _P, _P]),
    "sz_compare": (C.c_int, [_P, _P, _U64, _U32, _P, _P]),
    "sz_group_members": (C.c_int, [_P, _U64, C.POINTER(SzParams), _U64, _P, _P]),
    "sz_synth_words": (C.c_int, [_P, _U64, _U32, _U64, _P, _P, _U32, _P]),
    "sz_encode_segments": (C.c_int, [_P, _U64, _U64, C.POINTER(SzParams), C.POINTER(SzEncoded),
                                     _P, C.c_size_t, _P]),
    "sz_encode_segments_va": (C.c_int, [_P, _U64, _U64, _U64, _U64, C.POINTER(SzParams),
                                        C.POINTER(SzEncoded), _P, C.c_size_t, _P]),
    "sz_decode_segments": (C.c_int, [C.POINTER(SzEncodedIn), C.POINTER(SzParams), _P, _U64, _U64,
                                     _P, _P, C.c_size_t, _P]),
    "sz_peer_signal": (C.c_int, [_P, _U64, _P]),
    "sz_peer_wait": (C.c_int, [_P, _U64, _U64, _P, _P]),
    "sz_device_alloc": (C.c_int, [_U64, C.POINTER(C.c_void_p)]),
    "sz_device_free": (C.c_int, [_P]),
    "sz_ipc_export": (C.c_int, [_P, _P]),
    "sz_ipc_import": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "sz_ipc_close": (C.c_int, [_P]),
    "sz_container_prefix_bytes": (C.c_size_t, [C.POINTER(SzParams)]),
    "sz_container_bytes": (_U64, [_U64, _U64, C.POINTER(SzParams)]),
    "sz_frame_container": (C.c_int, [C.POINTER(SzParams), _U64, C.POINTER(SzEncoded), _P, _U64,
                                     _P, _P]),
}
EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lock = threading.Lock()
_lib = None


def load_library(require_gpu: bool = True):
    """Load (once) and return the ctypes handle; raise NativeError when the
    library is absent or, with ``require_gpu``, when CUDA is unavailable."""
    global _lib
    if require_gpu and not torch.cuda.is_available():
        raise NativeError("SplitZip-B200 needs a CUDA device (sm_100a); none is visible")
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeError(
                    f"CUDA extension {LIB_PATH.name} is not built — run "
                    "`python -m paper_2605_01708_b200._build` (no CPU fallback exists)")
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.sz_abi_version() != ABI_VERSION:
                raise NativeError("libsz_b200.so ABI version mismatch; rebuild it")
            _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc == SZ_OK:
        return
    lib = load_library(require_gpu=False)
    if rc == SZ_ECONFIG:
        raise ConfigError(f"{what}: unsupported or inconsistent parameters")
    if rc == SZ_EALIGN:
        raise NativeError(f"{what}: misaligned device buffer")
    if rc == SZ_EWORKSPACE:
        raise NativeError(f"{what}: workspace too small")
    if rc == SZ_EOUTPUT:
        raise NativeError(f"{what}: output buffer too small")
    raise NativeError(f"{what}: CUDA error {lib.sz_last_cuda_error().decode()}")


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def aligned_device_copy(t: torch.Tensor, align: int = 32) -> torch.Tensor:
    """Contiguous CUDA tensor whose data pointer is ``align``-byte aligned."""
    load_library()  # no device / no library -> NativeError, never a CPU path
    if t.device.type != "cuda":
        t = t.to(device(), non_blocking=t.is_pinned())
    if not t.is_contiguous():
        t = t.contiguous()
    if t.data_ptr() % align:
        t = t.clone()
    return t
