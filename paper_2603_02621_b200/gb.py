"""Thin ctypes binding of libgb (include/gb.h): argument marshalling only.

Every step of the verification path runs in libgb's CUDA kernels; PyTorch is
used only for device memory (workspace / result / dump tensors), the CUDA stream
handle and, in dist.py, the process group.  There is no CPU fallback: if
libgb.so is missing or cannot load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_PATH = os.environ.get("GB_LIB") or os.path.join(PKG, "libgb.so")   # GB_LIB: A/B experiments
HEADER = os.path.join(ROOT, "include", "gb.h")

# status codes and result layout, parsed from the header (single source of truth)
_hdr = open(HEADER).read()
_defs = {m.group(1): m.group(2) for m in re.finditer(r"#define\s+(GB_\w+)\s+([^\s/]+)", _hdr)}


def _c_int(v: str) -> int:
    return int(v.rstrip("uUlL"), 0)


GB_OK, GB_EINVAL, GB_ERANGE, GB_EWORKSPACE, GB_ECUDA, GB_EINTERNAL = range(6)
R_VERSION = _c_int(_defs["GB_R_VERSION"])
R_EVENS = _c_int(_defs["GB_R_EVENS"])
R_VERIFIED = _c_int(_defs["GB_R_VERIFIED"])
R_FASTPATH_UNRESOLVED = _c_int(_defs["GB_R_FASTPATH_UNRESOLVED"])
R_UNRESOLVED = _c_int(_defs["GB_R_UNRESOLVED"])
R_SUM_PMIN = _c_int(_defs["GB_R_SUM_PMIN"])
R_FIRST_UNRESOLVED_N = _c_int(_defs["GB_R_FIRST_UNRESOLVED_N"])
R_MAX_KEY = _c_int(_defs["GB_R_MAX_KEY"])
R_MAX_PMIN_RAW = _c_int(_defs["GB_R_MAX_PMIN_RAW"])
R_HIST = _c_int(_defs["GB_R_HIST"])
NBINS = _c_int(_defs["GB_NBINS"])
RESULT_WORDS = R_HIST + NBINS
KEY_SHIFT = _c_int(_defs["GB_KEY_SHIFT"])
KEY_PMAX = _c_int(_defs["GB_KEY_PMAX"])
PMAX_LIMIT = _c_int(_defs["GB_PMAX_LIMIT"])
RESULT_VERSION = _c_int(_defs["GB_RESULT_VERSION"])
U64_MAX = (1 << 64) - 1
INT64_MAX = (1 << 63) - 1

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
_lib = ctypes.CDLL(LIB_PATH)

_u64, _u32, _sz, _vp = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_size_t, ctypes.c_void_p
_sigs = {
    "gb_ctx_workspace_bytes": (_sz, [_u64, _u32]),
    "gb_ctx_create": (ctypes.c_int, [ctypes.POINTER(_vp), ctypes.c_int, _u64, _u64, _u32, _vp, _sz, _vp]),
    "gb_ctx_destroy": (None, [_vp]),
    "gb_ctx_info": (ctypes.c_int, [_vp, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
    "gb_ctx_tables": (ctypes.c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    "gb_sieve_segment": (ctypes.c_int, [_vp, _u64, _u64, _vp, _vp]),
    "gb_result_init": (ctypes.c_int, [_vp, _vp]),
    "gb_result_finalize": (ctypes.c_int, [_vp, _vp]),
    "gb_verify_range": (ctypes.c_int, [_vp, _u64, _u64, _u32, _vp, _vp, _vp]),
    "gb_verify_range_ex": (ctypes.c_int, [_vp, _u64, _u64, _u32, _u64, _vp, _vp, _vp]),
    "gb_verify_range_host": (ctypes.c_int, [_vp, _u64, _u64, _u32, _vp, _vp, _vp]),
    "gb_verify_range_pern": (ctypes.c_int, [_vp, _u64, _u64, _u32, _vp, _vp, _vp]),
    "gb_verify_range_resident": (ctypes.c_int, [_vp, _u64, _u64, _u32, _vp, _u64, _vp, _vp, _vp]),
    "gb_single_check": (ctypes.c_int, [_vp, _u64, _u64, _vp, _vp]),
    "gb_partition_counts": (ctypes.c_int, [_vp, _u64, _u64, _vp, _u64, _vp, _vp]),
    "gb_is_prime_u64": (ctypes.c_int, [_vp, _vp, _u64, _vp]),
    "gb_launch_count": (_u64, []),
    "gb_status_string": (ctypes.c_char_p, [ctypes.c_int]),
}
for _name, (_res, _args) in _sigs.items():
    _f = getattr(_lib, _name)          # raises if the library lacks a declared entry point
    _f.restype = _res
    _f.argtypes = _args


class GBError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {_lib.gb_status_string(status).decode()} ({status})")
        self.status = status


def _check(st: int, what: str) -> None:
    if st != GB_OK:
        raise GBError(st, what)


def _ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr() if hasattr(t, "data_ptr") else int(t)


# ---- C-ABI names, one-to-one ------------------------------------------------
def gb_ctx_workspace_bytes(hi_max: int, p_max: int) -> int:
    return int(_lib.gb_ctx_workspace_bytes(hi_max, p_max))


def gb_ctx_create(device: int, origin: int, hi_max: int, p_max: int, workspace, stream) -> int:
    out = _vp()
    nbytes = workspace.numel() * workspace.element_size()
    _check(_lib.gb_ctx_create(ctypes.byref(out), device, origin, hi_max, p_max, _ptr(workspace),
                              nbytes, _ptr_stream(stream)), "gb_ctx_create")
    return out.value


def gb_ctx_destroy(ctx: int) -> None:
    _lib.gb_ctx_destroy(ctx)


def gb_ctx_info(ctx: int) -> tuple[int, int]:
    n, r = _u64(), _u64()
    _check(_lib.gb_ctx_info(ctx, ctypes.byref(n), ctypes.byref(r)), "gb_ctx_info")
    return n.value, r.value


def gb_ctx_tables(ctx: int) -> tuple[int, int]:
    b, p = _vp(), _vp()
    _check(_lib.gb_ctx_tables(ctx, ctypes.byref(b), ctypes.byref(p)), "gb_ctx_tables")
    return b.value, p.value


def gb_sieve_segment(ctx: int, word_lo: int, n_words: int, d_words, stream) -> None:
    _check(_lib.gb_sieve_segment(ctx, word_lo, n_words, _ptr(d_words), _ptr_stream(stream)),
           "gb_sieve_segment")


def gb_result_init(d_result, stream) -> None:
    _check(_lib.gb_result_init(_ptr(d_result), _ptr_stream(stream)), "gb_result_init")


def gb_result_finalize(d_result, stream) -> None:
    _check(_lib.gb_result_finalize(_ptr(d_result), _ptr_stream(stream)), "gb_result_finalize")


def gb_verify_range(ctx: int, lo: int, hi: int, p_max: int, d_result, d_dump, stream) -> None:
    _check(_lib.gb_verify_range(ctx, lo, hi, p_max, _ptr(d_result), _ptr(d_dump),
                                _ptr_stream(stream)), "gb_verify_range")


def gb_verify_range_pern(ctx: int, lo: int, hi: int, p_max: int, d_result, d_dump, stream) -> None:
    _check(_lib.gb_verify_range_pern(ctx, lo, hi, p_max, _ptr(d_result), _ptr(d_dump), _ptr_stream(stream)),
           "gb_verify_range_pern")


def gb_verify_range_resident(ctx: int, lo: int, hi: int, p_max: int, d_bits, n_words: int, d_result, d_dump,
                             stream) -> None:
    _check(_lib.gb_verify_range_resident(ctx, lo, hi, p_max, _ptr(d_bits), n_words, _ptr(d_result), _ptr(d_dump),
                                         _ptr_stream(stream)), "gb_verify_range_resident")


def gb_single_check(ctx: int, n: int, p_limit: int, d_out, stream) -> None:
    _check(_lib.gb_single_check(ctx, n, p_limit, _ptr(d_out), _ptr_stream(stream)), "gb_single_check")


def gb_partition_counts(ctx: int, lo: int, hi: int, d_bits, n_words: int, d_counts, stream) -> None:
    _check(_lib.gb_partition_counts(ctx, lo, hi, _ptr(d_bits), n_words, _ptr(d_counts), _ptr_stream(stream)),
           "gb_partition_counts")


def gb_verify_range_ex(ctx: int, lo: int, hi: int, p_max: int, cap: int, d_result, d_dump,
                       stream) -> None:
    _check(_lib.gb_verify_range_ex(ctx, lo, hi, p_max, cap, _ptr(d_result), _ptr(d_dump),
                                   _ptr_stream(stream)), "gb_verify_range_ex")


def gb_verify_range_host(ctx: int, lo: int, hi: int, p_max: int, h_result, h_dump, stream) -> None:
    """h_result / h_dump: host buffers (numpy arrays or pinned torch CPU tensors)."""
    def hp(a):
        if a is None:
            return None
        return a.ctypes.data if hasattr(a, "ctypes") else a.data_ptr()
    _check(_lib.gb_verify_range_host(ctx, lo, hi, p_max, hp(h_result), hp(h_dump),
                                     _ptr_stream(stream)), "gb_verify_range_host")


def gb_is_prime_u64(d_x, d_out, n: int, stream) -> None:
    _check(_lib.gb_is_prime_u64(_ptr(d_x), _ptr(d_out), n, _ptr_stream(stream)), "gb_is_prime_u64")


def gb_launch_count() -> int:
    return int(_lib.gb_launch_count())


def gb_status_string(s: int) -> str:
    return _lib.gb_status_string(s).decode()


def _ptr_stream(stream) -> int | None:
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


# ---- result decoding (host side, plain integer bookkeeping) ------------------
def decode_result(words, origin: int = 0) -> dict:
    """Decode a finalized GB_RESULT_WORDS int64 vector into named fields.
    (The exact sum n * p_min, the position-sensitive check, comes from a per-n
    dump; the result vector carries no checksum.)  If some p_min
    reached GB_KEY_PMAX the key's p field saturates: max_pmin is then the raw
    maximum and max_pmin_n is -1 (unknown)."""
    w = [int(x) for x in (words.tolist() if hasattr(words, "tolist") else words)]
    if w[R_VERSION] != RESULT_VERSION:
        raise ValueError("result vector has a bad version word (not initialised?)")
    key = w[R_MAX_KEY]
    if key:
        p = key >> KEY_SHIFT
        idx = (1 << KEY_SHIFT) - 1 - (key & ((1 << KEY_SHIFT) - 1))
        max_p, max_n = p, origin + 2 * idx
    else:
        max_p, max_n = 0, 0
    if w[R_MAX_PMIN_RAW] > max_p:
        max_p, max_n = w[R_MAX_PMIN_RAW], -1
    out = {
        "evens": w[R_EVENS], "verified": w[R_VERIFIED],
        "fastpath_unresolved": w[R_FASTPATH_UNRESOLVED], "unresolved": w[R_UNRESOLVED],
        "first_unresolved_n": w[R_FIRST_UNRESOLVED_N], "max_pmin": max_p, "max_pmin_n": max_n,
        "sum_pmin": w[R_SUM_PMIN],
    }
    out["hist"] = w[R_HIST:R_HIST + NBINS]
    return out
