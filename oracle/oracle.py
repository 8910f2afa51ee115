"""ctypes binding for the CPU oracle (oracle/gb_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package
paper_2603_02621_b200/.  It shares no code with that package; the only shared
artifact is the list of result field names.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "gb_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
NBINS = 6544
U64_MAX = (1 << 64) - 1
FIELDS = ("evens", "verified", "fastpath_unresolved", "unresolved",
          "first_unresolved_n", "max_pmin", "max_pmin_n", "sum_pmin", "chk")
# the aggregates libgb's result vector carries (chk = sum n*p_min needs the per-n
# values: tests compare it through dumps, see chk_of_dump)
AGG_FIELDS = tuple(f for f in FIELDS if f != "chk")


class OrResult(ctypes.Structure):
    _fields_ = [("evens", ctypes.c_int64), ("verified", ctypes.c_int64),
                ("fastpath_unresolved", ctypes.c_int64), ("unresolved", ctypes.c_int64),
                ("first_unresolved_n", ctypes.c_int64), ("max_pmin", ctypes.c_int64),
                ("max_pmin_n", ctypes.c_int64), ("sum_pmin", ctypes.c_int64),
                ("chk", ctypes.c_uint64), ("hist", ctypes.c_int64 * NBINS)]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (the checker is built, not used, by build())."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = f"{LIB}.{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-pthread", "-shared",
                               "-fPIC", SRC, "-o", tmp])
        os.replace(tmp, LIB)      # new inode: never rewrite a library a running process maps
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        L.or_isqrt.restype = ctypes.c_uint64
        L.or_isqrt.argtypes = [ctypes.c_uint64]
        L.or_is_prime_td.restype = ctypes.c_int
        L.or_is_prime_td.argtypes = [ctypes.c_uint64]
        L.or_verify.restype = ctypes.c_int
        L.or_verify.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(OrResult),
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64]
        L.or_sieve_window.restype = ctypes.c_int
        L.or_sieve_window.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p]
        L.or_prime_pi.restype = ctypes.c_uint64
        L.or_prime_pi.argtypes = [ctypes.c_uint64, ctypes.c_int]
        L.or_partition_counts.restype = ctypes.c_int
        L.or_partition_counts.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
        L.or_result_size.restype = ctypes.c_size_t
        assert L.or_result_size() == ctypes.sizeof(OrResult)
        _lib = L
    return _lib


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def isqrt(x: int) -> int:
    return int(lib().or_isqrt(x))


def is_prime_td(x: int) -> bool:
    return bool(lib().or_is_prime_td(x))


def prime_pi(x: int, threads: int | None = None) -> int:
    r = int(lib().or_prime_pi(x, threads or default_threads()))
    if r == U64_MAX:
        raise MemoryError("or_prime_pi failed")
    return r


def sieve_window(a: int, b: int) -> np.ndarray:
    """uint8 array, one entry per odd q in [a, b) (a odd): 1 iff q prime."""
    out = np.zeros(max(0, (b - a + 1) // 2), dtype=np.uint8)
    rc = lib().or_sieve_window(a, b, out.ctypes.data if out.size else None)
    if rc != 0:
        raise RuntimeError(f"or_sieve_window rc={rc}")
    return out


def lo_even(lo: int) -> int:
    return 4 if lo < 4 else lo + (lo & 1)


def n_evens(lo: int, hi: int) -> int:
    e = lo_even(lo)
    return 0 if hi <= e else (hi - e + 1) // 2


def verify(lo: int, hi: int, p_fast: int = 65521, cap: int = U64_MAX,
           threads: int | None = None, dump: bool = False, chunk_evens: int | None = None):
    """Aggregates (dict with FIELDS + 'hist') and optional per-n u32 dump.
    chunk_evens (a power of two): also out['chunk_chk'], a uint64 array with the
    chk (sum n * p_min mod 2^64) of each chunk of that many evens from lo_e."""
    res = OrResult()
    ne = n_evens(lo, hi)
    d = np.zeros(ne, dtype=np.uint32) if dump else None
    ch = None
    if chunk_evens:
        ch = np.zeros(max(1, -(-ne // chunk_evens)), dtype=np.uint64)
    rc = lib().or_verify(lo, hi, p_fast, cap, threads or default_threads(), ctypes.byref(res),
                         d.ctypes.data if (d is not None and d.size) else None,
                         ch.ctypes.data if ch is not None else None, chunk_evens or 0)
    if rc != 0:
        raise RuntimeError(f"or_verify rc={rc}")
    out = {f: int(getattr(res, f)) for f in FIELDS}
    out["hist"] = np.ctypeslib.as_array(res.hist).copy()
    if ch is not None:
        out["chunk_chk"] = ch
    return out, d


def partition_counts(lo: int, hi: int, threads: int | None = None) -> np.ndarray:
    """c(n) = #{p prime <= n/2 : n - p prime} for every even n in [lo_e, hi)
    (NEXT-4; reading R13), as a uint64 array indexed (n - lo_e)/2."""
    out = np.zeros(n_evens(lo, hi), dtype=np.uint64)
    if out.size:
        rc = lib().or_partition_counts(lo, hi, threads or default_threads(), out.ctypes.data)
        if rc != 0:
            raise RuntimeError(f"or_partition_counts rc={rc}")
    return out
