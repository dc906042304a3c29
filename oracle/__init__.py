"""oracle -- TEST INFRASTRUCTURE ONLY.

Plain fp64 CPU reference for Hetis' head-granular paged decode Attention
(arXiv 2509.08309, Eq. 2a/2b PAPER.md:363-372, head-granular pages PAPER.md:539).
The arithmetic lives in ``oracle.c`` (see its header for the per-function
citations); this module only compiles it with gcc and marshals numpy arrays.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  It never imports
``paper_2509_08309_b200`` and that package never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

F32 = 0
BF16 = 1

_ERRORS = {
    -1: "invalid argument",
    -2: "empty sequence (seq_len < 1): softmax over the empty set",
    -3: "page id outside [0, num_pages)",
    -4: "seq_len > max_pages * page_size",
}


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, -O2, OpenMP).  Returns the path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fopenmp", "-shared", "-fPIC",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            i32, i64, vp, dp = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p
            lib.oracle_decode_f64.argtypes = [i32] * 6 + [vp, vp, vp, i64, vp, i32, vp, dp, i32]
            lib.oracle_decode_pairs_f64.argtypes = [i32] * 6 + [vp, vp, vp, i64, vp, i32, vp, i64, vp, dp, i32]
            lib.oracle_decode_range_f64.argtypes = [i32] * 6 + [vp, vp, vp, i64, vp, i32, vp,
                                                               i32, i32, i32, i32, dp, dp]
            lib.oracle_kv_append.argtypes = [i32] * 5 + [vp, vp, vp, vp, i64, vp, i32, vp]
            lib.oracle_lse_merge_f64.argtypes = [i32, i32, dp, dp, dp, dp]
            lib.oracle_kv_migrate.argtypes = [i32, vp, i32, i32, i32, vp, vp, i64, vp, i32, vp, vp, i64, vp, i32]
            for f in (lib.oracle_decode_f64, lib.oracle_decode_pairs_f64, lib.oracle_decode_range_f64,
                      lib.oracle_kv_append, lib.oracle_lse_merge_f64, lib.oracle_kv_migrate):
                f.restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int):
    if rc != 0:
        raise OracleError(_ERRORS.get(rc, f"oracle error {rc}"))


def _as_storage(x: np.ndarray, dtype: int) -> np.ndarray:
    """bf16 data travels as uint16 bit patterns; fp32 as float32."""
    if dtype == BF16:
        if x.dtype != np.uint16:
            raise TypeError("bf16 arrays must be passed as uint16 bit patterns")
    elif x.dtype != np.float32:
        raise TypeError("fp32 arrays must be float32")
    return np.ascontiguousarray(x)


def decode(q, k_pool, v_pool, block_table, seq_lens, *, num_kv_heads: int, dtype: int,
           nthreads: int = 0) -> np.ndarray:
    """Full fp64 output [B][H][D] (global head order).

    q: [B][H][D]; k_pool, v_pool: [num_pages][P][D]; block_table: int32
    [B][Hkv][max_pages]; seq_lens: int32 [B].  bf16 arrays as uint16 bits.
    """
    q = _as_storage(q, dtype)
    k_pool = _as_storage(k_pool, dtype)
    v_pool = _as_storage(v_pool, dtype)
    bt = np.ascontiguousarray(block_table, dtype=np.int32)
    sl = np.ascontiguousarray(seq_lens, dtype=np.int32)
    B, H, D = q.shape
    num_pages, P, D2 = k_pool.shape
    assert D2 == D and v_pool.shape == k_pool.shape
    assert bt.shape[0] == B and bt.shape[1] == num_kv_heads and sl.shape == (B,)
    out = np.empty((B, H, D), dtype=np.float64)
    _check(_load().oracle_decode_f64(B, H, num_kv_heads, D, P, dtype, _ptr(q), _ptr(k_pool), _ptr(v_pool),
                                     num_pages, _ptr(bt), bt.shape[2], _ptr(sl), _ptr(out), nthreads))
    return out


def decode_pairs(q, k_pool, v_pool, block_table, seq_lens, pairs, *, num_kv_heads: int, dtype: int,
                 nthreads: int = 0) -> np.ndarray:
    """fp64 outputs [n_pairs][D] for (seq, global head) pairs."""
    q = _as_storage(q, dtype)
    k_pool = _as_storage(k_pool, dtype)
    v_pool = _as_storage(v_pool, dtype)
    bt = np.ascontiguousarray(block_table, dtype=np.int32)
    sl = np.ascontiguousarray(seq_lens, dtype=np.int32)
    pr = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
    B, H, D = q.shape
    num_pages, P, _ = k_pool.shape
    out = np.empty((pr.shape[0], D), dtype=np.float64)
    _check(_load().oracle_decode_pairs_f64(B, H, num_kv_heads, D, P, dtype, _ptr(q), _ptr(k_pool),
                                           _ptr(v_pool), num_pages, _ptr(bt), bt.shape[2], _ptr(sl),
                                           pr.shape[0], _ptr(pr), _ptr(out), nthreads))
    return out


def decode_range(q, k_pool, v_pool, block_table, seq_lens, j: int, h: int, t0: int, t1: int, *,
                 num_kv_heads: int, dtype: int):
    """(o [D], lse) of head (j, h) over tokens [t0, t1) only."""
    q = _as_storage(q, dtype)
    k_pool = _as_storage(k_pool, dtype)
    v_pool = _as_storage(v_pool, dtype)
    bt = np.ascontiguousarray(block_table, dtype=np.int32)
    sl = np.ascontiguousarray(seq_lens, dtype=np.int32)
    B, H, D = q.shape
    num_pages, P, _ = k_pool.shape
    out = np.empty((D,), dtype=np.float64)
    lse = np.empty((1,), dtype=np.float64)
    _check(_load().oracle_decode_range_f64(B, H, num_kv_heads, D, P, dtype, _ptr(q), _ptr(k_pool),
                                           _ptr(v_pool), num_pages, _ptr(bt), bt.shape[2], _ptr(sl),
                                           j, h, t0, t1, _ptr(out), _ptr(lse)))
    return out, float(lse[0])


def lse_merge(o_parts: np.ndarray, lse_parts: np.ndarray):
    """Merge [S][D] partial results with natural-log normalisers [S] -> (o [D], lse)."""
    o = np.ascontiguousarray(o_parts, dtype=np.float64)
    l = np.ascontiguousarray(lse_parts, dtype=np.float64)
    S, D = o.shape
    out = np.empty((D,), dtype=np.float64)
    lse = np.empty((1,), dtype=np.float64)
    _check(_load().oracle_lse_merge_f64(S, D, _ptr(o), _ptr(l), _ptr(out), _ptr(lse)))
    return out, float(lse[0])


def kv_append(k_new, v_new, k_pool, v_pool, block_table, seq_lens) -> None:
    """In-place head-granular store of the new token's K/V rows.

    k_new, v_new: [B][Hkv][D]; pools [num_pages][P][D] (same element type,
    uint16 for bf16 or float32); modified in place.
    """
    assert k_pool.flags.c_contiguous and v_pool.flags.c_contiguous
    k_new = np.ascontiguousarray(k_new)
    v_new = np.ascontiguousarray(v_new)
    bt = np.ascontiguousarray(block_table, dtype=np.int32)
    sl = np.ascontiguousarray(seq_lens, dtype=np.int32)
    B, Hkv, D = k_new.shape
    num_pages, P, _ = k_pool.shape
    eb = k_pool.dtype.itemsize
    _check(_load().oracle_kv_append(B, Hkv, D, P, eb, _ptr(k_new), _ptr(v_new), _ptr(k_pool), _ptr(v_pool),
                                    num_pages, _ptr(bt), bt.shape[2], _ptr(sl)))


def kv_migrate(entries, src_k, src_v, src_bt, dst_k, dst_v, dst_bt) -> None:
    """Token-by-token copy of migrated (request, kv head) caches, in place on
    dst_k / dst_v.  entries: int32 [n][3] (src_row, dst_row, num_tokens); tables are [rows][max_pages]
    (any leading shape, flattened); pools [num_pages][P][D], same element type (uint16 / float32)."""
    assert dst_k.flags.c_contiguous and dst_v.flags.c_contiguous
    en = np.ascontiguousarray(entries, dtype=np.int32).reshape(-1, 3)
    src_k, src_v = np.ascontiguousarray(src_k), np.ascontiguousarray(src_v)
    sbt = np.ascontiguousarray(src_bt, dtype=np.int32)
    dbt = np.ascontiguousarray(dst_bt, dtype=np.int32)
    _, P, D = src_k.shape
    assert dst_k.shape[1:] == (P, D) and src_k.dtype == dst_k.dtype
    _check(_load().oracle_kv_migrate(en.shape[0], _ptr(en), D, P, src_k.dtype.itemsize, _ptr(src_k), _ptr(src_v),
                                     src_k.shape[0], _ptr(sbt), sbt.shape[-1], _ptr(dst_k), _ptr(dst_v),
                                     dst_k.shape[0], _ptr(dbt), dbt.shape[-1]))
