"""Test-side helpers: numpy views of generated batches and host-side placement.

Everything here is test infrastructure.  The arithmetic comparisons live in
the oracle (oracle/) or, for pins, in independent brute force code in the
test files themselves.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle
from paper_2509_08309_b200 import workload


def dtype_code(shape: workload.Shape) -> int:
    return oracle.BF16 if shape.dtype == "bf16" else oracle.F32


def host_batch(b: workload.DecodeBatch) -> dict:
    """numpy copies of one rank's batch with the new token placed by the oracle's kv_append."""
    out = {
        "q": workload.to_numpy_bits(b.q).copy(),
        "k_new": workload.to_numpy_bits(b.k_new).copy(),
        "v_new": workload.to_numpy_bits(b.v_new).copy(),
        "k_pool": workload.to_numpy_bits(b.k_pool).copy(),
        "v_pool": workload.to_numpy_bits(b.v_pool).copy(),
        "block_table": b.block_table.cpu().numpy().astype(np.int32),
        "seq_lens": b.seq_lens.cpu().numpy().astype(np.int32),
    }
    oracle.kv_append(out["k_new"], out["v_new"], out["k_pool"], out["v_pool"], out["block_table"],
                     out["seq_lens"])
    return out


def host_batch_once(b: workload.DecodeBatch) -> dict:
    """Like host_batch, but without the second host copy of the pools (full-size configs hold several GB):
    a device tensor's .cpu() is already a fresh, writable host buffer."""
    def bits(t):
        a = workload.to_numpy_bits(t)
        return a if t.is_cuda else a.copy()
    out = {k: bits(getattr(b, k)) for k in ("q", "k_new", "v_new", "k_pool", "v_pool")}
    out["block_table"] = b.block_table.cpu().numpy().astype(np.int32)
    out["seq_lens"] = b.seq_lens.cpu().numpy().astype(np.int32)
    oracle.kv_append(out["k_new"], out["v_new"], out["k_pool"], out["v_pool"], out["block_table"],
                     out["seq_lens"])
    return out


def to_f64(x: np.ndarray) -> np.ndarray:
    """Exact widening of stored bits (uint16 bf16 / float32) to float64 -- test side."""
    if x.dtype == np.uint16:
        return (x.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return x.astype(np.float64)


def oracle_full(b: workload.DecodeBatch, nthreads: int = 0) -> np.ndarray:
    """Oracle output [B][q_count][D] for this rank's heads (local head order)."""
    hb = host_batch(b)
    s = b.shape
    # the oracle sees a problem whose heads are this rank's heads: H' = q_count, Hkv' = kv_count
    return oracle.decode(hb["q"], hb["k_pool"], hb["v_pool"], hb["block_table"], hb["seq_lens"],
                         num_kv_heads=b.kv_count, dtype=dtype_code(s), nthreads=nthreads)


def dense_logical_kv(hb: dict, P: int):
    """Walk the block table page by page and return per (j, g) dense [L][D] float64 K and V."""
    bt, lens = hb["block_table"], hb["seq_lens"]
    K = to_f64(hb["k_pool"])
    V = to_f64(hb["v_pool"])
    B, G, _ = bt.shape
    ks, vs = {}, {}
    for j in range(B):
        L = int(lens[j])
        for g in range(G):
            rows_k, rows_v = [], []
            for p in range((L + P - 1) // P):
                page = int(bt[j, g, p])
                for slot in range(P):
                    if p * P + slot >= L:
                        break
                    rows_k.append(K[page, slot])
                    rows_v.append(V[page, slot])
            ks[j, g] = np.stack(rows_k)
            vs[j, g] = np.stack(rows_v)
    return ks, vs


def err_stats(got: np.ndarray, ref: np.ndarray) -> dict:
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    diff = np.abs(got - ref)
    idx = np.unravel_index(int(np.argmax(diff)), diff.shape) if diff.size else ()
    return {
        "max_abs": float(diff.max()) if diff.size else 0.0,
        "argmax": tuple(int(i) for i in idx),
        "rel_fro": float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)),
        "nonfinite": int((~np.isfinite(got)).sum()),
    }


def small_batch(H=8, Hkv=8, D=8, P=4, dtype="f32", lens=(5, 1, 13, 40), seed=3, q_begin=0, q_count=None,
                rank_salt=0):
    shape = workload.Shape(H, Hkv, D, P, dtype)
    return workload.make_decode_batch(shape, torch.tensor(lens, dtype=torch.int32), seed, "cpu",
                                      q_begin=q_begin, q_count=q_count, rank_salt=rank_salt)
