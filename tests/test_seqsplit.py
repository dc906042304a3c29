"""CPU tests (`-m "not gpu"`) of the sequence-wise split (row f3): its host-side
bookkeeping, the oracle's log-sum-exp (pinned independently), and the split +
merge composition on one and two (gloo) processes.

The split is the alternative the paper argues against (PAPER.md:292-304,
:356-358): every device attends all heads over a subset of the tokens and the
results are merged with the per-head log-sum-exp.  Layout: page striping
(page k of every (request, kv head) on device k mod N; reading f3).
"""
from __future__ import annotations

import math
import os
import socket

import mpmath as mp
import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import oracle
from paper_2509_08309_b200 import seqsplit, workload
from tests.helpers import dense_logical_kv, dtype_code, host_batch, small_batch, to_f64


# ---------------------------------------------------------------- bookkeeping (brute force)
def _pages_of(L, N, rank, P):
    """Brute force: enumerate the token positions held by `rank` under page striping."""
    return [t for t in range(L) if (t // P) % N == rank]


@pytest.mark.parametrize("P", [4, 16])
def test_local_len_and_owner_match_enumeration(P):
    for N in (1, 2, 3, 5, 8):
        for L in list(range(0, 5 * P * N + 3)) + [32768, 10240, 4097]:
            held = [_pages_of(L, N, r, P) if L <= 4000 else None for r in range(N)]
            lens = [seqsplit.local_len(L, N, r, P) for r in range(N)]
            assert sum(lens) == L
            if held[0] is not None:
                assert lens == [len(h) for h in held]
            if L > 0:
                owner = seqsplit.owner_of_newest(L, N, P)
                assert ((L - 1) // P) % N == owner
                # only the owner's local last page is partial: its local length minus its full pages
                for r in range(N):
                    if r != owner:
                        assert lens[r] % P == 0


def test_local_tables_partition_the_global_pages():
    torch.manual_seed(0)
    B, G, maxp, P = 5, 3, 23, 16
    lens = torch.tensor([1, 16, 17, 300, 23 * 16], dtype=torch.int32)
    bt = torch.full((B, G, maxp), -1, dtype=torch.int32)
    ids = torch.randperm(B * G * maxp, dtype=torch.int64).to(torch.int32).view(B, G, maxp)
    for j in range(B):
        n = (int(lens[j]) + P - 1) // P
        bt[j, :, :n] = ids[j, :, :n]
    for N in (1, 2, 3, 8):
        seen = {}
        for r in range(N):
            lb = seqsplit.local_block_table(bt, N, r)
            for j in range(B):
                nl = (seqsplit.local_len(int(lens[j]), N, r, P) + P - 1) // P
                for g in range(G):
                    for m in range(nl):
                        pid = int(lb[j, g, m])
                        assert pid >= 0
                        seen.setdefault((j, g), []).append((r + m * N, pid))
                    assert bool((lb[j, g, nl:] == -1).all())
        for j in range(B):
            n = (int(lens[j]) + P - 1) // P
            for g in range(G):
                got = sorted(seen.get((j, g), []))
                assert got == [(k, int(bt[j, g, k])) for k in range(n)]


def test_comm_bytes_head_split_matches_eq4():
    """Head split volume per device: (2 + 2/r) * x * d elements (Eq. 4; q + o + k + v)."""
    shape = workload.LLAMA2_70B
    B, N = 128, 8
    c = seqsplit.comm_bytes(B, shape, N, o_bytes=2)
    x = shape.num_q_heads // N
    eq4 = B * (2 + 2 / shape.r) * x * shape.head_dim * 2     # q in + k, v in + own o out, bf16
    assert c["head_in"] + c["head_out"] / (N - 1) == pytest.approx(eq4)


# ---------------------------------------------------------------- oracle lse pins
def _brute_lse(q, K, scale):
    mp.mp.dps = 50
    return float(mp.log(mp.fsum(mp.exp(mp.fsum(mp.mpf(a) * mp.mpf(b) for a, b in zip(q, K[t])) * scale)
                                for t in range(K.shape[0]))))


@pytest.mark.parametrize("H,Hkv,D,dtype", [(4, 4, 4, "f32"), (8, 2, 8, "bf16")])
def test_oracle_lse_brute_force_tiny(H, Hkv, D, dtype):
    b = small_batch(H=H, Hkv=Hkv, D=D, P=4, dtype=dtype, lens=(1, 9, 40), seed=71 + D)
    hb = host_batch(b)
    ks, _ = dense_logical_kv(hb, 4)
    q = to_f64(hb["q"])
    args = [hb[k] for k in ("q", "k_pool", "v_pool", "block_table", "seq_lens")]
    r = H // Hkv
    for j, L in enumerate((1, 9, 40)):
        for h in range(H):
            for t0, t1 in ((0, L), (0, 1), (L // 2, L)):
                if t1 <= t0:
                    continue
                _, lse = oracle.decode_range(*args, j, h, t0, t1, num_kv_heads=Hkv, dtype=dtype_code(b.shape))
                ref = _brute_lse(q[j, h], ks[j, h // r][t0:t1], 1 / mp.sqrt(D))
                assert abs(lse - ref) <= 1e-12


def test_oracle_lse_closed_forms():
    b = small_batch(H=2, Hkv=2, D=8, P=4, dtype="f32", lens=(1, 13), seed=5)
    hb = host_batch(b)
    ks, _ = dense_logical_kv(hb, 4)
    q = to_f64(hb["q"])
    args = [hb[k] for k in ("q", "k_pool", "v_pool", "block_table", "seq_lens")]
    # L = 1: lse = the single score
    _, lse = oracle.decode_range(*args, 0, 1, 0, 1, num_kv_heads=2, dtype=oracle.F32)
    assert abs(lse - float(q[0, 1] @ ks[0, 1][0]) / math.sqrt(8)) <= 1e-14
    # q = 0: every score is 0, lse = ln L
    hb["q"][:] = 0
    _, lse = oracle.decode_range(*args, 1, 0, 0, 13, num_kv_heads=2, dtype=oracle.F32)
    assert abs(lse - math.log(13)) <= 1e-14


# ---------------------------------------------------------------- split + merge composition (oracle)
def _local_problem(hb, N, rank, P):
    bt = torch.from_numpy(hb["block_table"])
    lbt = seqsplit.local_block_table(bt, N, rank).numpy()
    ll = np.array([seqsplit.local_len(int(L), N, rank, P) for L in hb["seq_lens"]], dtype=np.int32)
    return lbt, ll


def _seq_split_oracle(hb, shape, N, ranks=None):
    """Per device: (o, lse) of every head over its striped pages (oracle on the local problem)."""
    B, H, D = hb["q"].shape
    out = {}
    for rank in (range(N) if ranks is None else ranks):
        lbt, ll = _local_problem(hb, N, rank, shape.page_size)
        o = np.zeros((B, H, D))
        lse = np.full((B, H), -np.inf)
        for j in range(B):
            if ll[j] == 0:
                continue
            for h in range(H):
                o[j, h], lse[j, h] = oracle.decode_range(hb["q"], hb["k_pool"], hb["v_pool"], lbt, ll, j, h, 0,
                                                         int(ll[j]), num_kv_heads=shape.num_kv_heads,
                                                         dtype=dtype_code(shape))
        out[rank] = (o, lse)
    return out


def _merge(parts):
    B, H, D = parts[0][0].shape
    o = np.zeros((B, H, D))
    for j in range(B):
        for h in range(H):
            live = [p for p in parts if np.isfinite(p[1][j, h])]
            o[j, h], _ = oracle.lse_merge(np.stack([p[0][j, h] for p in live]), np.array([p[1][j, h] for p in live]))
    return o


@pytest.mark.parametrize("N", [1, 2, 3, 8])
def test_oracle_seq_split_merge_equals_unsplit(N):
    b = small_batch(H=8, Hkv=2, D=8, P=4, dtype="bf16", lens=(1, 5, 16, 17, 61), seed=40 + N)
    hb = host_batch(b)
    ref = oracle.decode(hb["q"], hb["k_pool"], hb["v_pool"], hb["block_table"], hb["seq_lens"], num_kv_heads=2,
                        dtype=oracle.BF16)
    parts = _seq_split_oracle(hb, b.shape, N)
    assert np.max(np.abs(_merge([parts[r] for r in range(N)]) - ref)) <= 1e-13


# ---------------------------------------------------------------- two processes (gloo)
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, lens, out_q):
    # file rendezvous: no free TCP port to race for
    dist.init_process_group("gloo", init_method="file://" + port, rank=rank, world_size=world)
    try:
        b = small_batch(H=8, Hkv=4, D=8, P=4, dtype="bf16", lens=lens, seed=123)
        hb = host_batch(b)
        o, lse = _seq_split_oracle(hb, b.shape, world, ranks=[rank])[rank]
        rec = torch.cat([torch.from_numpy(o).flatten(), torch.from_numpy(lse).flatten()])
        bufs = [torch.empty_like(rec) for _ in range(world)]
        dist.all_gather(bufs, rec)
        B, H, D = o.shape
        parts = [(x[:B * H * D].view(B, H, D).numpy(), x[B * H * D:].view(B, H).numpy()) for x in bufs]
        out_q.put((rank, _merge(parts)))
    finally:
        dist.destroy_process_group()


def test_two_rank_seq_split_step_equals_unsplit():
    lens = (3, 4, 9, 40)
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    import tempfile
    port = os.path.join(tempfile.mkdtemp(), "rendezvous")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, lens, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    b = small_batch(H=8, Hkv=4, D=8, P=4, dtype="bf16", lens=lens, seed=123)
    hb = host_batch(b)
    ref = oracle.decode(hb["q"], hb["k_pool"], hb["v_pool"], hb["block_table"], hb["seq_lens"], num_kv_heads=4,
                        dtype=oracle.BF16)
    for rank, o in results:
        assert np.max(np.abs(o - ref)) <= 1e-13, rank
