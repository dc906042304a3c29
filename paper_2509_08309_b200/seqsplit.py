"""Sequence-wise split of decode attention across devices (row f3).

The design the paper argues against (PAPER.md:292-304 `fig:head_wise_advantage`,
:356-358): instead of giving each device a subset of the heads (Hetis), every
device attends ALL heads over a subset of each request's tokens, and the
partial results are merged with their per-head log-sum-exp ("aggregate global
softmax attributes").  It exists here to measure that comparison on B200 /
NVLink (scripts/seq_vs_head_probe.py).

Layout (reading f3, "page striping"): page k of every (request, kv
head) lives on device k mod N.  A device's block table is the global table's
columns rank, rank + N, ... -- so only its last page can be partial, the
newest token always lands on the device holding page ceil(L/P) - 1, and no
page moves as the request grows.  Page allocation stays the caller's job
(SURVEY.md §8 a0); this module only holds the host-side bookkeeping of that
layout.  Every per-step computation runs in libhetis.so:

    hetis_seq_broadcast_q       q of all heads (+ new k, v) to every device (NCCL)
    hetis_seq_split_lens        local token counts / append lengths (kernel)
    hetis_kv_append             the owner of the newest page stores the new rows
    hetis_attn_partial          split-KV attention over the local pages
    hetis_attn_combine_lse      local o and lse per head
    hetis_seq_allgather_merge   all-gather of (o, lse) + the LSE merge (NCCL + kernel)
"""
from __future__ import annotations

import torch

from . import hetis, workload


def local_len(L: int, num_ranks: int, rank: int, page_size: int) -> int:
    """Tokens of a length-L request held by `rank` (pages k = rank, rank + N, ... < ceil(L/P))."""
    np_ = (L + page_size - 1) // page_size
    mine = (np_ - 1 - rank) // num_ranks + 1 if np_ > rank else 0
    owns_last = np_ > 0 and (np_ - 1) % num_ranks == rank
    return mine * page_size - ((np_ * page_size - L) if owns_last else 0)


def owner_of_newest(L: int, num_ranks: int, page_size: int) -> int:
    """Device that stores the token at position L - 1."""
    return ((L + page_size - 1) // page_size - 1) % num_ranks


def local_pages(num_pages: int, num_ranks: int, rank: int) -> int:
    """How many of pages 0 .. num_pages-1 device `rank` holds (pages rank, rank + N, ...)."""
    return (num_pages - 1 - rank) // num_ranks + 1 if num_pages > rank else 0


def local_block_table(block_table: torch.Tensor, num_ranks: int, rank: int) -> torch.Tensor:
    """This device's table [B][G][max(1, local_pages(max_pages))]: the global columns rank, rank + N,
    ... (entries past a request's pages keep the global table's -1; one -1 column if it holds none)."""
    t = block_table[:, :, rank::num_ranks]
    if t.shape[2] == 0:
        return torch.full((*block_table.shape[:2], 1), -1, dtype=block_table.dtype, device=block_table.device)
    return t.contiguous()


def comm_bytes(num_seqs: int, shape: workload.Shape, num_ranks: int, o_bytes: int = 4) -> dict:
    """Bytes one non-root device receives per step, sequence split vs head split (both all-gather O).

    sequence split: q of all heads + new k, v of all kv heads (broadcast), then the all-gather of
    every other device's (o, lse) for all heads;  head split (Eq. 4): q of its H/N
    heads + new k, v of its kv heads, then the all-gather of the other devices' O shards."""
    B, H, Hkv, D, e = num_seqs, shape.num_q_heads, shape.num_kv_heads, shape.head_dim, shape.elem_bytes
    N = num_ranks
    seq_in = B * (H + 2 * Hkv) * D * e
    seq_out = (N - 1) * B * H * (D + 1) * 4
    head_in = B * (H + 2 * Hkv) * D * e // N
    head_out = (N - 1) * B * (H // N) * D * o_bytes
    return {"seq_in": seq_in, "seq_out": seq_out, "head_in": head_in, "head_out": head_out}


class SeqSplitStep:
    """One device's decode step of one layer under the sequence split.

    q, k_new, v_new: [B][H][D] / [B][H_kv][D] buffers every device holds (filled by
    broadcast from `root`); the pools and the global block table are this device's
    (only its striped columns are read)."""

    def __init__(self, shape: workload.Shape, num_ranks: int, rank: int, num_seqs: int, max_seq_len: int, device,
                 o_dtype: str = "f32", comm_ptr: int | None = None, root: int = 0):
        self.shape = shape
        self.cshape = hetis.make_shape(shape, o_dtype)
        self.N, self.rank, self.root, self.comm_ptr = num_ranks, rank, root, comm_ptr
        self.B = num_seqs
        P = shape.page_size
        # the longest local length: this device's share of the longest request's pages
        self.max_local = max(1, local_pages((max_seq_len + P - 1) // P, num_ranks, rank) * P)
        H, Hkv, D = shape.num_q_heads, shape.num_kv_heads, shape.head_dim
        dt = shape.torch_dtype
        self.q = torch.empty((num_seqs, H, D), dtype=dt, device=device)
        self.k_new = torch.empty((num_seqs, Hkv, D), dtype=dt, device=device)
        self.v_new = torch.empty((num_seqs, Hkv, D), dtype=dt, device=device)
        self.local_lens = torch.zeros(num_seqs, dtype=torch.int32, device=device)
        self.append_lens = torch.zeros(num_seqs, dtype=torch.int32, device=device)
        rows = num_seqs * H
        self.part = torch.empty(rows * (D + 1), dtype=torch.float32, device=device)   # o | lse
        self.part_o = self.part[:rows * D].view(num_seqs, H, D)
        self.part_lse = self.part[rows * D:].view(num_seqs, H)
        self.staging = torch.empty((num_ranks, rows * (D + 1)), dtype=torch.float32, device=device) \
            if num_ranks > 1 else None
        self.workspace = hetis.alloc_workspace(hetis.attn_decode_workspace(self.cshape, num_seqs, H, self.max_local),
                                               device)
        self.o_dtype = torch.bfloat16 if o_dtype == "bf16" else torch.float32

    def launches_per_step(self) -> int:
        return 5 if self.N > 1 else 4   # lens, append, partial, combine_lse [, merge]

    def broadcast(self, stream=None):
        hetis.seq_broadcast_q(self.cshape, self.comm_ptr, self.N, self.rank, self.root, self.q, self.k_new,
                              self.v_new, stream)

    def run(self, k_pool, v_pool, local_bt, seq_lens, o, stream=None, flags: int = 0):
        """lens -> append (owner only) -> partial -> combine_lse -> [all-gather + merge] -> o [B][H][D]."""
        hetis.seq_split_lens(self.N, self.rank, self.shape.page_size, seq_lens, self.local_lens, self.append_lens,
                             stream)
        hetis.kv_append(self.cshape, self.k_new, self.v_new, k_pool, v_pool, local_bt, self.append_lens, stream)
        hetis.attn_partial(self.cshape, self.q, k_pool, v_pool, local_bt, self.local_lens, self.max_local,
                           self.workspace, flags=flags, stream=stream)
        hetis.attn_combine_lse(self.cshape, self.local_lens, self.max_local, self.part_o, self.part_lse,
                               self.workspace, stream=stream)
        if self.N > 1:
            hetis.seq_allgather_merge(self.cshape, self.comm_ptr, self.N, self.rank, self.B, self.part, self.staging,
                                      o, stream)
        else:
            hetis.seq_merge(self.cshape, self.part_o.unsqueeze(0), self.part_lse.unsqueeze(0), o, stream)
        return o
