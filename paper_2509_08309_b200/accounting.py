"""Byte / FLOP accounting for the roofline and the comm-volume model.

Definitions:

* KV bytes read by one decode step of one layer on one device holding
  kv heads G:  sum_j L_j * |G| * d * 2 (K and V) * sizeof(kv)   -- the dominant
  term; decode attention must read every cached K/V byte once.
* algorithmic bytes = KV bytes + Q read + O written + block-table entries
  read + seq_lens read.
* comm volume per sequence and layer (Eq. 4):
  d_i = (2 + 2/r) * h_i head-vectors (q and o per query head, k and v shared by r).
"""
from __future__ import annotations

from dataclasses import dataclass


def kv_cache_bytes(layers: int, kv_heads: int, head_dim: int, elem_bytes: int, tokens: int) -> int:
    """Total K+V bytes of `tokens` cached tokens (PAPER.md:64 closed form check)."""
    return 2 * layers * kv_heads * head_dim * elem_bytes * tokens


@dataclass(frozen=True)
class StepBytes:
    kv: int
    q: int
    o: int
    table: int
    seq_lens: int
    new_kv: int

    @property
    def attention(self) -> int:
        """Algorithmic bytes of the attention kernel (a4): KV + Q + O + table + seq_lens."""
        return self.kv + self.q + self.o + self.table + self.seq_lens


def step_bytes(seq_lens, q_heads: int, r: int, head_dim: int, page_size: int, kv_elem_bytes: int,
               q_elem_bytes: int, o_elem_bytes: int) -> StepBytes:
    lens = [int(x) for x in seq_lens]
    kv_heads = q_heads // r
    tokens = sum(lens)
    pages = sum((L + page_size - 1) // page_size for L in lens)
    B = len(lens)
    return StepBytes(
        kv=tokens * kv_heads * head_dim * 2 * kv_elem_bytes,
        q=B * q_heads * head_dim * q_elem_bytes,
        o=B * q_heads * head_dim * o_elem_bytes,
        table=pages * kv_heads * 4,
        seq_lens=B * 4,
        new_kv=B * kv_heads * head_dim * 2 * kv_elem_bytes,
    )


def comm_head_vectors(h: int, r: int) -> float:
    """Eq. 4: d_i = (2 + 2/r) * h_i head-vectors moved per sequence per layer."""
    return (2.0 + 2.0 / r) * h


def attention_flops(seq_lens, q_heads: int, head_dim: int) -> int:
    """2 flops per MAC for q.k and for p.v: 4 * L * H * d per sequence."""
    return sum(4 * int(L) * q_heads * head_dim for L in seq_lens)
