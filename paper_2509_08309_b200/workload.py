"""Seeded synthetic decode workloads (shapes, lengths, paged layout).

This module is the ONE place both the CUDA path's tests/bench and the oracle
draw inputs from.  It holds none of the method's arithmetic: it only draws
random numbers, rounds them to the storage dtype, allocates pages and
NaN-poisons unused slots.  Recipe:

* Q, K, V ~ N(0, 1) drawn in fp32 from a seeded torch generator, then rounded
  to bf16 (round-to-nearest-even) or kept fp32 (config c1).
* The logical cache of kv head g is drawn from its own generator seeded with
  (seed, g), so any subset of kv heads (one rank's share) is generated
  independently and the union over ranks is the single-device problem.
* Physical page ids are a seeded random permutation of a pool with >= 10%
  slack; slack pages, tail slots past L_j and the slot of the new token
  (position L_j - 1, filled by kv_append) hold NaN.
* Unused block-table entries are -1.

Shapes come from BASELINE.json's configs (LLaMA2-13B: 40 heads x 128, MHA;
LLaMA2-70B: 64 q / 8 kv heads x 128, GQA r = 8; page size 16 following
SPEC.md:471).  Context lengths: fixed, or log-uniform in [512, 10240] for the
"mixed context lengths" config (stand-in for ShareGPT/HumanEval/LongBench
diversity).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

NAN_BF16 = 0x7FC0
NAN_F32 = 0x7FC00000


@dataclass(frozen=True)
class Shape:
    """Model-side attention shape (D9 in SURVEY.md §2.2)."""
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    page_size: int = 16
    dtype: str = "bf16"          # kv / q storage dtype: "bf16" or "f32"

    @property
    def r(self) -> int:
        """GQA group size r = H / H_kv."""
        return self.num_q_heads // self.num_kv_heads

    @property
    def torch_dtype(self) -> torch.dtype:
        return torch.bfloat16 if self.dtype == "bf16" else torch.float32

    @property
    def elem_bytes(self) -> int:
        return 2 if self.dtype == "bf16" else 4


@dataclass(frozen=True)
class Config:
    name: str
    shape: Shape
    batch: int
    seq_len: int | None                 # fixed context length (incl. the new token)
    seq_len_range: tuple[int, int] | None = None   # log-uniform [lo, hi] when seq_len is None
    split: tuple[int, ...] | None = None            # fixed per-device query-head counts, or None = even over N
    seed: int = 0
    description: str = ""
    notes: dict = field(default_factory=dict)

    def seq_lens(self) -> torch.Tensor:
        if self.seq_len is not None:
            return torch.full((self.batch,), self.seq_len, dtype=torch.int32)
        lo, hi = self.seq_len_range
        g = torch.Generator().manual_seed(self.seed * 7919 + 17)
        u = torch.rand(self.batch, generator=g, dtype=torch.float64)
        lens = torch.exp(math.log(lo) + u * (math.log(hi) - math.log(lo)))
        return lens.round().clamp(lo, hi).to(torch.int32)

    def head_split(self, n_devices: int) -> tuple[int, ...]:
        if self.split is not None and len(self.split) == n_devices:
            return self.split
        H, r = self.shape.num_q_heads, self.shape.r
        groups = H // r
        if groups % n_devices != 0:
            raise ValueError(f"{self.name}: {groups} kv groups do not split evenly over {n_devices} devices")
        return tuple([H // n_devices] * n_devices)


LLAMA2_13B = Shape(40, 40, 128, 16, "bf16")
LLAMA2_70B = Shape(64, 8, 128, 16, "bf16")

CONFIGS: dict[str, Config] = {
    "c1": Config("c1", Shape(8, 8, 64, 16, "f32"), batch=4, seq_len=128, split=(4, 4), seed=1001,
                 description="1 layer, 8 heads, head_dim 64, 4 sequences x 128 tokens, page size 16, fp32, "
                             "heads split 2 ways on one device"),
    "c2": Config("c2", LLAMA2_13B, batch=64, seq_len=4096, seed=1002,
                 description="LLaMA2-13B decode attention: 40 heads, head_dim 128, batch 64, context 4k, "
                             "bf16 paged KV, 1 GPU"),
    "c3": Config("c3", LLAMA2_70B, batch=128, seq_len=2048, seed=1003,
                 description="LLaMA2-70B-shaped GQA: 64 Q heads / 8 KV heads, head_dim 128, batch 128, "
                             "context 2k, heads sharded over 2/4/8 GPUs"),
    "c4": Config("c4", LLAMA2_13B, batch=64, seq_len=None, seq_len_range=(512, 10240), split=(16, 8, 8, 4, 4),
                 seed=1004,
                 description="Uneven Hetis-style dispatch: 40 heads split 16/8/8/4/4 across 5 GPUs, mixed "
                             "context lengths 512-10k (batch 64: our reading, unspecified upstream)"),
    "c5": Config("c5", LLAMA2_13B, batch=16, seq_len=32768, split=(5,) * 8, seed=1005,
                 description="Long-context decode: LLaMA2-13B shape, batch 16 x 32k tokens, split-KV across "
                             "8 GPUs with NVLink O all-gather"),
}


def _gen(device, seed: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def _fill_nan_(t: torch.Tensor) -> torch.Tensor:
    if t.dtype == torch.bfloat16:
        t.view(torch.int16).fill_(NAN_BF16)
    else:
        t.view(torch.int32).fill_(NAN_F32)
    return t


def _randn(shape, dtype, gen, device) -> torch.Tensor:
    return torch.randn(shape, generator=gen, device=device, dtype=torch.float32).to(dtype)


def pages_needed(seq_lens: torch.Tensor, page_size: int) -> torch.Tensor:
    return (seq_lens.to(torch.int64) + page_size - 1) // page_size


@dataclass
class DecodeBatch:
    """One rank's share of one decode step (one layer).

    q: [B][x][D] for this rank's query heads (x = q_count), k_new/v_new:
    [B][x/r][D]; k_pool/v_pool: [num_pages][P][D]; block_table:
    int32 [B][x/r][max_pages]; seq_lens: int32 [B] (length AFTER the append).
    """
    shape: Shape
    q_begin: int
    q_count: int
    q: torch.Tensor
    k_new: torch.Tensor
    v_new: torch.Tensor
    k_pool: torch.Tensor
    v_pool: torch.Tensor
    block_table: torch.Tensor
    seq_lens: torch.Tensor

    @property
    def kv_begin(self) -> int:
        return self.q_begin // self.shape.r

    @property
    def kv_count(self) -> int:
        return self.q_count // self.shape.r

    @property
    def max_seq_len(self) -> int:
        return int(self.seq_lens.max().item()) if self.seq_lens.numel() else 0


def _kv_head_stream(shape: Shape, seed: int, g: int, T: int, device):
    """K and V rows [T][D] of every cached token (all requests, positions ascending) of global kv head g."""
    gen = _gen(device, seed * 1000003 + 101 + 2 * g)
    kg = _randn((T, shape.head_dim), shape.torch_dtype, gen, device)
    vg = _randn((T, shape.head_dim), shape.torch_dtype, gen, device)
    return kg, vg


def make_new_rows(shape: Shape, seq_lens: torch.Tensor, seed: int, device="cpu", kv_begin: int = 0,
                  kv_count: int | None = None):
    """The new token's K and V rows [B][kv_count][D] of kv heads [kv_begin, kv_begin + kv_count) -- the same
    bits make_decode_batch puts in k_new / v_new, without allocating pools (the Primary's scatter input)."""
    if kv_count is None:
        kv_count = shape.num_kv_heads - kv_begin
    lens64 = seq_lens.to(torch.int64).cpu()
    B, T = int(lens64.numel()), int(lens64.sum().item())
    new_idx = (torch.cumsum(lens64, 0) - 1).to(device)                # flat index of each request's newest token
    k_new = torch.empty((B, kv_count, shape.head_dim), dtype=shape.torch_dtype, device=device)
    v_new = torch.empty_like(k_new)
    for gl in range(kv_count):
        kg, vg = _kv_head_stream(shape, seed, kv_begin + gl, T, device)
        k_new[:, gl] = kg[new_idx]
        v_new[:, gl] = vg[new_idx]
    return k_new, v_new


def make_q(shape: Shape, batch: int, seed: int, device="cpu") -> torch.Tensor:
    """Full query tensor [B][H][D] for all global heads."""
    return _randn((batch, shape.num_q_heads, shape.head_dim), shape.torch_dtype, _gen(device, seed * 1000003 + 1),
                  device)


def make_decode_batch(shape: Shape, seq_lens: torch.Tensor, seed: int, device="cpu", q_begin: int = 0,
                      q_count: int | None = None, slack: float = 0.10, rank_salt: int = 0) -> DecodeBatch:
    """Generate the paged KV cache + new-token K/V + Q for query heads [q_begin, q_begin+q_count)."""
    H, Hkv, D, P = shape.num_q_heads, shape.num_kv_heads, shape.head_dim, shape.page_size
    r = shape.r
    if q_count is None:
        q_count = H - q_begin
    if q_begin % r or q_count % r or q_count <= 0 or q_begin + q_count > H:
        raise ValueError("head range must be whole kv groups inside [0, H)")
    dt = shape.torch_dtype
    seq_lens = seq_lens.to(torch.int32).cpu()
    B = int(seq_lens.numel())
    g0, gn = q_begin // r, q_count // r
    npg = pages_needed(seq_lens, P)                       # [B]
    max_pages = max(int(npg.max().item()) if B else 1, 1)
    used = int(npg.sum().item()) * gn
    num_pages = int(math.ceil(used * (1.0 + slack))) + 1
    perm = torch.randperm(num_pages, generator=_gen("cpu", seed * 31 + 7 + 1000 * rank_salt), dtype=torch.int64)

    bt = torch.full((B, gn, max_pages), -1, dtype=torch.int32)
    # allocate pages in (seq, kv head, page) order from the permutation
    cursor = 0
    for j in range(B):
        n = int(npg[j])
        for gl in range(gn):
            bt[j, gl, :n] = perm[cursor:cursor + n].to(torch.int32)
            cursor += n

    q_full = make_q(shape, B, seed, device)
    q = q_full[:, q_begin:q_begin + q_count].contiguous()

    k_pool = _fill_nan_(torch.empty((num_pages, P, D), dtype=dt, device=device))
    v_pool = _fill_nan_(torch.empty((num_pages, P, D), dtype=dt, device=device))
    k_new = torch.empty((B, gn, D), dtype=dt, device=device)
    v_new = torch.empty((B, gn, D), dtype=dt, device=device)

    lens64 = seq_lens.to(torch.int64)
    T = int(lens64.sum().item())
    # flat token index -> (seq j, position t)
    seq_of_tok = torch.repeat_interleave(torch.arange(B, dtype=torch.int64), lens64)
    starts = torch.cumsum(lens64, 0) - lens64
    pos_of_tok = torch.arange(T, dtype=torch.int64) - starts[seq_of_tok]
    is_new = pos_of_tok == (lens64[seq_of_tok] - 1)
    hist = ~is_new
    for gl in range(gn):
        kg, vg = _kv_head_stream(shape, seed, g0 + gl, T, device)
        pages = bt[:, gl, :].to(torch.int64)                              # [B][max_pages]
        rows = pages[seq_of_tok, pos_of_tok // P] * P + pos_of_tok % P      # [T]
        rows_h = rows[hist].to(device)
        hist_d = hist.to(device)
        k_pool.view(num_pages * P, D).index_copy_(0, rows_h, kg[hist_d])
        v_pool.view(num_pages * P, D).index_copy_(0, rows_h, vg[hist_d])
        new_d = is_new.to(device)
        k_new[:, gl] = kg[new_d]
        v_new[:, gl] = vg[new_d]
    return DecodeBatch(shape, q_begin, q_count, q, k_new, v_new, k_pool, v_pool, bt.to(device),
                       seq_lens.to(device))


def to_numpy_bits(t: torch.Tensor):
    """Host numpy view of a tensor's storage: bf16 -> uint16 bits, fp32 -> float32."""
    t = t.detach().contiguous().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view("uint16")
    return t.numpy()
